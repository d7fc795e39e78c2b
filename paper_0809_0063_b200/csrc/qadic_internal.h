// Host-side internals shared by the translation units of libqadic_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qadic_b200.h"

namespace qadic {

// operand-plane reuse across successive GF matmul calls (fp4k engine; see run_kara)
enum : int { REUSE_B_READY = 1, REUSE_COL_PANEL = 2, REUSE_A_READY = 4, F64_TWO_SIDED = 8 };  // + F64 engine form

// RU(1/p): the smallest double >= 1/p (fdiv.py:166-180, mode UP).
double host_reciprocal_up(int64_t p);
// First r at which floor(RN(r*RU(1/p))) may exceed floor(r/p) -- the fdiv
// case-2 bound for beta = 53 (fdiv.py:250-260, 317-335): 3002399751580331.
double host_case2_bound();

void set_error(int code, const char* fmt, ...);
// keep the current device's stream-ordered pool from returning freed blocks to the
// OS at every synchronisation (cudaMallocAsync scratch reused across calls)
void keep_mempool();
// multiprocessor count of the current device (cached per device)
int num_sms_cached();
// `launched`: kernels this call site launched outside QADIC_TIMED (those count themselves)
int check_launch(const char* what, int launched);
void count_launch(int n = 1);
int prof_begin(cudaStream_t s, const char* name);
void prof_end(int idx, cudaStream_t s);

// PDL launches are on unless QADIC_NO_PDL=1
bool pdl_enabled();
// the batched kernels' L2 prefetch ahead of pdl_wait() (qadic_common.cuh), on with PDL
int pdl_prefetch_enabled();

// Launch with programmatic stream serialisation (see pdl_wait in qadic_common.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace qadic

// launch a kernel bracketed by the (optional) per-kernel event timer
#define QADIC_TIMED(name, stream, ...)                          \
    do {                                                        \
        int _qadic_pi = ::qadic::prof_begin((stream), (name));  \
        ::qadic::count_launch(1);                               \
        __VA_ARGS__;                                            \
        ::qadic::prof_end(_qadic_pi, (stream));                 \
    } while (0)
