// Tensor-pipe peak probes (diagnostics; BASELINE.md section 2 asks for measured
// FP64 DMMA and tcgen05 pipe peaks next to the nominal datasheet figures).
//
// Each probe keeps its operands on chip, so the number is the pipe's own
// throughput on this board under its power management -- no HBM, no L2, no
// TMA traffic:
//   kind 0  tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32, M=256 N=256 K=64
//           (the fp4k / fp4 engines' instruction), one CTA pair per two SMs,
//           operands resident in shared memory;
//   kind 1  tcgen05.mma.cta_group::2.kind::i8, M=256 N=256 K=32 (the i8 engine);
//   kind 2  mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4, the f64 engine),
//           operands in registers, 8 independent accumulator chains per warp.
// `data` picks the operand bits, which set the power draw and with it the
// clock the power cap allows: 0 = zeros, 1 = residue-like values (E2M1 codes of
// 0..6, bytes 0..6, integers < 2^17 for f64 -- what the engines feed), 2 =
// full-range random bits.
#include "qadic_common.cuh"
#include "qadic_internal.h"
#include "sm100_ptx.cuh"

namespace qadic {
namespace probe {

constexpr int MMA_THREADS = 128;
constexpr int ROWS = 128;      // A rows per CTA (pair M = 256) and B rows per CTA (pair N = 256)
constexpr int ROW_BYTES = 128;  // one 128B-swizzled K-major row: 4 MMAs of 32 bytes
constexpr int TILE_BYTES = ROWS * ROW_BYTES;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// operand word i: zeros, residue-like, or full-range random bits
__device__ __forceinline__ uint32_t operand_word(int kind, int data, uint32_t i) {
    if (data == 0) return 0u;
    const uint32_t h = mix32(i * 0x9E3779B9u + 0x632BE5ABu);
    if (data == 2) return h;
    uint32_t w = 0;
    if (kind == 0) {  // 8 E2M1 nibbles, non-negative codes 0..7 (values 0 .. 6)
#pragma unroll
        for (int j = 0; j < 8; ++j) w |= (((h >> (3 * j)) * 7u >> 3) & 7u) << (4 * j);
        return w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) w |= (((h >> (8 * j)) & 0xFFu) * 7u >> 8) << (8 * j);  // bytes 0..6
    return w;
}

template <int KIND>  // 0 mxf4, 1 i8
__global__ void __launch_bounds__(MMA_THREADS, 1) mma_peak_kernel(int64_t iters, int data) {
    using namespace sm100;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;
    uint8_t* sb = smem + TILE_BYTES;
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + 2 * TILE_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_ctarank();

    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 2 * TILE_BYTES / 4; i += MMA_THREADS)
        w[i] = operand_word(KIND, data, (uint32_t)(blockIdx.x * (2 * TILE_BYTES / 4) + i));
    // generic-proxy stores -> visible to the tensor core's async-proxy reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    constexpr uint32_t SF_COL = 256;  // accumulator in columns 0..255, scale factors after it
    if (KIND == 0) {
        tmem_fill_sf(tmem_base + ((uint32_t)(warp * 32) << 16) + SF_COL, 0x7F7F7F7Fu);
        tc_fence_before();
    }
    cluster_sync();
    tc_fence_after();

    if (rank == 0 && warp == 0) {
        if (elect_one()) {
            const uint32_t idesc = KIND == 0 ? idesc_mxf4(256, 256) : idesc_u8_s32(256, 256);
            const uint32_t a0 = smem_addr(sa), b0 = smem_addr(sb);
            for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
                for (int k = 0; k < ROW_BYTES / 32; ++k) {
                    const uint64_t ad = smem_desc_k_sw128(a0 + k * 32), bd = smem_desc_k_sw128(b0 + k * 32);
                    if (KIND == 0) umma_mxf4_pair(tmem_base, ad, bd, idesc, 1u, tmem_base + SF_COL, tmem_base + SF_COL);
                    else umma_i8_pair(tmem_base, ad, bd, idesc, 1u);
                }
            }
            umma_commit_pair(done, 0x3);
        }
        __syncwarp();
    }
    mbar_wait(done, 0);
    tc_fence_after();
    cluster_sync();
    if (warp == 0) tmem_dealloc_pair<512>(tmem_base);
}

constexpr int DMMA_THREADS = 256;
constexpr int CHAINS = 8;

__global__ void __launch_bounds__(DMMA_THREADS) dmma_peak_kernel(int64_t iters, int data, double* sink) {
    const uint32_t i = blockIdx.x * DMMA_THREADS + threadIdx.x;
    double a = 0.0, b = 0.0;
    if (data == 1) {  // DQT-word-like integers < 2^17
        a = (double)(mix32(2 * i) >> 15);
        b = (double)(mix32(2 * i + 1) >> 15);
    } else if (data == 2) {  // full 53-bit random mantissas in [1, 2)
        a = 1.0 + (double)(mix32(2 * i) >> 1) * 0x1p-31;
        b = 1.0 + (double)(mix32(2 * i + 1) >> 1) * 0x1p-31;
    }
    double c[CHAINS][2];
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) c[j][0] = c[j][1] = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < CHAINS; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1];
    if (s == -1.0) sink[i] = s;  // never true; keeps the chains live
}

}  // namespace probe
}  // namespace qadic

extern "C" QADIC_API int qadic_diag_pipe_peak(int32_t kind, int32_t data, int64_t iters, double* ops, float* ms,
                                              void* stream) {
    using namespace qadic;
    using namespace qadic::probe;
    if (kind < 0 || kind > 2 || data < 0 || data > 2 || iters <= 0 || ops == nullptr || ms == nullptr) {
        set_error(QADIC_ERR_VALUE, "pipe_peak: kind %d data %d iters %lld", kind, data, (long long)iters);
        return QADIC_ERR_VALUE;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int sms = num_sms_cached();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t err;
    if (kind < 2) {
        // more than half an SM's shared memory: exactly one CTA (one TMEM
        // allocation) per SM, so the grid covers every SM once
        const size_t smem = 150 * 1024;
        auto kern = kind == 0 ? mma_peak_kernel<0> : mma_peak_kernel<1>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = sms / 2 * 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(MMA_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaEventRecord(e0, s);
        err = cudaLaunchKernelEx(&cfg, kern, iters, (int)data);
        cudaEventRecord(e1, s);
        const double per_mma = kind == 0 ? 2.0 * 256 * 256 * 64 : 2.0 * 256 * 256 * 32;
        *ops = (double)(grid / 2) * (double)iters * (ROW_BYTES / 32) * per_mma;
    } else {
        const int grid = sms * 4;
        double* sink = nullptr;
        cudaMallocAsync(&sink, sizeof(double) * grid * DMMA_THREADS, s);
        cudaEventRecord(e0, s);
        dmma_peak_kernel<<<grid, DMMA_THREADS, 0, s>>>(iters, data, sink);
        err = cudaGetLastError();
        cudaEventRecord(e1, s);
        cudaFreeAsync(sink, s);
        *ops = (double)grid * (DMMA_THREADS / 32) * (double)iters * CHAINS * (2.0 * 8 * 8 * 4);
    }
    count_launch(1);
    if (err == cudaSuccess) err = cudaEventSynchronize(e1);
    float t = 0.f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (err != cudaSuccess) {
        set_error(QADIC_ERR_CUDA, "pipe_peak: %s", cudaGetErrorString(err));
        return QADIC_ERR_CUDA;
    }
    *ms = t;
    return QADIC_OK;
}

// ---------------------------------------------------------------------------
// Same-size copy ceiling for the single-wave batched kernels (diagnostics): out
// = a ^ b over 16-byte vectors -- the cfg1 / cfg2 traffic shape (two input
// streams, one output stream, no arithmetic worth the name), launched like
// those kernels (one balanced wave, programmatic dependent launch), so a CUDA
// graph of back-to-back calls measures what a call of that size can reach.
// ---------------------------------------------------------------------------
namespace qadic {
namespace probe {
template <int V>
__global__ void copy_like_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, int64_t n_in,
                                 uint4* __restrict__ out, int64_t n_out, int pf) {
    if (pf && threadIdx.x == 0) {  // as in the batched kernels: the block's inputs towards L2 before the wait
        const int64_t off = (int64_t)blockIdx.x * blockDim.x * V * 16, len = (int64_t)blockDim.x * V * 16;
        l2_prefetch_span(a, off, len, n_in * 16);
        l2_prefetch_span(b, off, len, n_in * 16);
    }
    pdl_wait();
    pdl_trigger();
    const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
    uint4 x[V], y[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        x[v] = j0 + v < n_in ? __ldg(a + j0 + v) : make_uint4(0, 0, 0, 0);
        y[v] = j0 + v < n_in ? __ldg(b + j0 + v) : make_uint4(0, 0, 0, 0);
    }
    // the output stream (n_out <= 2 n_in vectors) in two coalesced halves: vector i of
    // the inputs writes out[i] and out[n_in + i] (an earlier form wrote each thread's
    // n_out / n_in share contiguously -- lanes 1.75 vectors apart at cfg1's shape, a
    // partial-sector store pattern that made this ceiling slow)
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int64_t i = j0 + v;
        const uint4 p = x[v], q = y[v];
        if (i < n_out) out[i] = make_uint4(p.x ^ q.x, p.y ^ q.y, p.z ^ q.z, p.w ^ q.w);
        if (n_in + i < n_out) out[n_in + i] = make_uint4(p.x + q.x, p.y + q.y, p.z + q.z, p.w + q.w);
    }
}
}  // namespace probe
}  // namespace qadic

extern "C" QADIC_API int qadic_diag_copy(const void* a, const void* b, int64_t in_bytes, void* out, int64_t out_bytes,
                                         int32_t per_thread, int32_t threads, void* stream) {
    using namespace qadic;
    using namespace qadic::probe;
    if (in_bytes % 16 || out_bytes % 16 || out_bytes > 2 * in_bytes || threads < 32 || threads > 1024 ||
        !(per_thread == 1 || per_thread == 2 || per_thread == 4 || per_thread == 8)) {
        set_error(QADIC_ERR_VALUE, "diag_copy: bad geometry");
        return QADIC_ERR_VALUE;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n_in = in_bytes / 16, n_out = out_bytes / 16;
    const unsigned blocks = (unsigned)((n_in + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread));
    const uint4* pa = static_cast<const uint4*>(a);
    const uint4* pb = static_cast<const uint4*>(b);
    uint4* po = static_cast<uint4*>(out);
    cudaError_t e;
    const int pf = pdl_prefetch_enabled();
    switch (per_thread) {
        case 1: e = launch_pdl(copy_like_kernel<1>, dim3(blocks), dim3(threads), 0, s, pa, pb, n_in, po, n_out, pf); break;
        case 2: e = launch_pdl(copy_like_kernel<2>, dim3(blocks), dim3(threads), 0, s, pa, pb, n_in, po, n_out, pf); break;
        case 4: e = launch_pdl(copy_like_kernel<4>, dim3(blocks), dim3(threads), 0, s, pa, pb, n_in, po, n_out, pf); break;
        default: e = launch_pdl(copy_like_kernel<8>, dim3(blocks), dim3(threads), 0, s, pa, pb, n_in, po, n_out, pf); break;
    }
    (void)e;
    return check_launch("diag_copy", 1);
}
