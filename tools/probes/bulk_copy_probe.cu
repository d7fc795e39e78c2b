// Probe: can bulk TMA (cp.async.bulk, one instruction per block-sized chunk) beat the
// plain 16-byte-load copy ceiling of a ~16 MB single-wave step (cfg1 / cfg2 traffic)?
// Same harness as tools/small_copy_floor.py: 16 rotating buffer sets, 2000 launches in a graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_copy_probe bulk_copy_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// reads a and b (n_in vectors each), writes n_out <= 2 n_in vectors: out[i] = a[i] ^ b[i],
// out[n_in + i] = a[i] + b[i]
__global__ void plain_copy(const uint4* a, const uint4* b, int64_t n_in, uint4* out, int64_t n_out) {
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
        if (i < n_in) {
            uint4 x = a[i], y = b[i];
            if (i < n_out) out[i] = make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w);
            if (n_in + i < n_out) out[n_in + i] = make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
        }
    }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one block per chunk: bulk-load its a and b chunks into smem, XOR, bulk-store its out chunk
__global__ void bulk_copy(const uint8_t* a, const uint8_t* b, int64_t in_b, uint8_t* out, int64_t out_b, int chunk,
                          int ochunk) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint8_t* sa_ = sm;
    uint8_t* sb_ = sm + chunk;
    uint8_t* so_ = sm + 2 * chunk;  // output staging (ochunk bytes)
    const int64_t off = (int64_t)blockIdx.x * chunk;
    const int bytes = (int)(chunk < in_b - off ? (int64_t)chunk : in_b - off);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(2 * bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sa_)), "l"(a + off), "r"(bytes), "r"(sa(&bar)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sb_)), "l"(b + off), "r"(bytes), "r"(sa(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(sa(&bar)));
    const int64_t ooff = (int64_t)blockIdx.x * ochunk;
    const int obytes = (int)(out_b - ooff <= 0 ? 0 : (ochunk < out_b - ooff ? (int64_t)ochunk : out_b - ooff));
    uint4* o4 = reinterpret_cast<uint4*>(so_);
    const int nv = bytes / 16;
    for (int i = threadIdx.x; i < obytes / 16; i += blockDim.x) {
        const int k = i % nv;  // the output chunk is formed from the block's own inputs
        const uint4 x = reinterpret_cast<const uint4*>(sa_)[k], y = reinterpret_cast<const uint4*>(sb_)[k];
        o4[i] = i < nv ? make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w) : make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (threadIdx.x == 0 && obytes > 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + ooff), "r"(sa(so_)),
                     "r"(obytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;");
    }
}

int main() {
    const int sets = 16, K = 2000;
    struct Shape { const char* name; int64_t in_b, out_b; } shapes[2] = {{"cfg1", 4 << 20, 7 << 20}, {"cfg2", 8 << 20, 128 << 10}};
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (auto& sh : shapes) {
        uint8_t *A[16], *B[16], *O[16];
        for (int i = 0; i < sets; ++i) {
            cudaMalloc(&A[i], sh.in_b); cudaMalloc(&B[i], sh.in_b); cudaMalloc(&O[i], sh.out_b);
            cudaMemset(A[i], 1, sh.in_b); cudaMemset(B[i], 2, sh.in_b);
        }
        cudaStream_t s;
        cudaStreamCreate(&s);
        for (int mode = 0; mode < 3; ++mode) {
            int blocks_per_sm = mode == 2 ? 2 : 1;
            int nblk = sms * blocks_per_sm;
            int chunk = (int)(((sh.in_b + nblk - 1) / nblk + 15) / 16 * 16);
            int ochunk = (int)(((sh.out_b + nblk - 1) / nblk + 15) / 16 * 16);
            if (mode > 0) {
                int smem = 2 * chunk + ochunk;
                cudaFuncSetAttribute(bulk_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (smem > 227 * 1024) { printf("%s mode %d: chunk too big\n", sh.name, mode); continue; }
            }
            // one eager launch first, checked, before any graph
            if (mode == 0) {
                int64_t n = sh.in_b / 16;
                plain_copy<<<(unsigned)((n + 255) / 256), 128, 0, s>>>((uint4*)A[0], (uint4*)B[0], n, (uint4*)O[0], sh.out_b / 16);
            } else {
                bulk_copy<<<nblk, 256, 2 * chunk + ochunk, s>>>(A[0], B[0], sh.in_b, O[0], sh.out_b, chunk, ochunk);
            }
            cudaError_t err = cudaStreamSynchronize(s);
            if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
                printf("%s mode %d: eager launch failed: %s\n", sh.name, mode, cudaGetErrorString(err));
                return 1;
            }
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ge = nullptr;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < K; ++k) {
                int i = k % sets;
                if (mode == 0) {
                    int64_t n = sh.in_b / 16;
                    plain_copy<<<(unsigned)((n + 255) / 256), 128, 0, s>>>((uint4*)A[i], (uint4*)B[i], n, (uint4*)O[i], sh.out_b / 16);
                } else {
                    bulk_copy<<<nblk, 256, 2 * chunk + ochunk, s>>>(A[i], B[i], sh.in_b, O[i], sh.out_b, chunk, ochunk);
                }
            }
            if (cudaStreamEndCapture(s, &g) != cudaSuccess || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
                printf("%s mode %d: graph failed: %s\n", sh.name, mode, cudaGetErrorString(cudaGetLastError()));
                return 1;
            }
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaStreamSynchronize(s);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double us = ms * 1e3 / K;
            double gbs = (2.0 * sh.in_b + sh.out_b) / (us * 1e-6) / 1e9;
            printf("%s %s: %.3f us  %.1f GB/s (%s)\n", sh.name, mode == 0 ? "plain 16B loads" : (mode == 1 ? "bulk TMA 1/SM" : "bulk TMA 2/SM"), us, gbs,
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
    }
    return 0;
}
