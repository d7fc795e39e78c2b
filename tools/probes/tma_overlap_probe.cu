// Probe: does TMA accept a tensor map whose row stride (16 B) is smaller than its
// row extent (256 B) -- overlapping rows, i.e. a Toeplitz-like view of one buffer?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_overlap_probe tma_overlap_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void probe(const __grid_constant__ CUtensorMap map, const uint8_t* src, int r0, int* bad) {
    __shared__ __align__(1024) uint8_t tile[8 * 128];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(8 * 128));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(tile)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(sb), "r"(0), "r"(r0), "r"(1)
            : "memory");
    }
    __syncthreads();
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(sb));
    for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) {
        const int row = i / 128, c = i % 128;
        const uint8_t want = src[32768 + (r0 + row) * 16 + c];
        if (tile[i] != want) atomicAdd(bad, 1);
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    uint8_t* d;
    int* bad;
    cudaMalloc(&d, 65536);
    cudaMalloc(&bad, 4);
    uint8_t h[65536];
    for (int i = 0; i < 65536; ++i) h[i] = (uint8_t)((i * 7 + (i >> 8)) & 0xFF);
    cudaMemcpy(d, h, 65536, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Enc enc = (Enc)fn;
    for (int sw = 0; sw < 2; ++sw) {
        CUtensorMap map;
        cuuint64_t dims[3] = {256, 1000, 2};
        cuuint64_t strides[2] = {16, 32768};
        cuuint32_t box[3] = {128, 8, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("swizzle %d: encode -> %d\n", sw, (int)r);
        if (r != CUDA_SUCCESS) continue;
        cudaMemset(bad, 0, 4);
        probe<<<1, 128>>>(map, d, 37, bad);
        cudaError_t e = cudaDeviceSynchronize();
        int hb = -1;
        cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("swizzle %d: kernel %s, mismatches %d (swizzled layouts mismatch by design)\n", sw, cudaGetErrorString(e), hb);
    }
    return 0;
}
