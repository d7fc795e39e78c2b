// Layer K of the qadic operator API on B200: the five reference kernels
// (src/_kernels/_speed.pyx) with identical integer semantics, plus the bulk
// REDQ reduction (src/redq.py:318-343), the DQT row packers
// (src/cmm.py:72-85, 130-145) and the handle <-> coefficient gathers
// (src/gfext.py:136-146).
//
// These are exact-semantics primitives (uint64 wrap-around GEMM, any-width
// REDQ); the throughput engines for the configs live in engine_i8.cu,
// engine_f64.cu and batched.cu, behind the operation-level API where the
// parameters prove the digit bounds.
#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

// ---------------------------------------------------------------------------
// uint64 GEMM, wraps mod 2^64 (_speed.pyx:15-30).  64x64 tile, 4x4 per thread.
// ---------------------------------------------------------------------------
constexpr int MM_T = 64, MM_K = 16;

template <typename T>
__global__ void __launch_bounds__(256) mm_wrap_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                      T* __restrict__ c, int64_t m, int64_t k,
                                                      int64_t n, int64_t p, int64_t chunk) {
    __shared__ T sa[MM_K][MM_T + 1];
    __shared__ T sb[MM_K][MM_T];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t row0 = (int64_t)blockIdx.y * MM_T, col0 = (int64_t)blockIdx.x * MM_T;
    // unsigned accumulation == two's-complement wrap for both T
    uint64_t acc[4][4] = {}, tot[4][4] = {};
    const bool modular = p > 0;
    const int64_t step = modular ? chunk : k;
    for (int64_t kc = 0; kc < k; kc += step) {
        const int64_t kend = (kc + step < k) ? kc + step : k;
        for (int64_t k0 = kc; k0 < kend; k0 += MM_K) {
            for (int i = threadIdx.x; i < MM_K * MM_T; i += 256) {
                int kk = i % MM_K, r = i / MM_K;
                int64_t gr = row0 + r, gk = k0 + kk;
                sa[kk][r] = (gr < m && gk < kend) ? a[gr * k + gk] : T(0);
                int cc = i % MM_T, kr = i / MM_T;
                int64_t gc = col0 + cc, gk2 = k0 + kr;
                sb[kr][cc] = (gc < n && gk2 < kend) ? b[gk2 * n + gc] : T(0);
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < MM_K; ++kk) {
                uint64_t av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) av[i] = (uint64_t)sa[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = (uint64_t)sb[kk][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
            }
            __syncthreads();
        }
        if (modular) {  // c = (c + chunk_product) mod p, floor semantics (numpy %)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    int64_t v = (int64_t)(tot[i][j] + acc[i][j]);
                    int64_t r = v % p;
                    if (r != 0 && ((r < 0) != (p < 0))) r += p;
                    tot[i][j] = (uint64_t)r;
                    acc[i][j] = 0;
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t gr = row0 + ty * 4 + i;
        if (gr >= m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t gc = col0 + tx * 4 + j;
            if (gc < n) c[gr * n + gc] = (T)(modular ? tot[i][j] : acc[i][j]);
        }
    }
}

// ---------------------------------------------------------------------------
// full 1-D convolution (_speed.pyx:85-102): one thread per output index.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void conv_kernel(const T* __restrict__ a, int64_t na, const T* __restrict__ b, int64_t nb,
                            T* __restrict__ out) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= na + nb - 1) return;
    const int64_t i0 = o - nb + 1 > 0 ? o - nb + 1 : 0;
    const int64_t i1 = o < na - 1 ? o : na - 1;
    uint64_t s = 0;
    for (int64_t i = i0; i <= i1; ++i) s += (uint64_t)a[i] * (uint64_t)b[o - i];
    out[o] = (T)s;
}

// ---------------------------------------------------------------------------
// REDQ compression for arbitrary uint64 words (_speed.pyx:121-130).
// r < 2^53: FP64 reciprocal division (fdiv case 2, cold correction);
// otherwise exact integer division.  mode 0: raw u digits; mode 1: corrected
// digits (redq.py:308-315); mode 2: corrected and repacked (redq.py:318-332).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t div_p(uint64_t r, uint64_t p, double invp_up, double bound) {
    if (r < (1ull << 53)) {
        const double rd = (double)r;
        return (uint64_t)fdiv_floor(rd, invp_up, (double)p, bound);
    }
    return r / p;
}

__global__ void redq_words_kernel(const uint64_t* __restrict__ r, int64_t n, uint64_t p, int t, int d,
                                  double invp_up, double bound, uint64_t corr, int mode,
                                  uint64_t* __restrict__ digits, uint64_t* __restrict__ packed) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const uint64_t ri = r[idx];
    const uint64_t s = div_p(ri, p, invp_up, bound);
    uint64_t prev = ri - p * s;  // u_0
    uint64_t word = 0;
    for (int i = 0; i <= d; ++i) {
        const uint64_t next = (i < d) ? (ri >> ((i + 1) * t)) - p * (s >> ((i + 1) * t)) : 0;
        uint64_t out = prev;
        if (mode >= 1 && i < d) out = (prev + corr * next) % p;
        if (digits) digits[idx * (d + 1) + i] = out;
        if (mode == 2) word += out << (i * t);
        prev = next;
    }
    if (packed) packed[idx] = word;
}

// ---------------------------------------------------------------------------
// DQT row packing (cmm.py:72-85) and unpacking (cmm.py:130-145).
// ---------------------------------------------------------------------------
__global__ void pack_rows_kernel(const uint8_t* __restrict__ m, int64_t rows, int64_t cols, int k, int t,
                                 int reverse, uint64_t* __restrict__ words) {
    const int64_t width = (cols + k - 1) / k;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * width) return;
    const int64_t r = idx / width, g = idx % width;
    uint64_t w = 0;
    for (int j = 0; j < k; ++j) {
        const int64_t c = g * k + j;
        if (c < cols) {
            const int e = reverse ? (k - 1 - j) : j;
            w += (uint64_t)m[r * cols + c] << (e * t);
        }
    }
    words[idx] = w;
}

__global__ void unpack_rows_kernel(const uint64_t* __restrict__ words, int64_t rows, int64_t cols, int k,
                                   int t, int reverse, uint8_t* __restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * cols) return;
    const int64_t width = (cols + k - 1) / k;
    const int64_t r = idx / cols, c = idx % cols;
    const int j = (int)(c % k);
    const int e = reverse ? (k - 1 - j) : j;
    const uint64_t w = words[r * width + c / k];
    out[idx] = (uint8_t)((w >> (e * t)) & ((1ull << t) - 1));
}

// ---------------------------------------------------------------------------
// handle <-> coefficient conversion (gfext.py:136-146, 347-358)
// ---------------------------------------------------------------------------
__global__ void gather_u8_kernel(const int64_t* __restrict__ idx, int64_t n, const uint8_t* __restrict__ table,
                                 int64_t table_rows, int width, uint8_t* __restrict__ out) {
    // indices are range-checked by the caller (gfext.py:326-328 semantics);
    // an out-of-range handle maps to the zero element rather than faulting
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t v = idx[i];
    if (v < 0 || v >= table_rows) v = 0;
    for (int j = 0; j < width; ++j) out[i * width + j] = table[v * width + j];
}

__global__ void index_of_coeffs_kernel(const uint8_t* __restrict__ c, int64_t n, int k, int p,
                                       const int64_t* __restrict__ ioc, int64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t code = 0;
    for (int l = k - 1; l >= 0; --l) code = code * p + c[i * k + l];
    out[i] = ioc[code];
}

}  // namespace qadic

using namespace qadic;

static inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

extern "C" {

int qadic_matmul_exact_u64(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t m, int64_t k,
                           int64_t n, void* stream) {
    QADIC_REQUIRE(m >= 0 && k >= 0 && n >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    if (m == 0 || n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (k == 0) {
        cudaMemsetAsync(c, 0, (size_t)(m * n) * sizeof(uint64_t), s);
        return check_launch("matmul_exact_u64 (memset)");
    }
    dim3 grid(blocks_for(n, MM_T), blocks_for(m, MM_T));
    QADIC_REQUIRE(grid.y <= 65535, QADIC_ERR_UNSUPPORTED, "m too large for this kernel");
    mm_wrap_kernel<uint64_t><<<grid, 256, 0, s>>>(a, b, c, m, k, n, 0, 0);
    return check_launch("matmul_exact_u64", 1);
}

int qadic_matmul_mod_i64(const int64_t* a, const int64_t* b, int64_t* c, int64_t m, int64_t k, int64_t n,
                         int64_t p, int64_t chunk, void* stream) {
    QADIC_REQUIRE(m >= 0 && k >= 0 && n >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    QADIC_REQUIRE(p >= 1 && chunk >= 1, QADIC_ERR_VALUE, "need p >= 1 and chunk >= 1");
    if (m == 0 || n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (k == 0) {
        cudaMemsetAsync(c, 0, (size_t)(m * n) * sizeof(int64_t), s);
        return check_launch("matmul_mod_i64 (memset)");
    }
    dim3 grid(blocks_for(n, MM_T), blocks_for(m, MM_T));
    QADIC_REQUIRE(grid.y <= 65535, QADIC_ERR_UNSUPPORTED, "m too large for this kernel");
    mm_wrap_kernel<int64_t><<<grid, 256, 0, s>>>(a, b, c, m, k, n, p, chunk);
    return check_launch("matmul_mod_i64", 1);
}

int qadic_conv_exact_u64(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb, uint64_t* out,
                         void* stream) {
    QADIC_REQUIRE(na >= 1 && nb >= 1, QADIC_ERR_SHAPE, "convolution needs non-empty operands");
    conv_kernel<uint64_t><<<blocks_for(na + nb - 1, 256), 256, 0, (cudaStream_t)stream>>>(a, na, b, nb, out);
    return check_launch("conv_exact_u64", 1);
}

int qadic_conv_exact_i64(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t* out,
                         void* stream) {
    QADIC_REQUIRE(na >= 1 && nb >= 1, QADIC_ERR_SHAPE, "convolution needs non-empty operands");
    conv_kernel<int64_t><<<blocks_for(na + nb - 1, 256), 256, 0, (cudaStream_t)stream>>>(a, na, b, nb, out);
    return check_launch("conv_exact_i64", 1);
}

static int redq_launch(const uint64_t* r, int64_t n, int64_t p, int32_t t, int32_t d, int mode,
                       uint64_t* digits, uint64_t* packed, void* stream, const char* what) {
    QADIC_REQUIRE(n >= 0, QADIC_ERR_SHAPE, "negative length");
    QADIC_REQUIRE((int64_t)d * t < 64, QADIC_ERR_VALUE, "digit span exceeds the 64-bit word");
    QADIC_REQUIRE(p >= 2 && d >= 0 && t >= 1, QADIC_ERR_VALUE, "need p >= 2, d >= 0, t >= 1");
    if (n == 0) return QADIC_OK;
    const uint64_t q = 1ull << t;
    const uint64_t corr = (q % (uint64_t)p == 0) ? 0 : ((uint64_t)p - q % (uint64_t)p) % (uint64_t)p;
    redq_words_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        r, n, (uint64_t)p, t, d, host_reciprocal_up(p), host_case2_bound(), corr, mode, digits, packed);
    return check_launch(what, 1);
}

int qadic_redq_compress_u64(const uint64_t* r, int64_t n, int64_t p, int32_t t, int32_t d, uint64_t* out,
                            void* stream) {
    return redq_launch(r, n, p, t, d, 0, out, nullptr, stream, "redq_compress_u64");
}

int qadic_reduce_words(const uint64_t* words, int64_t n, int64_t p, int32_t t, int32_t d, uint64_t* packed_out,
                       uint64_t* digits_out, void* stream) {
    return redq_launch(words, n, p, t, d, packed_out ? 2 : 1, digits_out, packed_out, stream, "reduce_words");
}

int qadic_pack_rows_u8(const uint8_t* m, int64_t rows, int64_t cols, int32_t k, int32_t t, int32_t reverse,
                       uint64_t* words, void* stream) {
    QADIC_REQUIRE(rows >= 0 && cols >= 0 && k >= 1 && t >= 1 && (int64_t)k * t <= 64, QADIC_ERR_VALUE,
                  "bad pack geometry");
    const int64_t total = rows * ((cols + k - 1) / k);
    if (total == 0) return QADIC_OK;
    pack_rows_kernel<<<blocks_for(total, 256), 256, 0, (cudaStream_t)stream>>>(m, rows, cols, k, t, reverse, words);
    return check_launch("pack_rows_u8", 1);
}

int qadic_unpack_rows_u8(const uint64_t* words, int64_t rows, int64_t cols, int32_t k, int32_t t,
                         int32_t reverse, uint8_t* out, void* stream) {
    QADIC_REQUIRE(rows >= 0 && cols >= 0 && k >= 1 && t >= 1 && t <= 8 * 8, QADIC_ERR_VALUE, "bad unpack geometry");
    if (rows * cols == 0) return QADIC_OK;
    unpack_rows_kernel<<<blocks_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(words, rows, cols, k, t,
                                                                                        reverse, out);
    return check_launch("unpack_rows_u8", 1);
}

int qadic_gather_u8(const int64_t* idx, int64_t n, const uint8_t* table, int64_t table_rows, int32_t width,
                    uint8_t* out, void* stream) {
    QADIC_REQUIRE(n >= 0 && width >= 1, QADIC_ERR_VALUE, "bad gather geometry");
    if (n == 0) return QADIC_OK;
    gather_u8_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(idx, n, table, table_rows, width, out);
    return check_launch("gather_u8", 1);
}

int qadic_index_of_coeffs(const uint8_t* c, int64_t n, int32_t k, int32_t p, const int64_t* index_of_code,
                          int64_t* out, void* stream) {
    QADIC_REQUIRE(n >= 0 && k >= 1 && p >= 2, QADIC_ERR_VALUE, "bad conversion geometry");
    if (n == 0) return QADIC_OK;
    index_of_coeffs_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(c, n, k, p, index_of_code, out);
    return check_launch("index_of_coeffs", 1);
}

}  // extern "C"
