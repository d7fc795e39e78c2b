// Any-field DQT word path: the reference's own composition, every stage a CUDA
// kernel, for the fields and primes outside the uint8 coefficient engines
// (p > 127, k > 4, or L/H tables wider than shared memory).
//
// Reference domain (src/params.py:29, src/gfext.py:38-39, 311-358, src/cmm.py:86-94,
// 244-305): primes p < 2^26, field orders p^k <= 2^22, any reduced CMM entries.
// The heavy step is the uint64 word product, which runs on the byte-plane INT8
// tensor-core GEMM (qadic_matmul_exact_u64, layer_k.cu / engine_tc.cu); the
// kernels here are the HBM-bound stages around it:
//
//   gather_u64        pack_table[idx]                       gfext.py:329-330
//   words_dot         sum_j pack[v1[b,j]] * pack[v2[b,j]]    gfext.py:287-290 (batched)
//   gf_finish         REDQ compress (2k-1 digits) -> L/H index -> two lookups ->
//                     field addition on codes -> handle       gfext.py:331-358
//   pack/unpack i64   d+1 entries per word, any entry < q     cmm.py:72-85, 130-145
//   extract_middle    ((acc >> d t) & (q-1)) mod p            cmm.py:178-204
//   full_cmm_reduce   one REDQ per word, digits scattered to their
//                     (d_q+1) x (d_theta+1) tile               cmm.py:313-359
//   correct_digits    mu_i = (u_i + c u_{i+1}) mod p          redq.py:308-315
//
// Exactness: every accumulator the callers pass satisfies the reference's a-priori
// bound (sums < q^(2k-1) <= 2^beta), so the uint64 words never wrap.  s = r // p
// uses the FP64 reciprocal (fdiv case 2) below 2^53 and integer division above
// (beta > 53 is allowed by the parameter API); the digits u_i = (r >> it) -
// p (s >> it) are exact in wrap-around uint64 arithmetic because their true value
// lies in [0, p) (src/redq.py:6-8).
#include <cuda_runtime.h>

#include <algorithm>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {
namespace {

constexpr int TPB = 256;

unsigned grid_of(int64_t n, int per_thread = 1) {
    const int64_t want = (n + (int64_t)TPB * per_thread - 1) / ((int64_t)TPB * per_thread);
    const int64_t cap = (int64_t)num_sms_cached() * 16;
    return (unsigned)std::max<int64_t>(1, std::min(want, cap));
}

QADIC_D uint64_t floor_div(uint64_t r, uint64_t p, double invp_up, double bound) {
    if (r < (1ull << 53)) return (uint64_t)fdiv_floor((double)r, invp_up, (double)p, bound);
    return r / p;
}

__global__ void gather_u64_kernel(const int64_t* __restrict__ idx, int64_t n, const uint64_t* __restrict__ table,
                                  uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(table + __ldg(idx + i));
}

// one warp per dot: lanes stride the row, then a shuffle reduction (wrap-around
// uint64 adds, exact under the dot bound)
__global__ void words_dot_kernel(const int64_t* __restrict__ v1, const int64_t* __restrict__ v2, int64_t rows,
                                 int64_t len, const uint64_t* __restrict__ pack, uint64_t* __restrict__ acc) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const int64_t* x = v1 + r * len;
        const int64_t* y = v2 + r * len;
        uint64_t s = 0;
        for (int64_t j = lane; j < len; j += 32) s += __ldg(pack + __ldg(x + j)) * __ldg(pack + __ldg(y + j));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) acc[r] = s;
    }
}

__global__ void gf_finish_kernel(const uint64_t* __restrict__ acc, int64_t n, qadic_gf_generic_desc f,
                                 double invp_up, double bound, int64_t* __restrict__ out) {
    const uint64_t p = (uint64_t)f.p;
    const int k = f.k, t = f.t, bb = f.u_bits;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = acc[i];
        const uint64_t s = floor_div(r, p, invp_up, bound);
        uint64_t li = 0, hi = 0;
        for (int d = 0; d < 2 * k - 1; ++d) {
            const uint64_t u = (r >> (d * t)) - p * (s >> (d * t));  // in [0, p): exact under wrap-around
            if (d < k) li |= u << (bb * d);
            if (d >= k - 1) hi |= u << (bb * (d - (k - 1)));
        }
        int64_t a = __ldg(f.l_code + li), b = __ldg(f.h_code + hi);
        int64_t code = 0, mul = 1;
        for (int d = 0; d < k; ++d) {  // coefficient-wise addition of the two codes
            int64_t c = a % (int64_t)p + b % (int64_t)p;
            if (c >= (int64_t)p) c -= (int64_t)p;
            code += mul * c;
            a /= (int64_t)p;
            b /= (int64_t)p;
            mul *= (int64_t)p;
        }
        out[i] = __ldg(f.index_of_code + code);
    }
}

// words[r, w] = sum_j m[r, w k + j] << (t * (reverse ? k-1-j : j)), zero padded
__global__ void pack_rows_i64_kernel(const int64_t* __restrict__ m, int64_t rows, int64_t cols, int k, int t,
                                     int reverse, uint64_t* __restrict__ words) {
    const int64_t nw = (cols + k - 1) / k, n = rows * nw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nw, w = i - r * nw;
        const int64_t* src = m + r * cols + w * k;
        const int lim = (int)std::min<int64_t>(k, cols - w * k);
        uint64_t word = 0;
        for (int j = 0; j < lim; ++j) word |= (uint64_t)src[j] << (t * (reverse ? k - 1 - j : j));
        words[i] = word;
    }
}

__global__ void unpack_rows_i64_kernel(const uint64_t* __restrict__ words, int64_t rows, int64_t cols, int k, int t,
                                       int reverse, int64_t* __restrict__ out) {
    const int64_t nw = (cols + k - 1) / k, n = rows * cols;
    const uint64_t mask = t >= 64 ? ~0ull : ((1ull << t) - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        const int64_t w = c / k;
        const int j = (int)(c - w * k);
        out[i] = (int64_t)((words[r * nw + w] >> (t * (reverse ? k - 1 - j : j))) & mask);
    }
}

__global__ void extract_middle_kernel(const uint64_t* __restrict__ acc, int64_t n, int64_t p, int t, int d,
                                      int64_t* __restrict__ out) {
    const uint64_t mask = (1ull << t) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)(((acc[i] >> (d * t)) & mask) % (uint64_t)p);
}

// one word per thread: its (dq+1)(dth+1) digits at radix 2^t, corrected with c =
// (-q) mod p, land at out[i (dq+1) + a, j (dth+1) + b] for digit b (dq+1) + a
__global__ void full_cmm_reduce_kernel(const uint64_t* __restrict__ acc, int64_t mw, int64_t nw, int64_t p, int t,
                                       int dq, int dth, int64_t m, int64_t n, double invp_up, double bound,
                                       int64_t* __restrict__ out) {
    const int nd = (dq + 1) * (dth + 1);
    const uint64_t q_mod_p = (1ull << t) % (uint64_t)p;
    const uint64_t c = ((uint64_t)p - q_mod_p) % (uint64_t)p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mw * nw;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = acc[i];
        const uint64_t s = floor_div(r, (uint64_t)p, invp_up, bound);
        const int64_t wi = i / nw, wj = i - wi * nw;
        uint64_t u_next = (r >> (nd - 1) * t) - (uint64_t)p * (s >> (nd - 1) * t);
        for (int dd = nd - 1; dd >= 0; --dd) {
            const uint64_t u = (r >> (dd * t)) - (uint64_t)p * (s >> (dd * t));
            // mu_dd = (u_dd + c u_{dd+1}) mod p, mu_top = u_top (redq.py:118-128)
            const uint64_t mu = dd == nd - 1 ? u : (u + (c * u_next) % (uint64_t)p) % (uint64_t)p;
            u_next = u;
            const int a = dd % (dq + 1), b = dd / (dq + 1);
            const int64_t row = wi * (dq + 1) + a, col = wj * (dth + 1) + b;
            if (row < m && col < n) out[row * n + col] = (int64_t)mu;
        }
    }
}

// the reference's vectorised correction on arbitrary uint64 digits: wrap-around
// (u_d + c u_{d+1}) mod 2^64, then mod p; the top digit is kept; identity when
// p | q (identity != 0)
__global__ void correct_digits_kernel(const uint64_t* __restrict__ u, int64_t n, int w, int64_t p, uint64_t c,
                                      int identity, uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t* x = u + i * w;
        uint64_t* y = out + i * w;
        for (int d = 0; d < w; ++d)
            y[d] = (identity || d + 1 == w) ? x[d] : (x[d] + c * x[d + 1]) % (uint64_t)p;
    }
}

// Tabulated correction (redq.py:194-300) over a batch: digits u_0..u_d of each
// word (REDQ-compressed here from the word, or given), then overlapping width-j
// block lookups (ceil(d/j) per word, the last block shifted down to end at digit
// d-1) in a table of packed corrected residues -- staged in shared memory when it
// fits, else read through L1/L2 -- and the top digit passes through (mod p).
struct TabArgs {
    const uint64_t* words;   // [n] words (compress first) or null
    const uint64_t* digits;  // [n, d+1] compressed digits when words is null
    int64_t n;
    int64_t p;
    int t, d, j, base_p, bb, smem_entries;
    const uint64_t* table;
    double invp_up, bound;
    uint64_t* out;           // [n, d+1]
};

__global__ void tabulated_kernel(TabArgs A) {
    extern __shared__ uint64_t tab_s[];
    const uint64_t* tab = A.table;
    if (A.smem_entries > 0) {
        for (int i = threadIdx.x; i < A.smem_entries; i += blockDim.x) tab_s[i] = __ldg(A.table + i);
        __syncthreads();
        tab = tab_s;
    }
    const uint64_t p = (uint64_t)A.p;
    const uint64_t mask = (1ull << A.bb) - 1;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < A.n; w += (int64_t)gridDim.x * blockDim.x) {
        uint64_t u[64];
        if (A.words) {
            const uint64_t r = A.words[w];
            const uint64_t s = floor_div(r, p, A.invp_up, A.bound);
            for (int i = 0; i <= A.d; ++i) u[i] = (r >> (i * A.t)) - p * (s >> (i * A.t));
        } else {
            for (int i = 0; i <= A.d; ++i) u[i] = A.digits[w * (A.d + 1) + i];
        }
        uint64_t* o = A.out + w * (A.d + 1);
        o[A.d] = u[A.d] % p;
        if (A.d == 0) continue;
        int nblocks = A.d - A.j + 1 > 0 ? (A.d - A.j) / A.j + 1 : 1;
        for (int b = 0; b <= nblocks; ++b) {
            int s0;
            if (b < nblocks) s0 = b * A.j;
            else if ((nblocks - 1) * A.j + A.j < A.d) s0 = A.d - A.j;  // trailing block, shifted down
            else break;
            uint64_t idx = 0, mul = 1;
            for (int i = 0; i <= A.j; ++i) {
                const uint64_t v = s0 + i <= A.d && s0 + i >= 0 ? u[s0 + i] : 0;  // zero padding past the top
                if (A.base_p) {
                    idx += v * mul;
                    mul *= p;
                } else {
                    idx |= v << (A.bb * i);
                }
            }
            const uint64_t e = tab[idx];
            for (int i = 0; i < A.j; ++i)
                if (s0 + i < A.d && s0 + i >= 0) o[s0 + i] = (e >> (A.bb * i)) & mask;
        }
    }
}

}  // namespace
}  // namespace qadic

using namespace qadic;

extern "C" {

int qadic_gather_u64(const int64_t* idx, int64_t n, const uint64_t* table, uint64_t* out, void* stream) {
    QADIC_REQUIRE(n >= 0, QADIC_ERR_VALUE, "bad gather size");
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("gather_u64", s, gather_u64_kernel<<<grid_of(n), TPB, 0, s>>>(idx, n, table, out));
    return check_launch("gather_u64");
}

int qadic_gf_words_dot(const int64_t* v1, const int64_t* v2, int64_t rows, int64_t len, const uint64_t* pack,
                       uint64_t* acc, void* stream) {
    QADIC_REQUIRE(rows >= 0 && len >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    if (rows == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (len == 0) {
        cudaMemsetAsync(acc, 0, (size_t)rows * sizeof(uint64_t), s);
        return check_launch("gf_words_dot (empty)");
    }
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, num_sms_cached() * 16));
    QADIC_TIMED("gf_words_dot", s, words_dot_kernel<<<g, TPB, 0, s>>>(v1, v2, rows, len, pack, acc));
    return check_launch("gf_words_dot");
}

int qadic_gf_words_finish(const uint64_t* acc, int64_t n, const qadic_gf_generic_desc* f, int64_t* out,
                          void* stream) {
    QADIC_REQUIRE(f != nullptr && n >= 0, QADIC_ERR_VALUE, "bad arguments");
    QADIC_REQUIRE(f->p >= 2 && f->p < (1ll << 26) && f->k >= 1 && f->t >= 1 && f->u_bits >= 1, QADIC_ERR_VALUE,
                  "bad field description");
    QADIC_REQUIRE((int64_t)(2 * f->k - 1) * f->t <= 64 && (int64_t)f->k * f->u_bits <= 40, QADIC_ERR_PARAMS,
                  "digit span exceeds the 64-bit word");
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("gf_words_finish", s,
                gf_finish_kernel<<<grid_of(n), TPB, 0, s>>>(acc, n, *f, host_reciprocal_up(f->p), host_case2_bound(),
                                                           out));
    return check_launch("gf_words_finish");
}

int qadic_pack_rows_i64(const int64_t* m, int64_t rows, int64_t cols, int32_t k, int32_t t, int32_t reverse,
                        uint64_t* words, void* stream) {
    QADIC_REQUIRE(rows >= 0 && cols >= 0 && k >= 1 && t >= 1 && (int64_t)k * t <= 64, QADIC_ERR_VALUE,
                  "bad packing geometry");
    const int64_t n = rows * ((cols + k - 1) / k);
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("pack_rows_i64", s, pack_rows_i64_kernel<<<grid_of(n), TPB, 0, s>>>(m, rows, cols, k, t, reverse, words));
    return check_launch("pack_rows_i64");
}

int qadic_unpack_rows_i64(const uint64_t* words, int64_t rows, int64_t cols, int32_t k, int32_t t, int32_t reverse,
                          int64_t* out, void* stream) {
    QADIC_REQUIRE(rows >= 0 && cols >= 0 && k >= 1 && t >= 1 && (int64_t)k * t <= 64, QADIC_ERR_VALUE,
                  "bad packing geometry");
    const int64_t n = rows * cols;
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("unpack_rows_i64", s,
                unpack_rows_i64_kernel<<<grid_of(n), TPB, 0, s>>>(words, rows, cols, k, t, reverse, out));
    return check_launch("unpack_rows_i64");
}

int qadic_extract_middle(const uint64_t* acc, int64_t n, int64_t p, int32_t t, int32_t d, int64_t* out,
                         void* stream) {
    QADIC_REQUIRE(n >= 0 && p >= 2 && t >= 1 && d >= 0 && (int64_t)(d + 1) * t <= 64, QADIC_ERR_VALUE,
                  "bad extraction geometry");
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("extract_middle", s, extract_middle_kernel<<<grid_of(n), TPB, 0, s>>>(acc, n, p, t, d, out));
    return check_launch("extract_middle");
}

int qadic_full_cmm_reduce(const uint64_t* acc, int64_t mw, int64_t nw, int64_t p, int32_t t, int32_t dq,
                          int32_t dth, int64_t m, int64_t n, int64_t* out, void* stream) {
    QADIC_REQUIRE(mw >= 0 && nw >= 0 && p >= 2 && p < (1ll << 26) && t >= 1 && dq >= 0 && dth >= 0,
                  QADIC_ERR_VALUE, "bad arguments");
    QADIC_REQUIRE((int64_t)(dq + 1) * (dth + 1) * t <= 64, QADIC_ERR_PARAMS, "digit span exceeds the 64-bit word");
    if (mw * nw == 0 || m == 0 || n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("full_cmm_reduce", s,
                full_cmm_reduce_kernel<<<grid_of(mw * nw), TPB, 0, s>>>(acc, mw, nw, p, t, dq, dth, m, n,
                                                                       host_reciprocal_up(p), host_case2_bound(), out));
    return check_launch("full_cmm_reduce");
}

int qadic_redq_tabulated(const uint64_t* words, const uint64_t* digits, int64_t n, int64_t p, int32_t t, int32_t d,
                         const uint64_t* table, int64_t table_entries, int32_t j, int32_t base_p, uint64_t* out,
                         void* stream) {
    QADIC_REQUIRE(n >= 0 && p >= 2 && p < (1ll << 26) && d >= 0 && d < 64 && j >= 1 && table != nullptr,
                  QADIC_ERR_VALUE, "bad tabulated-correction arguments");
    QADIC_REQUIRE((words == nullptr) != (digits == nullptr), QADIC_ERR_VALUE, "give words or digits");
    QADIC_REQUIRE(words == nullptr || (t >= 1 && (int64_t)(d + 1) * t <= 64), QADIC_ERR_VALUE,
                  "digit span exceeds the 64-bit word");
    if (n == 0) return QADIC_OK;
    TabArgs A;
    A.words = words;
    A.digits = digits;
    A.n = n;
    A.p = p;
    A.t = t;
    A.d = d;
    A.j = j;
    A.base_p = base_p;
    int bb = 1;
    while ((1ll << bb) < p) ++bb;  // ceil(log2 p), at least 1 (redq.py:238)
    A.bb = bb;
    A.table = table;
    A.invp_up = host_reciprocal_up(p);
    A.bound = host_case2_bound();
    A.out = out;
    A.smem_entries = table_entries <= 6144 ? (int)table_entries : 0;  // <= 48 KB: shared memory
    cudaStream_t s = (cudaStream_t)stream;
    QADIC_TIMED("redq_tabulated", s,
                tabulated_kernel<<<grid_of(n), TPB, (size_t)A.smem_entries * sizeof(uint64_t), s>>>(A));
    return check_launch("redq_tabulated");
}

int qadic_correct_digits(const uint64_t* u, int64_t n, int32_t width, int64_t p, int64_t q_mod_p, uint64_t* out,
                         void* stream) {
    QADIC_REQUIRE(n >= 0 && width >= 1 && p >= 2 && q_mod_p >= 0 && q_mod_p < p, QADIC_ERR_VALUE, "bad arguments");
    if (n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t c = (uint64_t)((p - q_mod_p) % p);
    QADIC_TIMED("correct_digits", s,
                correct_digits_kernel<<<grid_of(n), TPB, 0, s>>>(u, n, width, p, c, q_mod_p == 0, out));
    return check_launch("correct_digits");
}

}  // extern "C"
