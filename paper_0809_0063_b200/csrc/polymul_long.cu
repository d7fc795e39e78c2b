// Batched long-polynomial products over GF(p) on packed words.
//
// Reference: polymul.polymul_fqt with _wordconv_reduce / _kara_words
// (src/polymul.py:159-271).  A polynomial of length L becomes ceil(L/k) words of
// k = d+1 digits at radix q = 2^t; the product of two word sequences is a word
// convolution whose output words carry 2k-1 digits; digits are kept below q by a
// REDQ fold (compress, correct, repack) every `chunk` inner terms -- the
// reference's _chunk_budget -- and one final REDQ recovers every digit mod p;
// digit r of word j lands on X^(jk + r) (overlap-add mod p).
//
// B200 design (not the reference's host loop):
//   * one launch for a whole batch of pairs (equal lengths per batch);
//   * conv_tile_kernel: a CTA owns 1024 output words of one pair (128 threads x
//     8 consecutive words in registers); a[i] and the b window are staged in
//     shared memory 256 inner terms at a time, each thread slides its 8-word b
//     window by one register per inner step, so an inner step is one broadcast
//     load of a, one load of b and 8 FMAs.  The accumulators are FP64 (the
//     paper's formulation: every sum is an integer < q^(2k-1) <= 2^53, exact);
//     with beta > 53 (sums up to 2^64) a uint64 instantiation runs instead;
//   * the fold is in registers: s = r // p by the FP64 reciprocal (fdiv case 2),
//     u_i = lo32(r >> it) - p lo32(s >> it), mu_i = (u_i + c u_{i+1}) mod p,
//     repack -- after every `chunk` inner steps (the fold count equals the
//     reference's: the longer operand is the inner one);
//   * conv_direct_kernel: one thread per output word for short operands (the
//     batched one-word products beyond cfg1's fused kernel: p > 127 or k > 8);
//   * Karatsuba (algo 1) breadth-first: each level splits every pair into the
//     three half-length products (a0 b0, a1 b1, (a0+a1)(b0+b1), word-wise sums --
//     the sum pair's digit bound doubles, so its fold budget shrinks) as a 3x
//     larger batch; the leaves run the convolution kernel once; the levels
//     recombine on residues, c = m0 + X^(hk) (m1 - m0 - m2) + X^(2hk) m2 mod p.
//     A level splits while the worst pair of the level still may (n > threshold,
//     2^(j+1) ma <= q-1, chunk >= 1), i.e. uniformly; results are identical to the
//     reference's per-pair recursion (exact arithmetic), the split points differ.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {
namespace {

constexpr int CT = 128;          // threads per conv CTA
#ifndef QADIC_POLY_CR
#define QADIC_POLY_CR 8
#endif
constexpr int CR = QADIC_POLY_CR;  // output words per thread (8 measured faster than 16: 0.187 vs 0.211 ms, occupancy)
constexpr int CR_SHIFT = CR == 16 ? 4 : 3;
constexpr int TJ = CT * CR;      // output words per CTA
constexpr int TI = 256;          // inner terms staged per round
constexpr int BW = TJ + TI - 1;  // b window length per round
// one pad double per CR: the stride-CR thread reads of the b window spread over the banks
QADIC_D int bpad(int x) { return x + (x >> CR_SHIFT); }
constexpr int BW_PAD = BW + (BW >> CR_SHIFT) + 2;

struct ConvArgs {
    const uint64_t* a;   // [batch][na] (the longer operand: the inner loop)
    const uint64_t* b;   // [batch][nb]
    const int8_t* jsum;  // per pair: Karatsuba sum depth (digit bound 2^j), or null
    int64_t batch, na, nb, nout;
    uint32_t p;
    int t, nd;           // radix bits, top digit index 2d
    uint64_t budget;     // q - 1 - (p - 1)
    uint64_t per0;       // k * ma * mb at depth 0
    uint32_t c;          // (-q) mod p
    double invp, bound, pd;
    uint32_t* mu;        // [segs][batch][nout][nd+1] digits mod p (one slab per inner segment)
    unsigned int* flag;  // validate: set when a value exceeds the top digit
    int validate;
    int segs;            // inner-dimension segments (split-K): slab s holds the partial sums of segment s
    uint32_t magic;      // small_magic(p) when small_p
    int small_p;         // p^3 < 2^32: (u + c u') mod p by one 32-bit reciprocal multiply
};

QADIC_D uint64_t chunk_of(const ConvArgs& A, int64_t pair) {
    const int j = A.jsum ? A.jsum[pair] : 0;
    const uint64_t per = A.per0 << (2 * j);
    const uint64_t ch = A.budget / per;
    return ch < 1 ? 1 : ch;
}

QADIC_D uint64_t mod_p53(uint64_t x, const ConvArgs& A) {  // x < 2^53
    const uint64_t q = (uint64_t)fdiv_floor((double)x, A.invp, A.pd, A.bound);
    return x - q * A.p;
}

// floor(r / p) for the accumulator's integer value
QADIC_D uint64_t div_p(uint64_t r, const ConvArgs& A) {
    return r < (1ull << 53) ? (uint64_t)fdiv_floor((double)r, A.invp, A.pd, A.bound) : r / A.p;
}

// REDQ of one accumulator value: digit i (mod p, corrected) passed to emit(i, mu)
// from the top digit down
template <typename F>
QADIC_D void redq_digits(uint64_t r, const ConvArgs& A, F emit) {
    const uint64_t s = div_p(r, A);
    uint32_t u_next = 0;
    for (int i = A.nd; i >= 0; --i) {
        const uint32_t u = (uint32_t)(r >> (i * A.t)) - A.p * (uint32_t)(s >> (i * A.t));
        uint32_t mu = u;
        if (i != A.nd) {
            if (A.small_p) {  // x < p^2 + p and p^3 < 2^32: the 32-bit reciprocal quotient is exact
                const uint32_t x = u + A.c * u_next;
                mu = x - A.p * __umulhi(x, A.magic);
            } else {
                mu = (uint32_t)mod_p53((uint64_t)u + (uint64_t)A.c * u_next, A);
            }
        }
        u_next = u;
        emit(i, mu);
    }
}

template <typename Acc>
QADIC_D uint64_t as_u64(Acc v) { return (uint64_t)v; }

template <typename Acc>
QADIC_D void fold(Acc& v, const ConvArgs& A) {
    const uint64_t r = as_u64(v);
    if (A.validate && (A.nd + 1) * A.t < 64 && (r >> ((A.nd + 1) * A.t))) atomicOr(A.flag, 1u);
    uint64_t w = 0;
    redq_digits(r, A, [&](int i, uint32_t mu) { w |= (uint64_t)mu << (i * A.t); });
    v = (Acc)w;
}

template <typename Acc>
QADIC_D void mac(Acc& acc, Acc x, Acc y);
template <>
QADIC_D void mac<double>(double& acc, double x, double y) { acc = fma(x, y, acc); }
template <>
QADIC_D void mac<uint64_t>(uint64_t& acc, uint64_t x, uint64_t y) { acc += x * y; }

template <typename Acc>
QADIC_D void store_digits(Acc v, int64_t pair, int64_t j, const ConvArgs& A, int seg = 0) {
    const uint64_t r = as_u64(v);
    if (A.validate && (A.nd + 1) * A.t < 64 && (r >> ((A.nd + 1) * A.t))) atomicOr(A.flag, 1u);
    uint32_t* dst = A.mu + (((int64_t)seg * A.batch + pair) * A.nout + j) * (A.nd + 1);
    redq_digits(r, A, [&](int i, uint32_t mu) { dst[i] = mu; });
}

template <typename Acc>
__global__ void __launch_bounds__(CT, 8) conv_tile_kernel(ConvArgs A) {
    __shared__ Acc a_s[TI];
    __shared__ Acc b_s[BW_PAD];
    const int64_t tiles = (A.nout + TJ - 1) / TJ;
    const int seg = (int)(blockIdx.x % A.segs);
    const int64_t tile_id = blockIdx.x / A.segs;
    const int64_t pair = tile_id / tiles;
    const int64_t j0 = (tile_id - pair * tiles) * TJ;
    const uint64_t* ap = A.a + pair * A.na;
    const uint64_t* bp = A.b + pair * A.nb;
    const uint64_t chunk = chunk_of(A, pair);
    // inner range touching this tile: i in [max(0, j0 - nb + 1), min(na, j0 + TJ)), split
    // into A.segs contiguous segments (whole staging rounds); this CTA sums segment `seg`
    const int64_t tlo = j0 - A.nb + 1 > 0 ? j0 - A.nb + 1 : 0;
    const int64_t thi = j0 + TJ < A.na ? j0 + TJ : A.na;
    const int64_t rounds = (thi - tlo + TI - 1) / TI;
    const int64_t per = (rounds + A.segs - 1) / A.segs;
    const int64_t ilo = tlo + (int64_t)seg * per * TI;
    const int64_t ihi = ilo + per * TI < thi ? ilo + per * TI : thi;
    Acc acc[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) acc[r] = (Acc)0;
    uint64_t since = 0;  // inner steps since the last fold (>= terms added to any accumulator)
    const int tj = threadIdx.x * CR;
    // b_s[bpad(x + 1)] = b[bbase + x]; b_s[0] = 0 stands for the one index (-1) the
    // last slide of thread 0 reads.  a_s is zero padded to TI: every round runs TI
    // unconditional steps (zero terms only count towards the fold budget).
    if (threadIdx.x == 0) b_s[0] = (Acc)0;
    const bool block_fold = chunk >= CR;  // fold decisions once per CR steps
    for (int64_t i0 = ilo; i0 < ihi; i0 += TI) {
        const int cnt = (int)(ihi - i0 < TI ? ihi - i0 : TI);
        __syncthreads();
        for (int x = threadIdx.x; x < TI; x += CT) a_s[x] = x < cnt ? (Acc)ap[i0 + x] : (Acc)0;
        const int64_t bbase = j0 - i0 - (TI - 1);
        for (int x = threadIdx.x; x < BW; x += CT) {
            const int64_t bi = bbase + x;
            b_s[bpad(x + 1)] = (bi >= 0 && bi < A.nb) ? (Acc)bp[bi] : (Acc)0;
        }
        __syncthreads();
        // thread's outputs j = j0 + tj + r; term (ii, r) uses b[bbase + tj + r + TI - 1 - ii]:
        // logical r lives in register slot (r - ii) mod CR, so a step loads one new value
        Acc w[CR];
#pragma unroll
        for (int r = 0; r < CR; ++r) w[r] = b_s[bpad(tj + r + TI)];
        if (block_fold) {
#pragma unroll 1
            for (int ii0 = 0; ii0 < TI; ii0 += CR) {
                if (since + CR > chunk) {
#pragma unroll
                    for (int r = 0; r < CR; ++r) fold(acc[r], A);
                    since = 0;
                }
#pragma unroll
                for (int u = 0; u < CR; ++u) {
                    const Acc av = a_s[ii0 + u];
#pragma unroll
                    for (int r = 0; r < CR; ++r) mac<Acc>(acc[r], av, w[(r - u + CR) % CR]);
                    w[(CR - 1 - u + CR) % CR] = b_s[bpad(tj + TI - 1 - ii0 - u)];
                }
                since += CR;
            }
        } else {  // fold budget below CR (fold-bound radix): plain loads, a fold every `chunk` steps
#pragma unroll 1
            for (int ii = 0; ii < TI; ++ii) {
                const Acc av = a_s[ii];
#pragma unroll
                for (int r = 0; r < CR; ++r) mac<Acc>(acc[r], av, b_s[bpad(tj + r + TI - ii)]);
                if (++since == chunk) {
#pragma unroll
                    for (int r = 0; r < CR; ++r) fold(acc[r], A);
                    since = 0;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < CR; ++r) {
        const int64_t j = j0 + tj + r;
        if (j < A.nout) store_digits(acc[r], pair, j, A, seg);
    }
}

// one thread per output word (short operands, large batches)
template <typename Acc>
__global__ void conv_direct_kernel(ConvArgs A) {
    const int64_t total = A.batch * A.nout;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pair = g / A.nout, j = g - pair * A.nout;
        const uint64_t* ap = A.a + pair * A.na;
        const uint64_t* bp = A.b + pair * A.nb;
        const uint64_t chunk = chunk_of(A, pair);
        const int64_t ilo = j - A.nb + 1 > 0 ? j - A.nb + 1 : 0;
        const int64_t ihi = j + 1 < A.na ? j + 1 : A.na;
        // fold schedule on the inner index as in the tiled kernel: after every `chunk`
        // steps of i counted from 0 (the reference folds after each chunk of a)
        Acc acc = (Acc)0;
        for (int64_t i = ilo; i < ihi; ++i) {
            mac<Acc>(acc, (Acc)__ldg(ap + i), (Acc)__ldg(bp + j - i));
            if ((uint64_t)(i - ilo + 1) % chunk == 0 && i + 1 < ihi) fold(acc, A);
        }
        store_digits(acc, pair, j, A);
    }
}

// out[pair][P] = (mu_r(j) + mu_{r+k}(j-1)) mod p, P = j k + r, for P < ncoef; flag when a
// position at or beyond ncoef (up to (nout+1)k-1) is nonzero
template <typename T>
__global__ void overlap_kernel(const uint32_t* __restrict__ mu, int64_t batch, int64_t nout, int k, uint32_t p,
                               int64_t ncoef, int64_t full, T* __restrict__ out, unsigned int* flag, int segs) {
    const int nd = 2 * k - 2;
    const int64_t span = full > ncoef ? full : ncoef;
    const int64_t slab = batch * nout * (nd + 1);
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < batch * span;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pair = g / span, P = g - pair * span;
        uint32_t v = 0;
        if (P < full) {
            const int64_t j = P / k;
            const int r = (int)(P - j * k);
            for (int sg = 0; sg < segs; ++sg) {  // partial sums of the inner segments, each < p
                const uint32_t* m = mu + sg * slab + pair * nout * (nd + 1);
                if (j < nout) v += m[j * (nd + 1) + r];
                if (j >= 1 && r + k <= nd) v += m[(j - 1) * (nd + 1) + r + k];
                v %= p;
            }
        }
        if (P < ncoef) out[pair * ncoef + P] = (T)v;
        else if (v) atomicOr(flag, 2u);
    }
}

// Karatsuba split: pair b of length n -> children 3b (lo), 3b+1 (lo + hi), 3b+2 (hi),
// each of length n - h (h = n / 2), zero padded; depth of the sum child + 1
__global__ void kara_split_kernel(const uint64_t* __restrict__ x, int64_t batch, int64_t n, int64_t h,
                                  uint64_t* __restrict__ y) {
    const int64_t hn = n - h;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < batch * hn;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / hn, i = g - b * hn;
        const uint64_t lo = i < h ? x[b * n + i] : 0ull;
        const uint64_t hi = x[b * n + h + i];
        uint64_t* dst = y + 3 * b * hn;
        dst[i] = lo;
        dst[hn + i] = lo + hi;
        dst[2 * hn + i] = hi;
    }
}

__global__ void kara_depth_kernel(const int8_t* __restrict__ jp, int64_t batch, int8_t* __restrict__ jc) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
        const int8_t j = jp ? jp[b] : 0;
        jc[3 * b] = j;
        jc[3 * b + 1] = j + 1;
        jc[3 * b + 2] = j;
    }
}

// parent[b][P] = m0 + X^(hk) (m1 - m0 - m2) + X^(2hk) m2 mod p over children coefficient
// rows of length lc (residues); parent rows of length lp
__global__ void kara_combine_kernel(const uint32_t* __restrict__ ch, int64_t batch, int64_t lc, int64_t hk,
                                    uint32_t p, int64_t lp, uint32_t* __restrict__ par) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < batch * lp;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / lp, P = g - b * lp;
        const uint32_t* m0 = ch + 3 * b * lc;
        const uint32_t* m1 = m0 + lc;
        const uint32_t* m2 = m1 + lc;
        int64_t v = 0;
        if (P < lc) v += m0[P];
        const int64_t P1 = P - hk;
        if (P1 >= 0 && P1 < lc) v += (int64_t)m1[P1] + 2 * (int64_t)p - m0[P1] - m2[P1];
        const int64_t P2 = P - 2 * hk;
        if (P2 >= 0 && P2 < lc) v += m2[P2];
        par[g] = (uint32_t)(v % p);
    }
}

template <typename T>
__global__ void emit_kernel(const uint32_t* __restrict__ c, int64_t batch, int64_t lc, int64_t ncoef,
                            T* __restrict__ out, unsigned int* flag) {
    const int64_t span = lc > ncoef ? lc : ncoef;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < batch * span;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / span, P = g - b * span;
        const uint32_t v = P < lc ? c[b * lc + P] : 0u;
        if (P < ncoef) out[b * ncoef + P] = (T)v;
        else if (v) atomicOr(flag, 2u);
    }
}

unsigned grid_for(int64_t n) {
    const int64_t want = (n + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms_cached() * 16));
}

int64_t coeff_len(int64_t nw, int k) { return nw ? (nw + 1) * k - 1 : 0; }

}  // namespace
}  // namespace qadic

namespace qadic {
size_t tc_toeplitz_workspace(int64_t batch, int64_t na, int64_t nb);
int tc_polymul_toeplitz(const uint8_t* a, int64_t na, const uint8_t* b, int64_t nb, int64_t batch, uint32_t p,
                        uint8_t* out, int64_t ncoef, void* ws, size_t ws_bytes, cudaStream_t s);
}  // namespace qadic

using namespace qadic;

extern "C" {

size_t qadic_polymul_tc_workspace(int64_t batch, int64_t na, int64_t nb) {
    if (batch < 0 || na < 1 || nb < 1) return 0;
    return tc_toeplitz_workspace(batch, na, nb);
}

int qadic_polymul_tc_u8(const uint8_t* a, int64_t na, const uint8_t* b, int64_t nb, int64_t batch, int64_t p,
                        uint8_t* out, int64_t ncoef, void* ws, size_t ws_bytes, void* stream) {
    QADIC_REQUIRE(na >= 1 && nb >= 1 && batch >= 0 && ncoef >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    if (batch == 0) return QADIC_OK;
    return tc_polymul_toeplitz(a, na, b, nb, batch, (uint32_t)p, out, ncoef, ws, ws_bytes, (cudaStream_t)stream);
}

int qadic_polymul_words_batch(const uint64_t* aw, int64_t na, const uint64_t* bw, int64_t nb, int64_t batch,
                              int64_t p, int32_t t, int32_t d, int64_t ma, int64_t mb, int32_t algo,
                              int64_t threshold, int32_t validate, int32_t out_u8, void* out, int64_t ncoef,
                              qadic_polymul_stats* stats, void* stream) {
    QADIC_REQUIRE(na >= 1 && nb >= 1 && batch >= 0 && ncoef >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    QADIC_REQUIRE(p >= 2 && p < (1ll << 26) && t >= 1 && d >= 0 && ma >= 1 && mb >= 1, QADIC_ERR_VALUE,
                  "bad polynomial product parameters");
    QADIC_REQUIRE((int64_t)(2 * d + 1) * t <= 64, QADIC_ERR_PARAMS, "word budget exceeded for 2d+1 digits");
    QADIC_REQUIRE(!out_u8 || p <= 256, QADIC_ERR_VALUE, "uint8 output needs p <= 256");
    QADIC_REQUIRE(algo == 0 || algo == 1, QADIC_ERR_VALUE, "algo must be 0 (classical) or 1 (karatsuba)");
    const int k = d + 1;
    const unsigned __int128 q = (unsigned __int128)1 << t;
    QADIC_REQUIRE(q - 1 >= (unsigned __int128)(p - 1), QADIC_ERR_PARAMS, "radix smaller than p");
    const uint64_t budget = (uint64_t)(q - 1 - (p - 1));
    const uint64_t per0 = (uint64_t)k * (uint64_t)ma * (uint64_t)mb;
    QADIC_REQUIRE(budget / per0 >= 1, QADIC_ERR_PARAMS, "accumulation budget too small for this packing");
    const bool f64 = (int64_t)(2 * d + 1) * t <= 53;  // every sum < q^(2k-1) <= 2^53: exact in FP64
    cudaStream_t s = (cudaStream_t)stream;
    if (stats) *stats = qadic_polymul_stats{0, 0, 0, 0, 0};
    if (batch == 0) return QADIC_OK;

    keep_mempool();
    std::vector<void*> allocs;
    auto alloc = [&](size_t bytes) -> void* {
        void* ptr = nullptr;
        if (cudaMallocAsync(&ptr, bytes ? bytes : 1, s) != cudaSuccess) return nullptr;
        allocs.push_back(ptr);
        return ptr;
    };
    auto release = [&]() {
        for (void* ptr : allocs) cudaFreeAsync(ptr, s);
    };
    unsigned int* flag = static_cast<unsigned int*>(alloc(sizeof(unsigned int)));
    if (!flag) {
        release();
        QADIC_REQUIRE(false, QADIC_ERR_CUDA, "polymul scratch allocation failed");
    }
    cudaMemsetAsync(flag, 0, sizeof(unsigned int), s);

    // ---- plan: Karatsuba levels (uniform split), leaves = one batched convolution ----
    const uint64_t* ca = aw;
    const uint64_t* cb = bw;
    int64_t n_a = na, n_b = nb, B = batch;
    const int8_t* jsum = nullptr;
    struct Level {
        int64_t B, n, h;
    };
    std::vector<Level> levels;
    if (algo == 1) {
        int64_t n = std::max(na, nb);
        if (na != nb) {  // pad both to n words
            uint64_t* pa = static_cast<uint64_t*>(alloc((size_t)B * n * 8));
            uint64_t* pb = static_cast<uint64_t*>(alloc((size_t)B * n * 8));
            if (!pa || !pb) {
                release();
                QADIC_REQUIRE(false, QADIC_ERR_CUDA, "polymul scratch allocation failed");
            }
            cudaMemset2DAsync(pa, n * 8, 0, n * 8, B, s);
            cudaMemset2DAsync(pb, n * 8, 0, n * 8, B, s);
            cudaMemcpy2DAsync(pa, n * 8, aw, na * 8, na * 8, B, cudaMemcpyDeviceToDevice, s);
            cudaMemcpy2DAsync(pb, n * 8, bw, nb * 8, nb * 8, B, cudaMemcpyDeviceToDevice, s);
            ca = pa;
            cb = pb;
        }
        n_a = n_b = n;
        int depth = 0;
        for (;;) {
            // the worst pair of the next level has sum depth depth+1: 2^(depth+1) ma <= q-1 and a
            // non-empty fold budget (polymul.py:243-249)
            const unsigned __int128 m2a = (unsigned __int128)ma << (depth + 1), m2b = (unsigned __int128)mb << (depth + 1);
            const bool can = n > threshold && n >= 2 && m2a <= q - 1 && m2b <= q - 1 &&
                             (unsigned __int128)budget / ((unsigned __int128)k * m2a * m2b) >= 1 && depth < 60;
            if (!can) break;
            const int64_t h = n / 2, hn = n - h;
            uint64_t* na_w = static_cast<uint64_t*>(alloc((size_t)3 * B * hn * 8));
            uint64_t* nb_w = static_cast<uint64_t*>(alloc((size_t)3 * B * hn * 8));
            int8_t* nj = static_cast<int8_t*>(alloc((size_t)3 * B));
            if (!na_w || !nb_w || !nj) {
                release();
                QADIC_REQUIRE(false, QADIC_ERR_CUDA, "polymul scratch allocation failed");
            }
            QADIC_TIMED("polymul kara split", s, kara_split_kernel<<<grid_for(B * hn), 256, 0, s>>>(ca, B, n, h, na_w));
            QADIC_TIMED("polymul kara split", s, kara_split_kernel<<<grid_for(B * hn), 256, 0, s>>>(cb, B, n, h, nb_w));
            QADIC_TIMED("polymul kara split", s, kara_depth_kernel<<<grid_for(B), 256, 0, s>>>(jsum, B, nj));
            levels.push_back({B, n, h});
            ca = na_w;
            cb = nb_w;
            jsum = nj;
            B *= 3;
            n = hn;
            n_a = n_b = n;
            ++depth;
        }
    } else if (na < nb) {  // the longer operand is the inner (folded) one, as in the reference
        std::swap(ca, cb);
        std::swap(n_a, n_b);
    }

    // ---- leaves: one batched convolution + REDQ ----
    const int64_t nout = n_a + n_b - 1;
    const int nd = 2 * d;
    const bool tiled = n_a >= 64;
    // split-K: enough CTAs for ~8 per SM, each segment at least one staging round
    int segs = 1;
    if (tiled) {
        const int64_t tiles = B * ((nout + TJ - 1) / TJ);
        // one full wave of resident CTAs
        static int occ = 0;
        if (!occ) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f64 ? (const void*)conv_tile_kernel<double>
                                                                    : (const void*)conv_tile_kernel<uint64_t>,
                                                          CT, 0);
            if (occ < 1) occ = 1;
        }
        // several waves of shorter segments: the tiles at both ends of a product have
        // triangular (shorter) inner ranges, so one wave of equal-count CTAs leaves SMs idle
        // (measured: one wave when the fold budget is >= CR -- FMA-bound, 0.192 vs 0.202 ms for
        // two; three when it is below -- fold-bound, 0.645 vs 0.868 ms)
        static const int waves_env = getenv("QADIC_POLY_WAVES") ? atoi(getenv("QADIC_POLY_WAVES")) : 0;
        const int waves = waves_env > 0 ? waves_env : (budget / per0 >= (uint64_t)CR ? 1 : 3);
        const int64_t want = (int64_t)num_sms_cached() * occ * waves;
        const int64_t max_rounds = std::min<int64_t>(n_a, TJ + n_b - 1) / TI + 1;
        if (tiles < want) segs = (int)std::min<int64_t>({want / tiles, max_rounds, 64});
        if (segs < 1) segs = 1;
    }
    uint32_t* mu = static_cast<uint32_t*>(alloc((size_t)segs * B * nout * (nd + 1) * 4));
    if (!mu) {
        release();
        QADIC_REQUIRE(false, QADIC_ERR_CUDA, "polymul scratch allocation failed");
    }
    ConvArgs A;
    A.a = ca;
    A.b = cb;
    A.jsum = jsum;
    A.batch = B;
    A.na = n_a;
    A.nb = n_b;
    A.nout = nout;
    A.p = (uint32_t)p;
    A.t = t;
    A.nd = nd;
    A.budget = budget;
    A.per0 = per0;
    const uint64_t qmodp = (uint64_t)(q % (unsigned __int128)p);
    A.c = (uint32_t)(((uint64_t)p - qmodp) % (uint64_t)p);
    A.invp = host_reciprocal_up(p);
    A.bound = host_case2_bound();
    A.pd = (double)p;
    A.mu = mu;
    A.flag = flag;
    A.validate = validate;
    A.segs = segs;
    A.small_p = (uint64_t)p * p * p < (1ull << 32);
    A.magic = small_magic((uint32_t)p);
    if (tiled) {
        const int64_t grid = B * ((nout + TJ - 1) / TJ) * segs;
        QADIC_REQUIRE(grid < (1ll << 31), QADIC_ERR_UNSUPPORTED, "batch too large for one launch");
        if (f64) QADIC_TIMED("polymul conv", s, conv_tile_kernel<double><<<(unsigned)grid, CT, 0, s>>>(A));
        else QADIC_TIMED("polymul conv", s, conv_tile_kernel<uint64_t><<<(unsigned)grid, CT, 0, s>>>(A));
    } else {
        if (f64) QADIC_TIMED("polymul conv", s, conv_direct_kernel<double><<<grid_for(B * nout), 256, 0, s>>>(A));
        else QADIC_TIMED("polymul conv", s, conv_direct_kernel<uint64_t><<<grid_for(B * nout), 256, 0, s>>>(A));
    }

    // ---- stats: the operation counts of this schedule (host arithmetic) ----
    if (stats) {
        const int L = (int)levels.size();
        const int64_t base = batch;
        int64_t binom = 1;
        for (int j = 0; j <= L; ++j) {  // leaves with j sum steps: C(L, j) 2^(L-j) per pair
            if (j > 0) binom = binom * (L - j + 1) / j;
            const int64_t cnt = base * binom * (1ll << (L - j));
            const unsigned __int128 per = (unsigned __int128)per0 << (2 * j);
            int64_t chunk = (int64_t)((unsigned __int128)budget / per);
            if (chunk < 1) chunk = 1;
            stats->word_muls += cnt * n_a * n_b;
            stats->reductions += cnt * nout * ((n_a + chunk - 1) / chunk);
        }
        stats->levels = L;
        stats->leaves = B;
    }

    // ---- residues per coefficient: overlap-add at the leaves, recombine upwards ----
    int rc = QADIC_OK;
    if (levels.empty()) {
        const int64_t full = coeff_len(nout, k);
        if (out_u8)
            QADIC_TIMED("polymul overlap", s, overlap_kernel<uint8_t><<<grid_for(B * std::max(full, ncoef)), 256, 0, s>>>(
                mu, B, nout, k, (uint32_t)p, ncoef, full, static_cast<uint8_t*>(out), flag, segs));
        else
            QADIC_TIMED("polymul overlap", s, overlap_kernel<int64_t><<<grid_for(B * std::max(full, ncoef)), 256, 0, s>>>(
                mu, B, nout, k, (uint32_t)p, ncoef, full, static_cast<int64_t*>(out), flag, segs));
    } else {
        int64_t lc = coeff_len(nout, k);
        uint32_t* cur = static_cast<uint32_t*>(alloc((size_t)B * lc * 4));
        if (!cur) rc = QADIC_ERR_CUDA;
        if (rc == QADIC_OK)
            QADIC_TIMED("polymul overlap", s, overlap_kernel<uint32_t><<<grid_for(B * lc), 256, 0, s>>>(
                mu, B, nout, k, (uint32_t)p, lc, lc, cur, flag, segs));
        for (int li = (int)levels.size() - 1; li >= 0 && rc == QADIC_OK; --li) {
            const Level& Lv = levels[li];
            const int64_t lp = coeff_len(2 * Lv.n - 1, k);
            uint32_t* par = static_cast<uint32_t*>(alloc((size_t)Lv.B * lp * 4));
            if (!par) {
                rc = QADIC_ERR_CUDA;
                break;
            }
            QADIC_TIMED("polymul kara combine", s, kara_combine_kernel<<<grid_for(Lv.B * lp), 256, 0, s>>>(
                cur, Lv.B, lc, Lv.h * k, (uint32_t)p, lp, par));
            cur = par;
            lc = lp;
        }
        if (rc == QADIC_OK) {
            if (out_u8)
                QADIC_TIMED("polymul emit", s, emit_kernel<uint8_t><<<grid_for(batch * std::max(lc, ncoef)), 256, 0, s>>>(
                    cur, batch, lc, ncoef, static_cast<uint8_t*>(out), flag));
            else
                QADIC_TIMED("polymul emit", s, emit_kernel<int64_t><<<grid_for(batch * std::max(lc, ncoef)), 256, 0, s>>>(
                    cur, batch, lc, ncoef, static_cast<int64_t*>(out), flag));
        }
    }
    // the flags come back only when asked for (stats): without them the call stays
    // asynchronous on the stream
    unsigned int* hflag = nullptr;
    if (rc == QADIC_OK) {
        rc = check_launch("polymul_words_batch");
        if (stats) {
            static thread_local unsigned int* slot = nullptr;
            if (!slot && cudaHostAlloc(reinterpret_cast<void**>(&slot), sizeof(unsigned int), cudaHostAllocDefault) !=
                             cudaSuccess)
                slot = nullptr;
            hflag = slot;
            if (hflag) cudaMemcpyAsync(hflag, flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, s);
        }
    }
    release();
    if (rc != QADIC_OK) {
        set_error(rc, "polymul_words_batch: %s", rc == QADIC_ERR_CUDA ? "allocation or launch failure" : "failed");
        return rc;
    }
    if (stats) {
        QADIC_REQUIRE(hflag && cudaStreamSynchronize(s) == cudaSuccess, QADIC_ERR_CUDA, "polymul_words_batch: %s",
                      cudaGetErrorString(cudaGetLastError()));
        stats->flags = *hflag;
    }
    return QADIC_OK;
}

}  // extern "C"
