// Engine F64: the paper's own formulation on B200 FP64 tensor cores.
//
// DQT-packed words (GFqField._build_pack_table,
// src/gfext.py:158-174; cmm._pack_axis, src/cmm.py:72-85) are exact
// integers below 2^53, so FP64 matrix products of them are exact
// (PAPER.md:216-223).  tcgen05 has no f64 kind, so the product runs on
// warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) with a 3-stage
// cp.async pipeline, and the whole inverse DQT is fused into the epilogue:
//
//   REDQ compression with the FP64 reciprocal (qadic_common.cuh), then
//   * GF(p^k):  L/H correction+fold tables staged in shared memory
//               (src/gfext.py:176-213, 336-344) -> k coefficient bytes
//   * right_cmm: corrected digits (src/redq.py:308-315) -> d+1 entries
//
// When the inner dimension exceeds the a-priori bound (cfg5: fold budget 9,
// src/polymul.py:159-167), every `fold` inner terms the accumulators are
// digit-reduced in registers (compress + correct + repack,
// src/redq.py:318-332) -- the delayed-reduction fold of
// src/polymul.py:198-208 without leaving the register file.
#include <type_traits>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

int make_field_const(const qadic_field_desc* d, FieldConst* f);

namespace f64 {

#ifndef QADIC_F64_BK
#define QADIC_F64_BK 32
#endif
constexpr int BM = 128, BN = 128, BK = QADIC_F64_BK;  // BK 32: half the block barriers of 16
constexpr int SA = BK + 4;   // A smem row pitch (doubles): conflict-free fragment loads
constexpr int SB = BN + 4;   // B smem row pitch (doubles)
constexpr int STAGES = 3;
// warps along M (x 4 along N): WM = 2 -- 8 warps of 64 x 32 (32 DMMAs per 12 fragment
// loads, 238 registers) for plain and pseudo-Mersenne-fold kernels; WM = 4 -- 16 warps of
// 32 x 32 (128 registers) where the REDQ fold's temporaries would spill the 64-accumulator tile
template <int WM>
struct WarpTile {
    static constexpr int THREADS = 32 * WM * 4;
    static constexpr int MI = BM / (WM * 8);  // m8 fragments per warp
};
template <int FOLD>
constexpr int wm_for_fold() { return FOLD >= 1 ? 4 : 2; }
constexpr int TABLE_MAX = 4096;
constexpr size_t PIPE_BYTES = (size_t)STAGES * (BM * SA + BK * SB) * sizeof(double);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// EPI_GF: two-sided DQT words (both operands packed), REDQ + L/H fold per output.
// EPI_CMM: right_cmm, corrected digits of B-packed words.
// EPI_GF1: one-sided DQT (only A packed, B's coefficient planes side by side
//          in N): corrected digits of each word to a [M][N][k][k] byte buffer
//          that gf1_combine_kernel turns into coefficients.
enum Epi { EPI_GF = 0, EPI_CMM = 1, EPI_GF1 = 2 };

struct Params {
    const double* a;  // [Mp, Kp] packed words
    const double* b;  // [Kp, Np]
    int64_t M, Nw, Kp, Np;   // logical rows, logical word columns, padded dims
    int64_t n_out;           // output entries per row (GF: N; CMM: N)
    int fold;                // 0 = none; else multiple of 4
    int fold_mode;           // 0: fold_word; 1: fold_word_fast; 2: fast with lazy corrected digits
    int group_m;             // row blocks per raster group
    uint64_t pm_hi;          // fold mode 3: lane mask 2^(t-e) - 1 at every digit
    int pm_e;
    uint32_t pm_m;           // 2^e - (2^e mod p)
    int d;                   // CMM: digits per word - 1
    uint8_t* c;
};

// digit-reduce one accumulator in registers and repack (reduce_words_array)
template <int ND>
__device__ __forceinline__ double fold_word(double r, const FieldConst& f) {
    uint32_t u[ND + 1];
    redq_compress_f64<ND>(r, f.invp_up, (double)f.p, f.bound, f.p, (int)f.t, u);
    uint64_t w = u[ND];
#pragma unroll
    for (int i = ND - 1; i >= 0; --i) w = (w << f.t) | mod_small(u[i] + f.corr * u[i + 1], f.p, f.magic);
    return (double)w;
}

// The same fold on the FP64 pipe where the generic one uses conversions (F2I /
// I2F, quarter-rate, three per word -- they, not the DMMAs, bounded the fold
// schedule): for an exact integer r < 2^51 (< the case-2 bound B, so no
// correction step),
//   bits(r + 2^52)                       = 0x433.. | r
//   bits(RD(RN(r * RU(1/p)) + 2^52))     = 0x433.. | floor(RN(r * RU(1/p))) = s
// then the REDQ digits u_i = lo32(r >> it) - p lo32(s >> it) (src/redq.py:58-85) and,
// when the host cleared the budget for it (LAZY), the corrected digits are left
// unreduced: mu_i = u_i + c u_{i+1} < p^2 is congruent to the reduced digit and the
// next fold / the epilogue's REDQ sees it like any other digit sum.
// `acc` is a BIASED accumulator (2^52 + r, see dmma_gemm_kernel): its bit pattern is
// 0x433.. | r, so r needs no conversion and the folded word goes back as bits.
template <int ND, bool LAZY, int T>  // T > 0: the radix exponent f.t as a compile-time constant
__device__ __forceinline__ double fold_word_fast(double acc, const FieldConst& f) {
    const int t = T > 0 ? T : (int)f.t;
    constexpr double TWO52 = 4503599627370496.0;
    constexpr uint64_t MANT = (1ull << 52) - 1;
    const uint64_t rv = (uint64_t)__double_as_longlong(acc) & MANT;
    const double r = acc - TWO52;
    const uint64_t sv = (uint64_t)__double_as_longlong(__dadd_rd(__dmul_rn(r, f.invp_up), TWO52)) & MANT;
    uint32_t u[ND + 1];
#pragma unroll
    for (int i = 0; i <= ND; ++i) u[i] = (uint32_t)(rv >> (i * t)) - f.p * (uint32_t)(sv >> (i * t));
    uint64_t w = u[ND];
#pragma unroll
    for (int i = ND - 1; i >= 0; --i) {
        const uint32_t mu = u[i] + f.corr * u[i + 1];
        w = (w << t) | (LAZY ? mu : mod_small(mu, f.p, f.magic));
    }
    return __longlong_as_double((long long)(w | 0x4330000000000000ull));
}

// Digit-wise pseudo-Mersenne fold (fold mode 3): when 2^e = c (mod p) with c small
// (cfg5: p = 7, 2^6 = 1), every digit d of the word (lanes of t bits, d < 2^t) maps
// to (d mod 2^e) + c (d >> e) -- congruent mod p and at most (2^e - 1) + c ((2^t - 1) >> e)
// (cfg5: 78) -- on the whole word at once: a shift, a mask, a multiply-subtract (no lane
// carries: every new lane value is below 2^t), no quotient.  The intermediate folds
// only have to keep the digits congruent and below the budget; the epilogue's REDQ
// produces the reduced result.  For words below 2^52 (the 2^52 offset carries them).
// On the biased accumulator (bits 0x433.. | r): integer instructions only.  With
// hi = the digits' high parts d >> e, the folded word is w - (2^e - c) hi (each lane
// d - 2^e (d >> e) + c (d >> e)): one mask and one multiply-subtract on the FMA pipe
// instead of two masks and an add on the ALU pipe, and the exponent bits of w pass
// through untouched (hi stays below bit 50, no lane goes negative).
__device__ __forceinline__ double fold_word_pm(double acc, uint64_t mhi, int e, uint32_t m) {
    const uint64_t w = (uint64_t)__double_as_longlong(acc);  // the exponent bits lie outside the mask
    const uint64_t hi = (w >> e) & mhi;
    return __longlong_as_double((long long)(w - (uint64_t)m * hi));
}

// FOLD: the launch folds the packed accumulators every prm.fold terms (the fold
// code is compiled only into the kernels that need it): 0 none, else the
// fold_mode_for() flavour + 1 (1 fold_word, 2 fold_word_fast, 3 fast and lazy,
// 4 the pseudo-Mersenne digit fold)
template <int K, Epi EPI, bool SMEM_TABLES, int FOLD>
__global__ void __launch_bounds__(WarpTile<wm_for_fold<FOLD>()>::THREADS, 1) dmma_gemm_kernel(Params prm, FieldConst f) {
    constexpr int THREADS = WarpTile<wm_for_fold<FOLD>()>::THREADS;
    constexpr int MI = WarpTile<wm_for_fold<FOLD>()>::MI;
    constexpr int ND = EPI == EPI_GF ? 2 * K - 2 : (EPI == EPI_GF1 ? K - 1 : 0);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    double* sA = reinterpret_cast<double*>(smem_raw);
    double* sB = sA + STAGES * BM * SA;
    uint32_t* s_l = reinterpret_cast<uint32_t*>(sB + STAGES * BK * SB);
    const int tsize = EPI == EPI_GF && SMEM_TABLES ? 1 << (f.bb * K) : 0;
    uint32_t* s_h = s_l + tsize;

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int wm = warp / 4, wn = warp % 4;
    // grouped raster: consecutive blocks sweep prm.group_m row blocks of A per column
    // block of B, so a B column panel (K x 128 words) is reused from L2 by group_m row
    // blocks instead of streamed from DRAM once per row block
    int64_t m0, n0;
    {
        const int nt = (int)gridDim.x, mt = (int)gridDim.y, gm = prm.group_m > 0 ? prm.group_m : 1;
        const int id = (int)(blockIdx.y * gridDim.x + blockIdx.x);
        const int per = gm * nt, grp = id / per, first = grp * gm, g = min(mt - first, gm), r = id % per;
        m0 = (int64_t)(first + r % g) * BM;
        n0 = (int64_t)(r / g) * BN;
    }

    if (EPI == EPI_GF && SMEM_TABLES) {
        const int size = 1 << (f.bb * K);
        for (int i = tid; i < size; i += THREADS) {
            s_l[i] = f.l_table[i];
            s_h[i] = f.h_table[i];
        }
    }

    auto load_stage = [&](int slot, int64_t k0) {
        double* a_s = sA + slot * BM * SA;
        double* b_s = sB + slot * BK * SB;
        // A: 128 rows x 16 doubles = 1024 16-byte chunks; B: 16 rows x 128 doubles
#pragma unroll
        for (int it = 0; it < BM * BK / 2 / THREADS; ++it) {  // BM x BK (= BK x BN) doubles, 2 per chunk
            const int c = tid + it * THREADS;
            const int r = c / (BK / 2), q = c % (BK / 2);
            cp_async16(a_s + r * SA + 2 * q, prm.a + (m0 + r) * prm.Kp + k0 + 2 * q);
            const int rb = c / (BN / 2), qb = c % (BN / 2);
            cp_async16(b_s + rb * SB + 2 * qb, prm.b + (k0 + rb) * prm.Np + n0 + 2 * qb);
        }
    };

    // Fast-fold kernels accumulate on a 2^52 bias: the DMMA sums stay exact integers in
    // [2^52, 2^53) (every word < 2^51), the bit pattern of 2^52 + r is 0x433.. | r, so the
    // folds read and write words as bits (no conversion, no FP64 instruction in the
    // pseudo-Mersenne fold); the epilogue removes the bias.
    constexpr bool BIAS = FOLD >= 2;
    constexpr double ACC0 = BIAS ? 4503599627370496.0 : 0.0;
    double acc[MI][4][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = ACC0;

    // the radix of this kernel's fold schedule as a compile-time constant (the
    // generic runtime-t shifts of 64-bit words cost ~2x the integer instructions):
    // two-sided DQT 2^(53/(2K-1)) (cfg5: 10), one-sided 2^min(53/K, 30)
    constexpr int FOLD_T = EPI == EPI_GF ? 53 / (2 * K - 1) : (53 / K > 30 ? 30 : 53 / K);
    auto fold_all = [&](auto tconst) {
        constexpr int TT = decltype(tconst)::value;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double& x = acc[i][j][h];
                    if constexpr (FOLD == 4) x = fold_word_pm(x, prm.pm_hi, prm.pm_e, prm.pm_m);
                    else if constexpr (FOLD == 3) x = fold_word_fast<ND, true, TT>(x, f);
                    else if constexpr (FOLD == 2) x = fold_word_fast<ND, false, TT>(x, f);
                    else x = fold_word<ND>(x, f);
                }
    };
    (void)fold_all;
    auto fold_now = [&]() {
        if constexpr (FOLD == 2 || FOLD == 3) {
            if (f.t == (uint32_t)FOLD_T) fold_all(std::integral_constant<int, FOLD_T>{});
            else fold_all(std::integral_constant<int, 0>{});
        } else {
            fold_all(std::integral_constant<int, 0>{});
        }
    };
    (void)fold_now;
    // fold phase of this warp (see the fold-8 stage loop): every accumulator still folds
    // at most every prm.fold terms, the odd warps' first fold comes after 4
    const int fold_off = (FOLD && prm.fold == 8 && (warp & 1)) ? 4 : 0;
    const int nk = (int)(prm.Kp / BK);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, (int64_t)s * BK);
        cp_async_commit();
    }
    const int ar = lane >> 2, ac = lane & 3;
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < nk) load_stage((kt + STAGES - 1) % STAGES, (int64_t)(kt + STAGES - 1) * BK);
        cp_async_commit();
        const double* a_s = sA + (kt % STAGES) * BM * SA + (wm * (MI * 8) + ar) * SA + ac;
        const double* b_s = sB + (kt % STAGES) * BK * SB + ac * SB + wn * 32 + ar;
        auto k4_step = [&](int k4) {
            double af[MI], bf[4];
#pragma unroll
            for (int i = 0; i < MI; ++i) af[i] = a_s[i * 8 * SA + k4 * 4];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = b_s[k4 * 4 * SB + j * 8];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        };
        // delayed-reduction folds land on k4 boundaries; a stage holds one only
        // every fold / BK stages, so the common stage runs the plain DMMA stream
        // and only a fold stage checks per k4 step (the per-step modulo cost
        // ~10% of the issue slots at cfg5)
        const int64_t kbase = (int64_t)kt * BK;
        const bool fold_here = FOLD && (EPI == EPI_GF || EPI == EPI_GF1) && prm.fold &&
                               (kbase + BK) / prm.fold != kbase / prm.fold && kbase + BK <= prm.Kp;
        if (!fold_here) {
#pragma unroll
            for (int k4 = 0; k4 < BK / 4; ++k4) k4_step(k4);
        } else if (prm.fold == 8 && (kbase % 8) == 0 && kbase + BK < prm.Kp) {
            // cfg5's schedule (fold every 8 terms, a stage boundary on a fold boundary, no
            // fold at the very end): pairs of unrolled DMMA k-steps, one fold code copy.
            // Odd warps fold half a period later (fold_off = 4), so at any time half the
            // warps feed the DMMA pipe while the other half run the integer fold (with
            // every warp folding at the same k-steps the block alternated between a
            // DMMA-only and an ALU-only phase)
            if (fold_off == 0) {
#pragma unroll 1
                for (int k8 = 0; k8 < BK / 8; ++k8) {
                    k4_step(2 * k8);
                    k4_step(2 * k8 + 1);
                    fold_now();
                }
            } else {
                k4_step(0);
                fold_now();
#pragma unroll 1
                for (int k8 = 0; k8 < BK / 8 - 1; ++k8) {
                    k4_step(2 * k8 + 1);
                    k4_step(2 * k8 + 2);
                    fold_now();
                }
                k4_step(BK / 4 - 1);
            }
        } else {
            // one copy of the DMMA step and of the fold code per radix case (the
            // fully unrolled form held 4 x 32 inlined folds -- instruction cache)
#pragma unroll 1
            for (int k4 = 0; k4 < BK / 4; ++k4) {
                k4_step(k4);
                const int64_t kdone = kbase + (k4 + 1) * 4;
                if ((kdone - fold_off) % prm.fold == 0 && kdone < prm.Kp) fold_now();
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // tables visible (loaded before the main loop)

    // ---- fused inverse DQT epilogue ----
    const uint32_t* ltab = SMEM_TABLES ? s_l : f.l_table;
    const uint32_t* htab = SMEM_TABLES ? s_h : f.h_table;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int64_t row = m0 + wm * (MI * 8) + i * 8 + ar;
        if (row >= prm.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t col = n0 + wn * 32 + j * 8 + ac * 2 + h;  // word column
                if (col >= prm.Nw) continue;
                const double r = BIAS ? acc[i][j][h] - ACC0 : acc[i][j][h];
                if (EPI == EPI_GF) {
                    uint32_t u[ND + 1];
                    redq_compress_f64<ND>(r, f.invp_up, (double)f.p, f.bound, f.p, (int)f.t, u);
                    uint32_t li = 0, hi = 0;
#pragma unroll
                    for (int q = 0; q < K; ++q) {
                        li |= u[q] << (f.bb * q);
                        hi |= u[K - 1 + q] << (f.bb * q);
                    }
                    const uint32_t res = add_coeff_bytes(ltab[li], htab[hi], f.p, K);
                    uint8_t* dst = prm.c + (row * prm.n_out + col) * K;
#pragma unroll
                    for (int l = 0; l < K; ++l) dst[l] = (uint8_t)(res >> (8 * l));
                } else if (EPI == EPI_GF1) {
                    // one-sided word: K corrected digits = P_{i,j} mod p, i = 0..K-1
                    uint32_t u[ND + 1];
                    redq_compress_f64<ND>(r, f.invp_up, (double)f.p, f.bound, f.p, (int)f.t, u);
                    uint8_t* dst = prm.c + row * prm.n_out + col * K;
#pragma unroll
                    for (int q = 0; q <= ND; ++q)
                        dst[q] = (uint8_t)(q < ND ? mod_small(u[q] + f.corr * u[q + 1], f.p, f.magic) : u[q]);
                } else {
                    // right_cmm: d+1 corrected digits of one word = d+1 output entries
                    const int dd = prm.d;
                    const uint64_t ri = (uint64_t)r;
                    const uint64_t si = (uint64_t)fdiv_floor(r, f.invp_up, (double)f.p, f.bound);
                    uint32_t prev = (uint32_t)ri - f.p * (uint32_t)si;
                    uint8_t* dst = prm.c + row * prm.n_out;
                    for (int q = 0; q <= dd; ++q) {
                        uint32_t next = 0;
                        if (q < dd) next = (uint32_t)(ri >> ((q + 1) * f.t)) - f.p * (uint32_t)(si >> ((q + 1) * f.t));
                        const uint32_t mu = q < dd ? mod_small(prev + f.corr * next, f.p, f.magic) : prev;
                        const int64_t oc = col * (dd + 1) + q;
                        if (oc < prm.n_out) dst[oc] = (uint8_t)mu;
                        prev = next;
                    }
                }
            }
        }
    }
}

// ---- DQT pack kernels (uint8 coefficients -> FP64 words, zero-padded) ----------
// GF: src[R, C, k] -> dst[Rp, Cp], word = sum_l c_l << l t   (gfext.py:158-174)
__global__ void pack_gf_kernel(const uint8_t* __restrict__ src, int64_t R, int64_t C, int k, int t,
                               double* __restrict__ dst, int64_t Rp, int64_t Cp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Rp * Cp) return;
    const int64_t r = i / Cp, c = i % Cp;
    uint64_t w = 0;
    if (r < R && c < C) {
        const uint8_t* e = src + (r * C + c) * k;
        for (int l = 0; l < k; ++l) w |= (uint64_t)e[l] << (l * t);
    }
    dst[i] = (double)w;
}
// CMM rows: src[R, C] uint8, groups of g entries -> word = sum_j e_j << j t (cmm.py:72-85)
__global__ void pack_rows_f64_kernel(const uint8_t* __restrict__ src, int64_t R, int64_t C, int g, int t,
                                     double* __restrict__ dst, int64_t Rp, int64_t Wp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Rp * Wp) return;
    const int64_t r = i / Wp, w = i % Wp;
    uint64_t v = 0;
    if (r < R) {
        for (int j = 0; j < g; ++j) {
            const int64_t c = w * g + j;
            if (c < C) v |= (uint64_t)src[r * C + c] << (j * t);
        }
    }
    dst[i] = (double)v;
}

// one-sided combine: T[m][n][j][i] = (sum_kk a_i b_j) mod p  ->
// c_s = sum_{i+j=s} T[..][j][i], folded by X^s mod f (gfext.py:200-205) -> k bytes
template <int K>
__global__ void gf1_combine_kernel(const uint8_t* __restrict__ T, int64_t total, FieldConst f,
                                   uint8_t* __restrict__ c) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const uint8_t* t = T + e * K * K;
    uint32_t cs[2 * K - 1];
#pragma unroll
    for (int q = 0; q < 2 * K - 1; ++q) cs[q] = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
        for (int i = 0; i < K; ++i) cs[i + j] += t[j * K + i];
    uint32_t out[K];
#pragma unroll
    for (int l = 0; l < K; ++l) out[l] = 0;
#pragma unroll
    for (int q = 0; q < 2 * K - 1; ++q) {
        const uint32_t v = mod_small(cs[q], f.p, f.magic);
#pragma unroll
        for (int l = 0; l < K; ++l) out[l] += v * f.xpow[q][l];
    }
#pragma unroll
    for (int l = 0; l < K; ++l) c[e * K + l] = (uint8_t)mod_small(out[l], f.p, f.magic);
}

static inline int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// one-sided parameters: radix 2^t1 with k digits in 53 bits, and the largest
// fold period (multiple of the DMMA k-step 4) keeping every digit below 2^t1
struct OneSided {
    int t1, fold;
};
static OneSided one_sided(uint32_t p, int k) {
    OneSided o;
    o.t1 = 53 / k;
    if (o.t1 > 30) o.t1 = 30;
    const int64_t q = 1ll << o.t1, per = (int64_t)(p - 1) * (p - 1);
    o.fold = per ? (int)(((q - 1 - (p - 1)) / per) / 4 * 4) : 1 << 30;
    return o;
}
// two-sided fold periods below this make the in-register folds the bottleneck
constexpr int ONE_SIDED_BELOW = 64;

// fold flavour: fast when every folded word is below 2^51 (< the fdiv case-2 bound),
// lazy when the unreduced corrected digits (< (p-1)(1+c)+1) still leave room for a
// whole fold period of terms below q (per = per-term digit increment)
static int fold_mode_for(const FieldConst& f, int nd, int fold, int64_t per, Params* prm = nullptr) {
    const int64_t q = 1ll << f.t;
    // pseudo-Mersenne digit fold: the split point e with the smallest post-fold digit bound
    int best_e = 0;
    int64_t best_b = q;
    if ((int64_t)(nd + 1) * f.t <= 52 && fold > 0) {
        for (int e = 1; e < (int)f.t; ++e) {
            const int64_t c = (1ll << e) % f.p;
            const int64_t b = ((1ll << e) - 1) + c * ((q - 1) >> e);
            if (b < best_b && (int64_t)fold * per <= q - 1 - b) {
                best_b = b;
                best_e = e;
            }
        }
    }
    if (prm && best_e) {
        prm->pm_e = best_e;
        prm->pm_m = (uint32_t)((1ll << best_e) - (1ll << best_e) % f.p);
        prm->pm_hi = 0;
        for (int i = 0; i <= nd; ++i) prm->pm_hi |= ((1ull << (f.t - best_e)) - 1) << (i * f.t);
    }
    if (getenv("QADIC_F64_FOLD_MODE")) {
        const int m = atoi(getenv("QADIC_F64_FOLD_MODE"));
        return m == 3 && !best_e ? 2 : m;
    }
    if (best_e) return 3;
    if ((int64_t)(nd + 1) * f.t > 51) return 0;
    return (int64_t)fold * per <= q - 1 - (int64_t)(f.p - 1) * (1 + f.corr) ? 2 : 1;
}

template <int K, Epi EPI>
static int launch(const Params& prm_in, const FieldConst& f, cudaStream_t s) {
    Params prm = prm_in;
    prm.group_m = getenv("QADIC_F64_GROUP_M") ? atoi(getenv("QADIC_F64_GROUP_M")) : 8;
    // L/H tables in shared memory when they fit next to the pipeline (cfg5: 2 x 512 entries)
    const size_t tbytes = 2 * ((size_t)1 << (f.bb * K)) * sizeof(uint32_t);
    const bool smem_tables = EPI == EPI_GF && (1 << (f.bb * K)) <= TABLE_MAX && PIPE_BYTES + tbytes <= 227 * 1024;
    const size_t smem = PIPE_BYTES + (smem_tables ? tbytes : 0);
    dim3 grid((unsigned)(prm.Np / BN), (unsigned)((prm.M + BM - 1) / BM));
    QADIC_REQUIRE(grid.y <= 65535, QADIC_ERR_UNSUPPORTED, "m too large");
    const int fold = (EPI == EPI_GF || EPI == EPI_GF1) && prm.fold ? 1 + prm.fold_mode : 0;
    auto pick = [&](auto tables) {
        constexpr bool T = decltype(tables)::value;
        if constexpr (EPI == EPI_CMM) return dmma_gemm_kernel<K, EPI, T, 0>;
        else return fold == 4 ? dmma_gemm_kernel<K, EPI, T, 4>
               : fold == 3 ? dmma_gemm_kernel<K, EPI, T, 3>
               : fold == 2 ? dmma_gemm_kernel<K, EPI, T, 2>
               : fold == 1 ? dmma_gemm_kernel<K, EPI, T, 1>
                           : dmma_gemm_kernel<K, EPI, T, 0>;
    };
    auto kern = smem_tables ? pick(std::true_type{}) : pick(std::false_type{});
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = fold >= 1 ? WarpTile<4>::THREADS : WarpTile<2>::THREADS;  // wm_for_fold
    QADIC_TIMED("f64 dmma gemm", s, kern<<<grid, threads, smem, s>>>(prm, f));
    return check_launch("f64 dmma gemm");
}

}  // namespace f64

size_t f64_gf_workspace(int64_t m, int64_t kdim, int64_t n, int k) {
    using namespace f64;
    const int64_t Mp = rup(m, BM), Kp = rup(kdim, BK), Np = rup(n, BN);
    const size_t two = (size_t)(Mp * Kp + Kp * Np) * sizeof(double);
    const int64_t Np1 = rup(n * k, BN);  // one-sided: B planes side by side, plus the digit buffer
    const size_t one = (size_t)(Mp * Kp + Kp * Np1) * sizeof(double) + (size_t)(m * n * k * k);
    return two > one ? two : one;
}

size_t f64_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int d) {
    using namespace f64;
    const int64_t W = (n + d) / (d + 1);
    const int64_t Mp = rup(m, BM), Kp = rup(kdim, BK), Np = rup(W, BN);
    return (size_t)(Mp * Kp + Kp * Np) * sizeof(double);
}

// One-sided DQT (only A's polynomials packed; B's k coefficient planes side by
// side along N): S[m][(n,j)] = sum_kk W_a[m,kk] b_j[kk,n] has k digits
// P_{i,j} = sum a_i b_j, so the radix can be 2^(53/k) and a fold is needed only
// every ~2^(53/k)/(p-1)^2 terms instead of every 2^(53/(2k-1))/(k(p-1)^2) -- k
// times the DMMA work, but no fold-bound ALU phase (cfg5: fold 3636 vs 9).
static int f64_gf_matmul_one_sided(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m,
                                   int64_t kdim, int64_t n, void* ws, uint8_t* c, cudaStream_t s) {
    using namespace f64;
    const int k = (int)f.k;
    const OneSided o = one_sided(f.p, k);
    FieldConst f1 = f;
    f1.t = (uint32_t)o.t1;
    const uint64_t q = 1ull << o.t1;
    f1.corr = (q % f.p == 0) ? 0u : (uint32_t)((f.p - q % f.p) % f.p);
    const int64_t Mp = rup(m, BM), Kp = rup(kdim, BK), Np1 = rup(n * k, BN);
    double* aw = static_cast<double*>(ws);
    double* bw = aw + Mp * Kp;
    uint8_t* T = reinterpret_cast<uint8_t*>(bw + Kp * Np1);
    QADIC_TIMED("f64 pack A", s, pack_gf_kernel<<<(unsigned)((Mp * Kp + 255) / 256), 256, 0, s>>>(a, m, kdim, k, o.t1, aw, Mp, Kp));
    int rc = check_launch("f64 pack A");
    if (rc) return rc;
    // B [K, N, k] read as [K, N*k] single entries: the planes side by side
    QADIC_TIMED("f64 pack B", s, pack_gf_kernel<<<(unsigned)((Kp * Np1 + 255) / 256), 256, 0, s>>>(b, kdim, n * k, 1, o.t1, bw, Kp, Np1));
    rc = check_launch("f64 pack B");
    if (rc) return rc;
    Params prm;
    prm.a = aw;
    prm.b = bw;
    prm.M = m;
    prm.Nw = n * k;
    prm.Kp = Kp;
    prm.Np = Np1;
    prm.n_out = n * k * k;
    prm.fold = kdim > o.fold ? o.fold : 0;
    prm.fold_mode = fold_mode_for(f1, k - 1, prm.fold, (int64_t)(f.p - 1) * (f.p - 1), &prm);
    prm.d = k - 1;
    prm.c = T;
    switch (k) {
        case 1: rc = launch<1, EPI_GF1>(prm, f1, s); break;
        case 2: rc = launch<2, EPI_GF1>(prm, f1, s); break;
        case 3: rc = launch<3, EPI_GF1>(prm, f1, s); break;
        default: rc = launch<4, EPI_GF1>(prm, f1, s); break;
    }
    if (rc) return rc;
    const int64_t total = m * n;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    switch (k) {
        case 1: QADIC_TIMED("f64 combine", s, gf1_combine_kernel<1><<<blocks, 256, 0, s>>>(T, total, f, c)); break;
        case 2: QADIC_TIMED("f64 combine", s, gf1_combine_kernel<2><<<blocks, 256, 0, s>>>(T, total, f, c)); break;
        case 3: QADIC_TIMED("f64 combine", s, gf1_combine_kernel<3><<<blocks, 256, 0, s>>>(T, total, f, c)); break;
        default: QADIC_TIMED("f64 combine", s, gf1_combine_kernel<4><<<blocks, 256, 0, s>>>(T, total, f, c)); break;
    }
    return check_launch("f64 combine");
}

int f64_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                  int fold, void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, bool two_sided) {
    using namespace f64;
    const int64_t Mp = rup(m, BM), Kp = rup(kdim, BK), Np = rup(n, BN);
    QADIC_REQUIRE(ws && ws_bytes >= f64_gf_workspace(m, kdim, n, (int)f.k), QADIC_ERR_VALUE, "workspace too small");
    // the two-sided DQT form with in-register folds every `fold` terms is the paper's own
    // schedule (cfg5: q = 2^10, fold every 8 <= 9 terms).  Below ONE_SIDED_BELOW its REDQ
    // folds make it ALU-bound, so AUTO takes the one-sided form -- unless the cheap
    // digit-wise pseudo-Mersenne fold applies (cfg5: 70 vs 111 ms) or asked (engine flag / env)
    const char* env = getenv("QADIC_F64_ONE_SIDED");
    const bool pm = fold > 0 && fold_mode_for(f, 2 * (int)f.k - 2, fold, (int64_t)f.k * (f.p - 1) * (f.p - 1)) == 3;
    const bool one = two_sided ? false
                               : (env ? atoi(env) != 0 : (fold > 0 && fold < ONE_SIDED_BELOW && f.k > 1 && !pm));
    if (one) return f64_gf_matmul_one_sided(f, a, b, m, kdim, n, ws, c, s);
    double* aw = static_cast<double*>(ws);
    double* bw = aw + Mp * Kp;
    QADIC_TIMED("f64 pack A", s, pack_gf_kernel<<<(unsigned)((Mp * Kp + 255) / 256), 256, 0, s>>>(a, m, kdim, (int)f.k, (int)f.t, aw, Mp, Kp));
    int rc = check_launch("f64 pack A");
    if (rc) return rc;
    QADIC_TIMED("f64 pack B", s, pack_gf_kernel<<<(unsigned)((Kp * Np + 255) / 256), 256, 0, s>>>(b, kdim, n, (int)f.k, (int)f.t, bw, Kp, Np));
    rc = check_launch("f64 pack B");
    if (rc) return rc;
    Params prm;
    prm.a = aw;
    prm.b = bw;
    prm.M = m;
    prm.Nw = n;
    prm.Kp = Kp;
    prm.Np = Np;
    prm.n_out = n;
    prm.fold = fold;
    prm.fold_mode = fold_mode_for(f, 2 * (int)f.k - 2, fold, (int64_t)f.k * (f.p - 1) * (f.p - 1), &prm);
    // diagnostics only (wrong results): the pseudo-Mersenne fold's multiply-subtract by 0
    if (getenv("QADIC_DIAG_F64_NOFOLDMATH")) prm.pm_m = 0, prm.pm_hi = 0;
    prm.d = 0;
    prm.c = c;
    switch (f.k) {
        case 1: return launch<1, EPI_GF>(prm, f, s);
        case 2: return launch<2, EPI_GF>(prm, f, s);
        case 3: return launch<3, EPI_GF>(prm, f, s);
        default: return launch<4, EPI_GF>(prm, f, s);
    }
}

int f64_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, int t, int d,
                  void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    using namespace f64;
    const int g = d + 1;
    const int64_t W = (n + d) / g;
    const int64_t Mp = rup(m, BM), Kp = rup(kdim, BK), Np = rup(W, BN);
    QADIC_REQUIRE(ws && ws_bytes >= f64_cmm_workspace(m, kdim, n, d), QADIC_ERR_VALUE, "workspace too small");
    double* aw = static_cast<double*>(ws);
    double* bw = aw + Mp * Kp;
    QADIC_TIMED("f64 pack A", s, pack_rows_f64_kernel<<<(unsigned)((Mp * Kp + 255) / 256), 256, 0, s>>>(a, m, kdim, 1, t, aw, Mp, Kp));
    int rc = check_launch("f64 pack A");
    if (rc) return rc;
    QADIC_TIMED("f64 pack B", s, pack_rows_f64_kernel<<<(unsigned)((Kp * Np + 255) / 256), 256, 0, s>>>(b, kdim, n, g, t, bw, Kp, Np));
    rc = check_launch("f64 pack B");
    if (rc) return rc;
    FieldConst f = {};
    f.p = p;
    f.k = 1;
    f.t = (uint32_t)t;
    const uint64_t q = 1ull << t;
    f.corr = (q % p == 0) ? 0u : (uint32_t)((p - q % p) % p);
    f.magic = small_magic(p);
    f.invp_up = host_reciprocal_up(p);
    f.bound = host_case2_bound();
    Params prm;
    prm.a = aw;
    prm.b = bw;
    prm.M = m;
    prm.Nw = W;
    prm.Kp = Kp;
    prm.Np = Np;
    prm.n_out = n;
    prm.fold = 0;
    prm.fold_mode = 0;
    prm.d = d;
    prm.c = c;
    return launch<1, EPI_CMM>(prm, f, s);
}

}  // namespace qadic
