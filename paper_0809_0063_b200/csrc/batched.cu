// HBM-bound batched kernels of the hot path:
//
//  * cfg1  polymul_batch : one packed product per pair of short polynomials,
//    then the simultaneous reduction of its 2k-1 digits.  Two forms, bit-identical:
//    the default for k = 4, p <= 5 runs the transform at q = 2^8, where the operand's
//    coefficient bytes ARE its DQT word (one 32 x 32 -> 64-bit multiply, byte-lane
//    reciprocal reduction, no correction step); the paper's form
//    (qadic_polymul_batch_redq_u8) packs at q = 2^t, and REDQ divides by p through the
//    FP64 reciprocal and runs the correction pass.
//    Reference: polymul.polymul_fqt for one-word operands
//    (src/polymul.py:274-313 -> _wordconv_reduce :175-216 with na = nb = 1).
//  * cfg2  gf_dot_batch  : GF(p^k) dot products with all products accumulated
//    unreduced (no modular work inside the sum), then REDQ and the L/H
//    correction+fold tables.  Two accumulation forms, bit-identical:
//    the default sums the packed product's DIGITS directly on the coefficient
//    bytes (IDP4A; the packed words are never formed), the paper's form
//    (qadic_gf_dot_batch_f64_u8) packs every element into a DQT word held in
//    a double and accumulates the packed products with DFMA.
//    Reference: GFqField.fgdp (src/gfext.py:268-309).
//
// Both read uint8 coefficients with 128-bit loads and never touch the
// packed words in HBM: DQT packing happens in registers.
#include <cstdlib>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

struct PolyConst {
    uint32_t p, t, corr, magic;
    uint32_t negp;  // -p mod 2^32: u = r + negp * s is one IMAD
    uint32_t lm, lsh, lmask, lfix;  // byte-lane quotient: floor(d / p) ~ (d * lm) >> lsh on every lane at once
    double invp_up, bound;
};

// ---- cfg1 fast path: k = 4 (degree-3 operands), 4 or 8 pairs per thread -------
// One thread of the REDQ form: 8 pairs = 2 x 16 B of a and of b in, 56 B out -- every
// HBM access a full vector (outputs staged per warp).  Per pair: DQT-pack both operands
// in registers, one FP64 product, s = floor(r * RU(1/p)) by a round-down add of
// 2^52 (the low mantissa bits are then the integer), 7 digits by the 32-bit
// wrap trick, correction on 4 byte lanes at once.
constexpr int PM_THREADS = 256;
// pairs per thread: 8 for the REDQ form (56 output bytes = 7 x 8-byte stores; 4 measured slower
// under the 32-register cap that 8 resident blocks impose), 4 for the byte-lane form (30
// registers, 8 resident blocks: 2.92 vs 3.51 us at cfg1 -- twice as many warps whose
// stores overlap the other warps' loads)
#ifndef QADIC_PM_PER
#define QADIC_PM_PER 8
#endif
#ifndef QADIC_PM_PER_LANES
#define QADIC_PM_PER_LANES 4
#endif
constexpr int pm_minb(int per) { return per >= 8 ? 4 : 8; }  // resident blocks per SM the register cap allows

QADIC_D uint32_t pack4_bytes(uint32_t x, int t, uint32_t m) {
    return (x & m) | (((x >> 8) & m) << t) | (((x >> 16) & m) << (2 * t)) | (((x >> 24) & m) << (3 * t));
}

// byte selector for 4 consecutive stream bytes: starting at byte `first` of
// the first operand, switching to byte 0 of the second after `take` bytes
// (take = 0: all four from the 8-byte concatenation starting at `first`)
__host__ __device__ constexpr uint32_t stream_sel(int first, int take) {
    uint32_t sel = 0;
    for (int i = 0; i < 4; ++i) {
        const int b = take == 0 ? first + i : (i < take ? first + i : 4 + (i - take));
        sel |= (uint32_t)b << (4 * i);
    }
    return sel;
}

// byte-lane v mod p for lanes < 2p
QADIC_D uint32_t lanes_mod_2p(uint32_t v, uint32_t p) {
    const uint32_t t = v + (0x80u - p) * 0x01010101u;
    return v - ((t >> 7) & 0x01010101u) * p;
}

// Byte-lane form (MODE 2 / 3), the B200-native shape of the same transform: at q = 2^8 the
// DQT word of a degree-3 operand IS its four coefficient bytes, so the packed product is one
// 32 x 32 -> 64-bit multiply of the words as loaded (every digit <= 4 (p-1)^2 <= 255 stays in
// its lane), and the simultaneous reduction of all digits is one lane-wise reciprocal
// multiply per 32-bit half: s = ((v * lm) >> lsh) & lmask holds floor(d / p) (MODE 2) or a
// quotient short by at most one (MODE 3, finished by lanes_mod_2p) of every lane, and
// v - p * s the residues.  Byte-aligned digits never borrow from their neighbours, so REDQ's
// correction step has nothing to correct.  (lm, lsh) come from the host's exhaustive search
// over d <= 4 (p-1)^2 (lane_quotient_consts); the result does not depend on the caller's q.
QADIC_D uint32_t lanes_mod_p(uint32_t v, const PolyConst& c, bool fix) {
    const uint32_t s = ((v * c.lm) >> c.lsh) & c.lmask;
    const uint32_t u = v + c.negp * s;
    return fix ? lanes_mod_2p(u, c.p) : u;
}

// MODE 0: REDQ with a general correction factor; 1: REDQ, correction factor 1 (byte-lane
// correction); 2 / 3: the byte-lane form above (exact quotient / quotient short by <= 1)
template <int T, int MODE, int PM_PER>
__global__ void __launch_bounds__(PM_THREADS, pm_minb(PM_PER)) polymul_k4_kernel(const uint8_t* __restrict__ a,
                                                                const uint8_t* __restrict__ b, int64_t n,
                                                                PolyConst c, uint8_t* __restrict__ out, int pf) {
    if (pf && threadIdx.x == 0) {  // the block's operand bytes towards L2 while the predecessor drains
        const int64_t off = (int64_t)blockIdx.x * blockDim.x * PM_PER * 4, len = (int64_t)blockDim.x * PM_PER * 4;
        l2_prefetch_span(a, off, len, n * 4);
        l2_prefetch_span(b, off, len, n * 4);
    }
    pdl_wait();  // predecessor complete before any global load or store
    pdl_trigger();
    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * PM_PER;
    if (__all_sync(0xffffffffu, p0 >= n)) return;  // whole warp past the end (warps stay converged)
    uint32_t av[PM_PER], bv[PM_PER];
    const bool full = p0 + PM_PER <= n;
    // Coalesced warp path (every pair of the warp in range, 16-byte aligned operands): the
    // warp's 32 * PM_PER pairs are read as lane-consecutive 16-byte vectors (vector v of
    // lane l = pairs wp0 + 128 v + 4 l .. +3), so every load instruction covers 512
    // contiguous bytes -- the per-thread-contiguous mapping put lanes 32 bytes apart and
    // fetched every sector twice.
    const int lane = threadIdx.x & 31;
    const int64_t wp0 = p0 - (int64_t)lane * PM_PER;  // the warp's first pair
    const bool wfast = PM_PER % 4 == 0 && wp0 + 32 * PM_PER <= n &&
                       ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                         reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (wfast) {
#pragma unroll
        for (int v = 0; v < PM_PER / 4; ++v) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + wp0 * 4) + 32 * v + lane);
            const uint4 y = __ldg(reinterpret_cast<const uint4*>(b + wp0 * 4) + 32 * v + lane);
            av[4 * v] = x.x; av[4 * v + 1] = x.y; av[4 * v + 2] = x.z; av[4 * v + 3] = x.w;
            bv[4 * v] = y.x; bv[4 * v + 1] = y.y; bv[4 * v + 2] = y.z; bv[4 * v + 3] = y.w;
        }
    } else if (full) {
#pragma unroll
        for (int v = 0; v < PM_PER / 4; ++v) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + p0 * 4) + v);
            const uint4 y = __ldg(reinterpret_cast<const uint4*>(b + p0 * 4) + v);
            av[4 * v] = x.x; av[4 * v + 1] = x.y; av[4 * v + 2] = x.z; av[4 * v + 3] = x.w;
            bv[4 * v] = y.x; bv[4 * v + 1] = y.y; bv[4 * v + 2] = y.z; bv[4 * v + 3] = y.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < PM_PER; ++j) {
            av[j] = p0 + j < n ? *reinterpret_cast<const uint32_t*>(a + (p0 + j) * 4) : 0u;
            bv[j] = p0 + j < n ? *reinterpret_cast<const uint32_t*>(b + (p0 + j) * 4) : 0u;
        }
    }
    constexpr uint32_t PK_LO = 1u | ((1u << T) << 8), PK_HI = (1u << 16) | ((1u << T) << 24);
    const double two52 = 4503599627370496.0;
    uint32_t vlo[PM_PER], vhi[PM_PER];  // pair j's 7 result bytes: vlo = bytes 0..3, vhi = bytes 4..6
#pragma unroll
    for (int j = 0; j < PM_PER; ++j) {
        const uint32_t x = av[j], y = bv[j];
        if constexpr (MODE >= 2) {
            const uint64_t r = (uint64_t)x * y;  // digits c_0..c_6 on byte lanes 0..6
            vlo[j] = lanes_mod_p((uint32_t)r, c, MODE == 3);
            vhi[j] = lanes_mod_p((uint32_t)(r >> 32), c, MODE == 3);
            continue;
        }
        constexpr bool CORR1 = MODE == 1;
        // DQT pack by two byte dot products: (a0 + a1 q) + (a2 + a3 q) q^2 (digits < p <= q, q <= 2^7)
        const uint32_t wa = __dp4a(x, PK_LO, 0u) + (__dp4a(x, PK_HI, 0u) << (2 * T));
        const uint32_t wb = __dp4a(y, PK_LO, 0u) + (__dp4a(y, PK_HI, 0u) << (2 * T));
        // every digit of the product is < q (checked on the host), so r < q^7 <= 2^49: the packed
        // product is one 32 x 32 -> 64-bit integer multiply (exact), and enters the FP64
        // reciprocal as the low mantissa bits of 2^52 + r (one DADD; the FP64 product of the
        // two packed words needed two of those plus a DMUL and a DADD back to r's bits)
        const uint64_t ri = (uint64_t)wa * wb;
        const double rr = __longlong_as_double((long long)(0x4330000000000000ull | ri)) - two52;
        // r < 2^49 < fdiv bound B: floor(RN(r * RU(1/p))) = r // p with no correction branch
        const uint64_t si = (uint64_t)__double_as_longlong(__dadd_rd(__dmul_rn(rr, c.invp_up), two52));
        // u_i only matters mod 2^8 (it is small): byte windows of r and s
        uint32_t u[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) u[i] = (uint32_t)(ri >> (i * T)) + c.negp * (uint32_t)(si >> (i * T));
        if (CORR1) {  // mu_i = (u_i + u_{i+1}) mod p on byte lanes
            // U0 = [u0 u1 u2 u3], U1 = [u1 u2 u3 u4], W0 = [u4 u5 u6 0], W1 = [u5 u6 0 0]
            const uint32_t U0 = __byte_perm(__byte_perm(u[0], u[1], 0x0040), __byte_perm(u[2], u[3], 0x0040), 0x5410);
            const uint32_t U1 = __byte_perm(U0, u[4], 0x4321);
            const uint32_t W0 = __byte_perm(__byte_perm(u[4], u[5], 0x0040), u[6], 0x0410) & 0xFFFFFFu;
            const uint32_t W1 = W0 >> 8;
            // lane 2 of W0 + W1 is u6 < p (unchanged by the reduction), lane 3 is 0
            const uint32_t V0 = lanes_mod_2p(U0 + U1, c.p), V1 = lanes_mod_2p(W0 + W1, c.p);
            vlo[j] = V0;
            vhi[j] = V1;
        } else {
            uint64_t v = 0;
#pragma unroll
            // only the low byte of a window is u_i: the high windows of s carry the 2^52 exponent bits
            for (int i = 0; i < 6; ++i)
                v |= (uint64_t)mod_small((u[i] & 0xFFu) + c.corr * (u[i + 1] & 0xFFu), c.p, c.magic) << (8 * i);
            v |= (uint64_t)(u[6] & 0xFF) << 48;
            vlo[j] = (uint32_t)v;
            vhi[j] = (uint32_t)(v >> 32);
        }
    }
    // the thread's 56-byte output stream (pair j at bytes 7j..7j+6): every
    // aligned word is one byte permute of two result words
    uint32_t o[PM_PER * 7 / 4];
#pragma unroll
    for (int w = 0; w < PM_PER * 7 / 4; ++w) {
        const int j = 4 * w / 7, k = 4 * w - 7 * j;  // the word starts at byte k of pair j
        if (k + 4 <= 7) o[w] = __byte_perm(vlo[j], vhi[j], stream_sel(k, 0));
        else o[w] = __byte_perm(vhi[j], vlo[j + 1], stream_sel(k - 4, 7 - k));
    }
    uint8_t* dst = out + p0 * 7;
    // a warp with all its pairs in range stages its 32 x 56 output bytes in shared
    // memory and stores them as lane-consecutive 16-byte vectors
    __shared__ __align__(16) uint32_t pstage[PM_THREADS / 32][32 * PM_PER * 7 / 4];
    uint8_t* wbase = dst - (int64_t)lane * PM_PER * 7;  // the warp's first output byte
    if (wfast) {  // o[7v .. 7v+6]: pairs wp0 + 128 v + 4 l .. +3 (28 bytes each)
        uint32_t* st = pstage[threadIdx.x >> 5];
#pragma unroll
        for (int v = 0; v < PM_PER / 4; ++v)
#pragma unroll
            for (int q = 0; q < 7; ++q) st[224 * v + 7 * lane + q] = o[7 * v + q];  // word stride 7: conflict-free
        __syncwarp();
        constexpr int NV = 32 * PM_PER * 7 / 16;  // 16-byte vectors per warp
#pragma unroll
        for (int v = lane; v < NV; v += 32)
            reinterpret_cast<uint4*>(wbase)[v] = *reinterpret_cast<const uint4*>(st + 4 * v);
    } else if (__all_sync(0xffffffffu, full) && ((reinterpret_cast<uintptr_t>(wbase) & 15) == 0)) {
        uint32_t* st = pstage[threadIdx.x >> 5];
#pragma unroll
        if constexpr (PM_PER * 7 % 8 == 0) {
#pragma unroll
            for (int q = 0; q < PM_PER * 7 / 8; ++q)
                *reinterpret_cast<uint2*>(st + lane * (PM_PER * 7 / 4) + 2 * q) = make_uint2(o[2 * q], o[2 * q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < PM_PER * 7 / 4; ++q) st[lane * (PM_PER * 7 / 4) + q] = o[q];
        }
        __syncwarp();
        constexpr int NV = 32 * PM_PER * 7 / 16;  // 16-byte vectors per warp
#pragma unroll
        for (int v = lane; v < NV; v += 32)
            reinterpret_cast<uint4*>(wbase)[v] = *reinterpret_cast<const uint4*>(st + 4 * v);
    } else if (p0 >= n) {
        return;
    } else if (full && PM_PER * 7 % 8 == 0 && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
#pragma unroll
        for (int q = 0; q < PM_PER * 7 / 8; ++q) reinterpret_cast<uint2*>(dst)[q] = make_uint2(o[2 * q], o[2 * q + 1]);
    } else {
#pragma unroll
        for (int e = 0; e < PM_PER * 7; ++e)
            if (p0 + e / 7 < n) dst[e] = (uint8_t)(o[e >> 2] >> (8 * (e & 3)));
    }
}

template <int T>
static void launch_polymul_k4(const uint8_t* a, const uint8_t* b, int64_t n, const PolyConst& c, uint8_t* out,
                              cudaStream_t s) {
    // One wave, balanced: 4 blocks on every SM with the block width trimmed so
    // that the pairs spread evenly (cfg1: 592 x 224 threads instead of 512 x 256,
    // which left 68 SMs with a fourth block and the rest with three).  Larger
    // batches run 256-thread blocks in several waves.
    constexpr int PM_PER = T == 0 ? QADIC_PM_PER_LANES : QADIC_PM_PER;
    const int64_t per_wave = (int64_t)pm_minb(PM_PER) * num_sms_cached();
    int64_t threads = (n + per_wave * PM_PER - 1) / (per_wave * PM_PER);
    threads = (threads + 31) / 32 * 32;
    if (threads > PM_THREADS) threads = PM_THREADS;
    if (threads < 32) threads = 32;
    static const int width_env = getenv("QADIC_PM_WIDTH") ? atoi(getenv("QADIC_PM_WIDTH")) : 0;  // A/B knob
    if (width_env >= 32 && width_env <= PM_THREADS) threads = width_env / 32 * 32;
    const unsigned blocks = (unsigned)((n + threads * PM_PER - 1) / (threads * PM_PER));
    const int pf = pdl_prefetch_enabled();
    if constexpr (T == 0) {  // byte-lane form
        if (c.lfix) launch_pdl(polymul_k4_kernel<0, 3, PM_PER>, dim3(blocks), dim3((unsigned)threads), 0, s, a, b, n, c, out, pf);
        else launch_pdl(polymul_k4_kernel<0, 2, PM_PER>, dim3(blocks), dim3((unsigned)threads), 0, s, a, b, n, c, out, pf);
    } else if (c.corr == 1) {  // (p = 2: q is even, the correction factor is 0 -> the general form)
        launch_pdl(polymul_k4_kernel<T, 1, PM_PER>, dim3(blocks), dim3((unsigned)threads), 0, s, a, b, n, c, out, pf);
    } else {
        launch_pdl(polymul_k4_kernel<T, 0, PM_PER>, dim3(blocks), dim3((unsigned)threads), 0, s, a, b, n, c, out, pf);
    }
}

// (lm, lsh) with d - p * ((d * lm) >> lsh) in [0, p) (exact) or [0, 2p) for every digit
// d <= dmax, and dmax * lm <= 255 so that no lane of v * lm carries into the next; checked
// exhaustively.  Returns 0 if no pair exists, 1 for an exact quotient, 2 for one short by <= 1.
static int lane_quotient_consts(uint32_t p, uint32_t dmax, uint32_t* lm, uint32_t* lsh) {
    for (int want = 1; want <= 2; ++want)
        for (uint32_t sh = 0; sh < 8; ++sh)
            for (uint32_t m = 1; m * dmax <= 255; ++m) {
                bool ok = true;
                for (uint32_t d = 0; d <= dmax && ok; ++d) {
                    const uint32_t qh = (d * m) >> sh;
                    ok = qh * p <= d && d - qh * p < (uint32_t)want * p;
                }
                if (ok) {
                    *lm = m;
                    *lsh = sh;
                    return want;
                }
            }
    return 0;
}

// ---- generic k (1..8): one pair per thread ---------------------------------------
__global__ void polymul_generic_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                       int64_t n, int k, PolyConst c, uint8_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t wa = 0, wb = 0;
    for (int j = 0; j < k; ++j) {
        wa |= (uint64_t)a[i * k + j] << (j * c.t);
        wb |= (uint64_t)b[i * k + j] << (j * c.t);
    }
    const double r = (double)wa * (double)wb;  // exact: q^(2k-1) <= 2^53
    const int nd = 2 * k - 2;
    const uint64_t ri = (uint64_t)r;
    const uint64_t si = (uint64_t)fdiv_floor(r, c.invp_up, (double)c.p, c.bound);
    uint32_t prev = (uint32_t)ri - c.p * (uint32_t)si;
    for (int j = 0; j <= nd; ++j) {
        uint32_t next = 0;
        if (j < nd) next = (uint32_t)(ri >> ((j + 1) * c.t)) - c.p * (uint32_t)(si >> ((j + 1) * c.t));
        out[i * (nd + 1) + j] = (uint8_t)(j < nd ? mod_small(prev + c.corr * next, c.p, c.magic) : prev);
        prev = next;
    }
}

// ---- cfg2: GF(p^k) dot products ----------------------------------------------------
// G lanes per dot product (G = 4 on the vector path: a warp covers 8 dots, each
// load instruction reads 64 contiguous bytes per dot).  The delayed reduction
// (no modular work inside the sum) accumulates the dot's DQT word
//     r = sum_e pack(x_e) * pack(y_e) = sum_j S_j q^j,
//     S_j = sum_e sum_{i+i'=j} x_e[i] y_e[i']          (every S_j < q: the bound)
// On the vector path (K | 4) the digit sums S_j are formed directly on the
// coefficient bytes by 4-lane byte dot products (IDP4A) -- the packed product's
// digits without materialising the packed words: K = 2 costs 3 IDP4A + 3 logic
// ops per 2 elements instead of two packings and a wide multiply each.  r is
// assembled once per dot (exact, < 2^53), then REDQ (FP64 reciprocal +
// correction) and the L/H fold tables finish it exactly as in src/gfext.py:fgdp.
constexpr int GD_THREADS = 256;

// byte selectors: Y_j[i] = y[j - i] (0 outside 0..3), so dp4a(x, Y_j) = sum_i x_i y_{j-i}
__host__ __device__ constexpr uint32_t conv_selector(int j) {
    uint32_t sel = 0;
    for (int i = 0; i < 4; ++i) sel |= (uint32_t)((j - i >= 0 && j - i < 4) ? (j - i) : 4) << (4 * i);
    return sel;
}

template <int K>
QADIC_D void digit_sums_word(uint32_t x, uint32_t y, uint32_t (&S)[2 * K - 1]) {
    if constexpr (K == 1) {
        S[0] = __dp4a(x, y, S[0]);
    } else if constexpr (K == 2) {  // two elements (bytes 0,1 and 2,3); S[0] holds S_0 + S_2 until the end
        S[0] = __dp4a(x, y, S[0]);
        S[2] = __dp4a(x & 0xFF00FF00u, y, S[2]);
        S[1] = __dp4a(x, __byte_perm(y, 0, 0x2301), S[1]);
    } else {  // K == 4: one element per word
#pragma unroll
        for (int j = 0; j < 7; ++j) S[j] = __dp4a(x, __byte_perm(y, 0, conv_selector(j)), S[j]);
    }
}

// QADIC_GD_SLOWTAIL=1: the generic REDQ tail everywhere (measurement switch)
__constant__ int c_gd_slowtail = 0;
QADIC_D bool tail_slow() { return c_gd_slowtail != 0; }

// NARROW: registers capped at 32 (8 resident blocks per SM) for short rows, where
// the 4-deep load loop never runs (its spills stay cold) and a wave holds the batch.
// the paper's accumulation (F64ACC): DQT words of the 4/K elements of one 32-bit chunk word
// (digits < p <= q at shifts it; every word < 2^(K t) <= 2^53, so exact in a double)
template <int K>
QADIC_D void packed_words_f64(uint32_t x, int t, double (&w)[4 / K]) {
#pragma unroll
    for (int e = 0; e < 4 / K; ++e) {
        uint64_t v = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) v |= (uint64_t)((x >> (8 * (e * K + i))) & 0xFFu) << (i * t);
        w[e] = (double)v;
    }
}

template <int K, int G, bool VEC, bool NARROW = false, bool F64ACC = false>
__global__ void __launch_bounds__(GD_THREADS, NARROW ? 8 : 1) gf_dot_kernel(const uint8_t* __restrict__ v1,
                                                            const uint8_t* __restrict__ v2, int64_t batch,
                                                            int64_t len, FieldConst f, int tab_smem,
                                                            uint8_t* __restrict__ out, int pf) {
    if (pf && threadIdx.x == 0) {  // the block's rows towards L2 while the predecessor drains
        const int64_t rb = len * K, off = (int64_t)blockIdx.x * (blockDim.x / G) * rb;
        l2_prefetch_span(v1, off, (int64_t)(blockDim.x / G) * rb, batch * rb);
        l2_prefetch_span(v2, off, (int64_t)(blockDim.x / G) * rb, batch * rb);
    }
    pdl_wait();  // predecessor complete before any global load or store
    pdl_trigger();
    const int lane = threadIdx.x % G;
    const int64_t dot = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool live = dot < batch;
    const int t = (int)f.t;
    uint64_t acc = 0;
    if (live) {
        const int64_t row_bytes = len * K;
        const uint8_t* r1 = v1 + dot * row_bytes;
        const uint8_t* r2 = v2 + dot * row_bytes;
        if constexpr (VEC) {  // 16-byte chunks hold 16/K whole elements (K | 4)
            const int64_t nchunks = row_bytes / 16;
            const uint4* c1 = reinterpret_cast<const uint4*>(r1);
            const uint4* c2 = reinterpret_cast<const uint4*>(r2);
            uint32_t S[2 * K - 1];
#pragma unroll
            for (int j = 0; j < 2 * K - 1; ++j) S[j] = 0;
            double accd = 0.0;  // F64ACC: the packed products summed in FP64 (every sum < 2^53)
            auto word = [&](uint32_t xw, uint32_t yw) {
                if constexpr (F64ACC) {
                    double wx[4 / K], wy[4 / K];
                    packed_words_f64<K>(xw, t, wx);
                    packed_words_f64<K>(yw, t, wy);
#pragma unroll
                    for (int e = 0; e < 4 / K; ++e) accd = fma(wx[e], wy[e], accd);
                } else {
                    digit_sums_word<K>(xw, yw, S);
                }
            };
            auto body = [&](const uint4& x, const uint4& y) {
                word(x.x, y.x);
                word(x.y, y.y);
                word(x.z, y.z);
                word(x.w, y.w);
            };
            if constexpr (NARROW) {  // short rows: at most 2 chunks per lane (host-checked), no loop
                const uint4 z = make_uint4(0, 0, 0, 0);
                const uint4 x0 = lane < nchunks ? __ldg(c1 + lane) : z, y0 = lane < nchunks ? __ldg(c2 + lane) : z;
                const uint4 x1 = lane + G < nchunks ? __ldg(c1 + lane + G) : z;
                const uint4 y1 = lane + G < nchunks ? __ldg(c2 + lane + G) : z;
                body(x0, y0);
                body(x1, y1);
            } else {
            // every load of a lane issued before the first use
            int64_t ch = lane;
            for (; ch + 3 * G < nchunks; ch += 4 * G) {
                uint4 x[4], y[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    x[i] = __ldg(c1 + ch + i * G);
                    y[i] = __ldg(c2 + ch + i * G);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) body(x[i], y[i]);
            }
            if (ch + G < nchunks) {
                const uint4 x0 = __ldg(c1 + ch), y0 = __ldg(c2 + ch), x1 = __ldg(c1 + ch + G), y1 = __ldg(c2 + ch + G);
                body(x0, y0);
                body(x1, y1);
                ch += 2 * G;
            }
            if (ch < nchunks) body(__ldg(c1 + ch), __ldg(c2 + ch));
            }
            if constexpr (F64ACC) {
                acc = (uint64_t)accd;
            } else {
                if constexpr (K == 2) S[0] -= S[2];
                // the packed word: every S_j < q (host-checked), so r < q^(2K-1) <= 2^53
#pragma unroll
                for (int j = 0; j < 2 * K - 1; ++j) acc += (uint64_t)S[j] << (j * t);
            }
        } else {
            for (int64_t e = lane; e < len; e += G) {
                uint64_t wx = 0, wy = 0;
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    wx |= (uint64_t)r1[e * K + l] << (l * t);
                    wy |= (uint64_t)r2[e * K + l] << (l * t);
                }
                acc += wx * wy;  // < q^(2k-1) <= 2^53: exact
            }
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    // the L/H correction tables (gfext.py:176-213) staged in shared memory when
    // small -- after the operand loads, so their latency overlaps the table's
    extern __shared__ uint32_t gd_tab[];
    const uint32_t* ltab = f.l_table;
    const uint32_t* htab = f.h_table;
    if (tab_smem > 0) {  // (tab_smem == 0: tiny tables are read through L1 directly -- no barrier)
        for (int i = threadIdx.x; i < tab_smem; i += blockDim.x) {
            gd_tab[i] = __ldg(f.l_table + i);
            gd_tab[tab_smem + i] = __ldg(f.h_table + i);
        }
        __syncthreads();
        ltab = gd_tab;
        htab = gd_tab + tab_smem;
    }
    constexpr int ND = 2 * K - 2;
    if (!live || lane != 0) return;
    uint32_t u[ND + 1];
    if ((ND + 1) * t <= 32 && !tail_slow()) {
        // r < 2^32 (cfg2: 30 bits): the same FP64 REDQ without the conversion instructions --
        // r enters as the low mantissa bits of 2^52 + r, s = floor(RN(r RU(1/p))) leaves as the
        // low bits of the round-down sum with 2^52 (r < 2^32 < B: no correction branch)
        const double two52 = 4503599627370496.0;
        const uint32_t r32 = (uint32_t)acc;
        const double rd = __hiloint2double(0x43300000, (int)r32) - two52;
        const uint32_t s32 = (uint32_t)__double_as_longlong(__dadd_rd(__dmul_rn(rd, f.invp_up), two52));
#pragma unroll
        for (int i = 0; i <= ND; ++i) u[i] = (r32 >> (i * t)) - f.p * (s32 >> (i * t));
    } else {
        redq_compress_f64<ND>((double)acc, f.invp_up, (double)f.p, f.bound, f.p, t, u);
    }
    uint32_t li = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        li |= u[i] << (f.bb * i);
        hi |= u[K - 1 + i] << (f.bb * i);
    }
    const uint32_t res = add_coeff_bytes(ltab[li], htab[hi], f.p, K);
    if (K == 2 && (reinterpret_cast<uintptr_t>(out) & 1) == 0) {
        reinterpret_cast<uint16_t*>(out)[dot] = (uint16_t)res;
    } else if (K == 4 && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
        reinterpret_cast<uint32_t*>(out)[dot] = res;
    } else {
#pragma unroll
        for (int l = 0; l < K; ++l) out[dot * K + l] = (uint8_t)(res >> (8 * l));
    }
}

template <int K, bool F64ACC = false>
static void launch_gf_dot(const uint8_t* v1, const uint8_t* v2, int64_t batch, int64_t len, const FieldConst& f,
                          uint8_t* out, cudaStream_t s) {
    // digit sums in 32-bit lanes: every S_j < q = 2^t
    const bool vec = (4 % K == 0) && ((len * K) % 16 == 0) && ((uintptr_t)v1 % 16 == 0) &&
                     ((uintptr_t)v2 % 16 == 0) && f.t <= 32;
    const int entries = 1 << (f.bb * K);
    // 256 < entries <= 2048 (<= 16 KB of tables): staged in shared memory; tiny tables
    // (cfg2: 16 entries) stay in L1 -- no staging loop, no block barrier in the tail
    static const int tiny = getenv("QADIC_GD_TINY") ? atoi(getenv("QADIC_GD_TINY")) : 256;
    const int ntab = (entries <= 2048 && entries > tiny) ? entries : 0;
    const size_t smem = (size_t)ntab * 2 * sizeof(uint32_t);
    if (vec) {
        // 4 lanes per dot.  Short rows (cfg2: 8 chunks, 2 per lane) use the narrow
        // variant, whose 32 registers let 8 blocks reside per SM: the batch is one
        // wave (the 48-register variant ran 1.4 waves: 5.14 vs 4.97 us).  The block
        // width is trimmed to spread the batch evenly over the resident slots.
        const int64_t nchunks = len * K / 16;
        static const int max_width = getenv("QADIC_GD_WIDTH") ? atoi(getenv("QADIC_GD_WIDTH")) : GD_THREADS;
        static const int lanes = getenv("QADIC_GD_LANES") ? atoi(getenv("QADIC_GD_LANES")) : 4;
        static bool slow_set = false;
        if (!slow_set && getenv("QADIC_GD_SLOWTAIL")) {
            const int v = atoi(getenv("QADIC_GD_SLOWTAIL"));
            cudaMemcpyToSymbol(c_gd_slowtail, &v, sizeof(int));
        }
        slow_set = true;
        auto go = [&](auto kern, int G) {
            static int occ = 0;
            if (!occ) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, GD_THREADS, smem);
                if (occ < 1) occ = 1;
            }
            const int64_t threads_total = batch * G, per_wave = (int64_t)occ * num_sms_cached();
            int64_t width = (threads_total + per_wave - 1) / per_wave;
            width = (width + 31) / 32 * 32;
            if (width > max_width) width = max_width;
            if (width < 64) width = 64;
            const unsigned blocks = (unsigned)((threads_total + width - 1) / width);
            launch_pdl(kern, dim3(blocks), dim3((unsigned)width), smem, s, v1, v2, batch, len, f, ntab, out,
                       pdl_prefetch_enabled());
        };
        if (lanes == 8 && nchunks <= 2 * 8) go(gf_dot_kernel<K, 8, (4 % K == 0), true, F64ACC>, 8);
        else if (nchunks <= 2 * 4) go(gf_dot_kernel<K, 4, (4 % K == 0), true, F64ACC>, 4);
        else go(gf_dot_kernel<K, 4, (4 % K == 0), false, F64ACC>, 4);
    } else {
        constexpr int G = 8;
        const unsigned blocks = (unsigned)((batch * G + GD_THREADS - 1) / GD_THREADS);
        launch_pdl(gf_dot_kernel<K, G, false>, dim3(blocks), dim3(GD_THREADS), smem, s, v1, v2, batch, len, f, ntab,
                   out, 0);
    }
}

}  // namespace qadic

using namespace qadic;

namespace qadic {
// shared with the engines: validate a field descriptor and build the device view
int make_field_const(const qadic_field_desc* d, FieldConst* f) {
    QADIC_REQUIRE(d != nullptr, QADIC_ERR_VALUE, "null field descriptor");
    QADIC_REQUIRE(d->p >= 2 && d->p <= 127, QADIC_ERR_UNSUPPORTED, "GPU path supports 2 <= p <= 127 (got %d)", d->p);
    QADIC_REQUIRE(d->k >= 1 && d->k <= kMaxK, QADIC_ERR_UNSUPPORTED, "GPU path supports 1 <= k <= %d", kMaxK);
    QADIC_REQUIRE(d->t >= 1 && (2 * d->k - 1) * d->t <= 53, QADIC_ERR_PARAMS,
                  "q**(2k-1) exceeds the 2**53 word budget");
    QADIC_REQUIRE(d->u_bits >= 1 && d->u_bits * d->k <= 24, QADIC_ERR_UNSUPPORTED, "L/H table too large");
    QADIC_REQUIRE(d->l_table && d->h_table, QADIC_ERR_VALUE, "missing L/H tables");
    f->p = (uint32_t)d->p;
    f->k = (uint32_t)d->k;
    f->t = (uint32_t)d->t;
    f->bb = (uint32_t)d->u_bits;
    f->nd = 2 * f->k - 2;
    const uint64_t q = 1ull << d->t;
    f->corr = (q % f->p == 0) ? 0u : (uint32_t)((f->p - q % f->p) % f->p);
    f->magic = small_magic(f->p);
    f->invp_up = host_reciprocal_up(d->p);
    f->bound = host_case2_bound();
    for (int i = 0; i < kMaxDigits; ++i)
        for (int l = 0; l < kMaxK; ++l) f->xpow[i][l] = (i < 2 * d->k - 1 && l < d->k) ? d->xpow[i][l] : 0;
    f->l_table = d->l_table;
    f->h_table = d->h_table;
    return QADIC_OK;
}
}  // namespace qadic

extern "C" {

static int polymul_batch(const uint8_t* a, const uint8_t* b, int64_t n, int32_t k, int64_t p, int32_t t,
                         uint8_t* out, void* stream, bool redq_form) {
    QADIC_REQUIRE(n >= 0, QADIC_ERR_SHAPE, "negative batch");
    QADIC_REQUIRE(k >= 1 && k <= 8, QADIC_ERR_UNSUPPORTED, "packing width k must be 1..8");
    QADIC_REQUIRE(p >= 2 && p <= 127, QADIC_ERR_UNSUPPORTED, "GPU path supports 2 <= p <= 127");
    QADIC_REQUIRE(t >= 1 && (int64_t)(2 * k - 1) * t <= 53, QADIC_ERR_PARAMS, "word budget exceeded for 2d+1 digits");
    QADIC_REQUIRE((int64_t)k * (p - 1) * (p - 1) < (1ll << t), QADIC_ERR_PARAMS,
                  "q=2**%d too small for k=%d, p=%lld", t, k, (long long)p);
    if (n == 0) return QADIC_OK;
    PolyConst c;
    c.p = (uint32_t)p;
    c.t = (uint32_t)t;
    const uint64_t q = 1ull << t;
    c.corr = (q % c.p == 0) ? 0u : (uint32_t)((c.p - q % c.p) % c.p);
    c.magic = small_magic(c.p);
    c.negp = 0u - c.p;
    c.lm = c.lsh = c.lmask = c.lfix = 0;
    c.invp_up = host_reciprocal_up(p);
    c.bound = host_case2_bound();
    cudaStream_t s = (cudaStream_t)stream;
    const bool aligned = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)out % 16 == 0);
    // QADIC_PM_LANES=0: the paper's q = 2^t FP64-reciprocal REDQ form everywhere (measurement switch)
    static const bool lanes_env = !(getenv("QADIC_PM_LANES") && atoi(getenv("QADIC_PM_LANES")) == 0);
    const uint32_t dmax = 4u * (c.p - 1) * (c.p - 1);
    int lanes = 0;
    if (k == 4 && aligned && lanes_env && !redq_form && dmax <= 255) lanes = lane_quotient_consts(c.p, dmax, &c.lm, &c.lsh);
    if (lanes) {
        c.lmask = (0xFFu >> c.lsh) * 0x01010101u;
        c.lfix = lanes == 2;
        const int pi = prof_begin(s, "polymul_k4");
        count_launch(1);
        launch_polymul_k4<0>(a, b, n, c, out, s);
        prof_end(pi, s);
    } else if (k == 4 && aligned && t <= 7) {  // words < 2^28, products < 2^49 (exact, below the fdiv bound)
        const int pi = prof_begin(s, "polymul_k4");
        count_launch(1);
        switch (t) {
            case 1: launch_polymul_k4<1>(a, b, n, c, out, s); break;
            case 2: launch_polymul_k4<2>(a, b, n, c, out, s); break;
            case 3: launch_polymul_k4<3>(a, b, n, c, out, s); break;
            case 4: launch_polymul_k4<4>(a, b, n, c, out, s); break;
            case 5: launch_polymul_k4<5>(a, b, n, c, out, s); break;
            case 6: launch_polymul_k4<6>(a, b, n, c, out, s); break;
            default: launch_polymul_k4<7>(a, b, n, c, out, s); break;
        }
        prof_end(pi, s);
    } else {
        QADIC_TIMED("polymul_generic", s,
                    polymul_generic_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n, k, c, out));
    }
    return check_launch("polymul_batch_u8");
}

int qadic_diag_lane_quotient(uint32_t p, uint32_t dmax, uint32_t* m, uint32_t* sh) {
    uint32_t mm = 0, ss = 0;
    const int r = (p >= 2 && dmax <= 255) ? lane_quotient_consts(p, dmax, &mm, &ss) : 0;
    if (m) *m = mm;
    if (sh) *sh = ss;
    return r;
}

int qadic_polymul_batch_u8(const uint8_t* a, const uint8_t* b, int64_t n, int32_t k, int64_t p, int32_t t,
                           uint8_t* out, void* stream) {
    return polymul_batch(a, b, n, k, p, t, out, stream, false);
}

int qadic_polymul_batch_redq_u8(const uint8_t* a, const uint8_t* b, int64_t n, int32_t k, int64_t p, int32_t t,
                                uint8_t* out, void* stream) {
    return polymul_batch(a, b, n, k, p, t, out, stream, true);
}

static int gf_dot_batch(const qadic_field_desc* fd, const uint8_t* v1, const uint8_t* v2, int64_t batch, int64_t len,
                        uint8_t* out, void* stream, bool f64acc) {
    FieldConst f;
    int rc = make_field_const(fd, &f);
    if (rc) return rc;
    QADIC_REQUIRE(batch >= 0 && len >= 0, QADIC_ERR_SHAPE, "negative shape");
    // dot-product bound: every digit of the accumulator stays below q
    QADIC_REQUIRE((__int128)len * f.k * (f.p - 1) * (f.p - 1) < ((__int128)1 << f.t), QADIC_ERR_PARAMS,
                  "length %lld exceeds the digit capacity of q=2**%u", (long long)len, f.t);
    if (batch == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int pi = prof_begin(s, "gf_dot");
    count_launch(1);
    if (f64acc) {  // the FP64 form exists for the vector path (K | 4); K = 3 rows fall back to digit sums
        switch (f.k) {
            case 1: launch_gf_dot<1, true>(v1, v2, batch, len, f, out, s); break;
            case 2: launch_gf_dot<2, true>(v1, v2, batch, len, f, out, s); break;
            case 3: launch_gf_dot<3>(v1, v2, batch, len, f, out, s); break;
            default: launch_gf_dot<4, true>(v1, v2, batch, len, f, out, s); break;
        }
    } else {
        switch (f.k) {
            case 1: launch_gf_dot<1>(v1, v2, batch, len, f, out, s); break;
            case 2: launch_gf_dot<2>(v1, v2, batch, len, f, out, s); break;
            case 3: launch_gf_dot<3>(v1, v2, batch, len, f, out, s); break;
            default: launch_gf_dot<4>(v1, v2, batch, len, f, out, s); break;
        }
    }
    prof_end(pi, s);
    return check_launch("gf_dot_batch_u8");
}

int qadic_gf_dot_batch_u8(const qadic_field_desc* fd, const uint8_t* v1, const uint8_t* v2, int64_t batch,
                          int64_t len, uint8_t* out, void* stream) {
    return gf_dot_batch(fd, v1, v2, batch, len, out, stream, false);
}

int qadic_gf_dot_batch_f64_u8(const qadic_field_desc* fd, const uint8_t* v1, const uint8_t* v2, int64_t batch,
                              int64_t len, uint8_t* out, void* stream) {
    return gf_dot_batch(fd, v1, v2, batch, len, out, stream, true);
}

}  // extern "C"
