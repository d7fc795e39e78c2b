// Exhaustive FDIV certification scans on the GPU.
//
// Reference: fdiv.exhaustive_check / applied_fdiv_exhaustive
// (/root/reference/pkg/src/qadic/fdiv.py:405-461) certify Table 1
// and Alg. 4 by brute force in a
// beta-bit binary arithmetic: for every (r, p) in [0, 2^beta) x [1, 2^beta),
//   x = round2(r * round1(1/p)),  diff = floor(x) - r // p.
// The reference loops over p in Python with numpy vectors over r; here one
// CTA owns one divisor p and its threads stride over r, so a beta = 16 case
// (2^32 pairs) is one launch of milliseconds and beta up to 22 (2^44 pairs)
// takes seconds.  Pure integer ALU work (a 32-bit division and a
// handful of shifts per pair): no memory traffic, bound by the SM integer
// pipes.
//
// Rounding restates fdiv._vec_round_floor (fdiv.py:389-402) on exact 64-bit
// products (r * mantissa < 2^48): keep beta significant bits, round the
// dropped remainder (up: any non-zero; nearest: above half, or exactly half
// with an odd kept mantissa), then scale by the exponent with a floor shift.
// One difference, immaterial to every reported count: for products that
// already fit beta bits (nothing dropped) the reference's nearest mode adds
// one to odd mantissas (its `half` is 0 there); such products need r <= 1,
// where floor(x) is 0 (p >= 2) or exact (p = 1, even mantissa) either way.
#include <cuda_runtime.h>

#include <algorithm>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

namespace {

enum : int { MODE_UP = 0, MODE_NEAREST = 1, MODE_DOWN = 2 };

// round(1/p) to beta significant bits: mantissa in [2^(beta-1), 2^beta), value m * 2^e
// (fdiv.sim_reciprocal: exact rational rounding, ties to even)
__device__ __forceinline__ void reciprocal(uint32_t p, int beta, int mode, uint64_t& m, int& e) {
    const int L = 32 - __clz(p);  // bit length
    if ((p & (p - 1)) == 0) {
        m = 1ull << (beta - 1);
        e = -(beta - 1) - (L - 1);
        return;
    }
    const uint64_t num = 1ull << (beta - 1 + L);  // 2^(L-1) < p < 2^L: num / p in (2^(beta-1), 2^beta)
    m = num / p;
    const uint64_t rem = num - m * p;
    e = -(beta - 1 + L);
    if (mode == MODE_UP) m += rem != 0;
    else if (mode == MODE_NEAREST) m += (2 * rem > p) || (2 * rem == p && (m & 1));
    if (m == (1ull << beta)) {
        m >>= 1;
        e += 1;
    }
}

// floor(round_mode(prod to beta bits) * 2^e1), prod >= 0
__device__ __forceinline__ int64_t round_floor(uint64_t prod, int e1, int beta, int mode) {
    const int nbits = prod ? 64 - __clzll((long long)prod) : 0;
    const int shift = nbits > beta ? nbits - beta : 0;
    uint64_t mant = prod >> shift;
    if (shift > 0) {
        const uint64_t rem = prod - (mant << shift);
        const uint64_t half = 1ull << (shift - 1);
        if (mode == MODE_UP) mant += rem != 0;
        else if (mode == MODE_NEAREST) mant += (rem > half) || (rem == half && (mant & 1));
    }
    const int e = shift + e1;
    return (int64_t)(e >= 0 ? mant << e : mant >> (-e));
}

struct ScanAcc {
    unsigned long long range_viol, bound_viol;
    unsigned long long km1_key, kp1_key;  // (p << 32) | r, ~0 when none
    unsigned long long overflow_r;        // ~0 when none
};

constexpr int SCAN_THREADS = 256;

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(SCAN_THREADS) fdiv_scan_kernel(int beta, int mode1, int mode2, int lo, int hi,
                                                                 long long thr, uint32_t p0, ScanAcc* acc) {
    const uint32_t p = p0 + blockIdx.x;  // one divisor per CTA
    uint64_t m;
    int e1;
    reciprocal(p, beta, mode1, m, e1);
    const uint32_t R = 1u << beta;
    uint32_t rv = 0, bv = 0;
    uint32_t km1 = 0xffffffffu, kp1 = 0xffffffffu, over = 0xffffffffu;  // first r of each (r increases)
    for (uint32_t r = threadIdx.x; r < R; r += SCAN_THREADS) {
        const int64_t d = round_floor((uint64_t)r * m, e1, beta, mode2) - (int64_t)(r / p);
        rv += (d < lo) | (d > hi);
        if (d > 0) {
            bv += thr >= 0 && (long long)r <= thr;
            over = min(over, r);
        }
        if (d == -1) km1 = min(km1, r);
        if (d == 1) kp1 = min(kp1, r);
    }
    __shared__ unsigned long long red[5][SCAN_THREADS / 32];
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    const unsigned long long s0 = warp_sum(rv), s1 = warp_sum(bv);
    const unsigned long long m0 = warp_min(km1), m1 = warp_min(kp1), m2 = warp_min(over);
    if (l == 0) {
        red[0][w] = s0;
        red[1][w] = s1;
        red[2][w] = m0;
        red[3][w] = m1;
        red[4][w] = m2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0, c = ~0ull, dd = ~0ull, f = ~0ull;
        for (int i = 0; i < SCAN_THREADS / 32; ++i) {
            a += red[0][i];
            b += red[1][i];
            c = min(c, red[2][i]);
            dd = min(dd, red[3][i]);
            f = min(f, red[4][i]);
        }
        if (a) atomicAdd(&acc->range_viol, a);
        if (b) atomicAdd(&acc->bound_viol, b);
        if (lo == -1 && c != 0xffffffffull) atomicMin(&acc->km1_key, ((unsigned long long)p << 32) | c);
        if (hi == 1 && dd != 0xffffffffull) atomicMin(&acc->kp1_key, ((unsigned long long)p << 32) | dd);
        if (f != 0xffffffffull) atomicMin(&acc->overflow_r, f);
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) fdiv_applied_kernel(int beta, long long b_up, long long b_near,
                                                                    long long b_down, uint32_t p0,
                                                                    unsigned long long* mism) {
    const uint32_t p = p0 + blockIdx.x;
    // fdiv._PAIRED_MODE1: product up <- reciprocal nearest; nearest <- up; down <- up
    uint64_t m_near, m_up;
    int e_near, e_up;
    reciprocal(p, beta, MODE_NEAREST, m_near, e_near);
    reciprocal(p, beta, MODE_UP, m_up, e_up);
    const uint32_t R = 1u << beta;
    uint32_t bad = 0;
    for (uint32_t r = threadIdx.x; r < R; r += SCAN_THREADS) {
        const int64_t k = r / p;
        int64_t y = round_floor((uint64_t)r * m_near, e_near, beta, MODE_UP);
        y -= (long long)r >= b_up && (int64_t)p * y > (int64_t)r;
        bad += y != k;
        y = round_floor((uint64_t)r * m_up, e_up, beta, MODE_NEAREST);
        y -= (long long)r >= b_near && (int64_t)p * y > (int64_t)r;
        bad += y != k;
        y = round_floor((uint64_t)r * m_up, e_up, beta, MODE_DOWN);
        y -= (long long)r >= b_down && (int64_t)p * y > (int64_t)r;
        bad += y != k;
    }
    const unsigned long long s = warp_sum(bad);
    if (threadIdx.x % 32 == 0 && s) atomicAdd(mism, s);
}

constexpr int64_t MAX_CTAS_PER_LAUNCH = 1 << 22;

// Native (IEEE binary64) applied division on sampled pairs (fdiv.native_applied_random,
// reference fdiv.py:464-488): y = floor(RN(r * RU(1/p))), one multiply-back decrement
// above the case-2 threshold, compared with the exact 64-bit r // p.  Block j of
// the grid-stride loop owns divisor j / per_p's numerators r[j*per_p ...].
__global__ void fdiv_native_kernel(const int64_t* __restrict__ r, int64_t per_p, const int64_t* __restrict__ p,
                                   const double* __restrict__ invp, int64_t n_p, long long thr,
                                   unsigned long long* mism) {
    unsigned long long bad = 0;
    const int64_t total = per_p * n_p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / per_p;
        const int64_t pj = p[j], ri = r[i];
        int64_t y = (int64_t)floor(__dmul_rn((double)ri, invp[j]));
        y -= (ri > thr) && (pj * y > ri);
        bad += y != ri / pj;
    }
    const unsigned long long sum = warp_sum(bad);
    if (threadIdx.x % 32 == 0 && sum) atomicAdd(mism, sum);
}

}  // namespace

}  // namespace qadic

using namespace qadic;

extern "C" {

int qadic_fdiv_scan(int32_t beta, int32_t mode1, int32_t mode2, int32_t range_lo, int32_t range_hi,
                    int64_t bound_threshold, qadic_fdiv_scan_report* out, void* stream) {
    QADIC_REQUIRE(beta >= 4 && beta <= 22, QADIC_ERR_VALUE, "exhaustive scans support beta in 4..22");
    QADIC_REQUIRE(mode1 >= 0 && mode1 <= 2 && mode2 >= 0 && mode2 <= 2, QADIC_ERR_VALUE, "mode must be 0..2");
    QADIC_REQUIRE(out != nullptr, QADIC_ERR_VALUE, "null report");
    cudaStream_t s = (cudaStream_t)stream;
    ScanAcc init = {0, 0, ~0ull, ~0ull, ~0ull}, res;
    ScanAcc* acc = nullptr;
    QADIC_REQUIRE(cudaMallocAsync(reinterpret_cast<void**>(&acc), sizeof(ScanAcc), s) == cudaSuccess,
                  QADIC_ERR_CUDA, "scan scratch allocation failed");
    cudaMemcpyAsync(acc, &init, sizeof(init), cudaMemcpyHostToDevice, s);
    const int64_t np = (1ll << beta) - 1;
    for (int64_t p0 = 1; p0 <= np; p0 += MAX_CTAS_PER_LAUNCH) {
        const int64_t cnt = np - p0 + 1 < MAX_CTAS_PER_LAUNCH ? np - p0 + 1 : MAX_CTAS_PER_LAUNCH;
        fdiv_scan_kernel<<<(unsigned)cnt, SCAN_THREADS, 0, s>>>(beta, mode1, mode2, range_lo, range_hi,
                                                               (long long)bound_threshold, (uint32_t)p0, acc);
    }
    cudaMemcpyAsync(&res, acc, sizeof(res), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(acc, s);
    int rc = check_launch("fdiv_scan", (int)((np + MAX_CTAS_PER_LAUNCH - 1) / MAX_CTAS_PER_LAUNCH));
    if (rc) return rc;
    QADIC_REQUIRE(cudaStreamSynchronize(s) == cudaSuccess, QADIC_ERR_CUDA, "fdiv_scan: %s",
                  cudaGetErrorString(cudaGetLastError()));
    out->pairs_checked = (uint64_t)np << beta;
    out->range_violations = res.range_viol;
    out->bound_violations = res.bound_viol;
    out->k_minus_1_p = res.km1_key == ~0ull ? -1 : (int64_t)(res.km1_key >> 32);
    out->k_minus_1_r = res.km1_key == ~0ull ? -1 : (int64_t)(res.km1_key & 0xffffffffu);
    out->k_plus_1_p = res.kp1_key == ~0ull ? -1 : (int64_t)(res.kp1_key >> 32);
    out->k_plus_1_r = res.kp1_key == ~0ull ? -1 : (int64_t)(res.kp1_key & 0xffffffffu);
    out->smallest_overflow_r = res.overflow_r == ~0ull ? -1 : (int64_t)res.overflow_r;
    return QADIC_OK;
}

int qadic_fdiv_applied_scan(int32_t beta, const int64_t bound[3], uint64_t* mismatches, void* stream) {
    QADIC_REQUIRE(beta >= 4 && beta <= 22, QADIC_ERR_VALUE, "exhaustive scans support beta in 4..22");
    QADIC_REQUIRE(bound != nullptr && mismatches != nullptr, QADIC_ERR_VALUE, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* acc = nullptr;
    unsigned long long res = 0;
    QADIC_REQUIRE(cudaMallocAsync(reinterpret_cast<void**>(&acc), sizeof(*acc), s) == cudaSuccess, QADIC_ERR_CUDA,
                  "scan scratch allocation failed");
    cudaMemsetAsync(acc, 0, sizeof(*acc), s);
    const int64_t np = (1ll << beta) - 1;
    for (int64_t p0 = 1; p0 <= np; p0 += MAX_CTAS_PER_LAUNCH) {
        const int64_t cnt = np - p0 + 1 < MAX_CTAS_PER_LAUNCH ? np - p0 + 1 : MAX_CTAS_PER_LAUNCH;
        fdiv_applied_kernel<<<(unsigned)cnt, SCAN_THREADS, 0, s>>>(beta, (long long)bound[0], (long long)bound[1],
                                                                  (long long)bound[2], (uint32_t)p0, acc);
    }
    cudaMemcpyAsync(&res, acc, sizeof(res), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(acc, s);
    int rc = check_launch("fdiv_applied_scan", (int)((np + MAX_CTAS_PER_LAUNCH - 1) / MAX_CTAS_PER_LAUNCH));
    if (rc) return rc;
    QADIC_REQUIRE(cudaStreamSynchronize(s) == cudaSuccess, QADIC_ERR_CUDA, "fdiv_applied_scan: %s",
                  cudaGetErrorString(cudaGetLastError()));
    *mismatches = res;
    return QADIC_OK;
}

int qadic_fdiv_native_check(const int64_t* r, int64_t per_p, const int64_t* p, const double* invp, int64_t n_p,
                            int64_t threshold, uint64_t* mismatches, void* stream) {
    QADIC_REQUIRE(per_p >= 0 && n_p >= 0 && mismatches != nullptr, QADIC_ERR_VALUE, "bad arguments");
    *mismatches = 0;
    if (per_p == 0 || n_p == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* acc = nullptr;
    unsigned long long res = 0;
    QADIC_REQUIRE(cudaMallocAsync(reinterpret_cast<void**>(&acc), sizeof(*acc), s) == cudaSuccess, QADIC_ERR_CUDA,
                  "scratch allocation failed");
    cudaMemsetAsync(acc, 0, sizeof(*acc), s);
    const int64_t total = per_p * n_p;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms_cached() * 8);
    QADIC_TIMED("fdiv_native", s,
                fdiv_native_kernel<<<(unsigned)blocks, 256, 0, s>>>(r, per_p, p, invp, n_p, (long long)threshold, acc));
    cudaMemcpyAsync(&res, acc, sizeof(res), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(acc, s);
    int rc = check_launch("fdiv_native_check", 0);
    if (rc) return rc;
    QADIC_REQUIRE(cudaStreamSynchronize(s) == cudaSuccess, QADIC_ERR_CUDA, "fdiv_native_check: %s",
                  cudaGetErrorString(cudaGetLastError()));
    *mismatches = res;
    return QADIC_OK;
}

}  // extern "C"
