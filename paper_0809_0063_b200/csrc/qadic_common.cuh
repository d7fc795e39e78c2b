// Shared device helpers for the qadic B200 kernels.
//
// REDQ on the GPU (reference: src/redq.py:58-128, src/_kernels/_speed.pyx:121-130,
// PAPER.md:312-342).  For an accumulator r < 2^53 held exactly in a double:
//
//   s   = floor(RN(r * RU(1/p)))          one DMUL, no integer division
//         (+ one multiply-back decrement when r >= B, B = fdiv case-2 bound,
//          src/fdiv.py:338-363 -- cold at every config: all r < 2^51 < B)
//   u_i = lo32(r >> i t) - p * lo32(s >> i t)   (mod 2^32)
//
// The true u_i lies in [0, p) (nested flooring, src/redq.py:6-8), so the
// 32-bit wrap-around difference is exact and each digit costs one funnel
// shift pair and one IMAD instead of the reference's 64-bit paired fields
// (src/redq.py:88-115).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define QADIC_HD __host__ __device__ __forceinline__
#define QADIC_D __device__ __forceinline__

namespace qadic {

// Programmatic dependent launch (the batched cfg1/cfg2 kernels: back-to-back
// single-wave launches): kernels launched with launch_pdl() may start while their
// stream predecessor drains; pdl_wait() (first thing, before any global memory
// access) blocks until the predecessor grid has completed and its writes are
// visible, pdl_trigger() lets this grid's successor begin launching.  Both are
// no-ops for an ordinary launch.  Not used for the tensor-core chain: there an
// early-resident GEMM CTA (227 KB smem) starves the preceding plane kernel's
// tail of SMs (measured 2% slower at cfg5).
QADIC_D void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
QADIC_D void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// L2 prefetch hint for the byte range [off, off + bytes) of a read-only operand of
// `total` bytes (clipped to the operand, 16-byte granules), issued by ONE thread
// BEFORE pdl_wait(): a block that became resident while the stream predecessor
// drains uses the wait to pull its inputs from HBM into L2.  A prefetch returns no
// data to the SM and L2 is the GPU's point of coherence, so a predecessor that is
// still writing the range is seen correctly by the loads after the wait.
QADIC_D void l2_prefetch_span(const void* base, int64_t off, int64_t bytes, int64_t total) {
    uintptr_t lo = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(off < 0 ? 0 : off);
    int64_t end = off + bytes > total ? total : off + bytes;
    uintptr_t hi = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(end < 0 ? 0 : end);
    lo = (lo + 15) & ~(uintptr_t)15;
    hi &= ~(uintptr_t)15;
    if (hi > lo) {
        const uint32_t sz = (uint32_t)(hi - lo);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(sz) : "memory");
    }
}

constexpr int kMaxK = 4;             // extension degree supported by the GF kernels
constexpr int kMaxDigits = 2 * kMaxK - 1;

// x mod p for 0 <= x < 2^24, p < 256:  q = umulhi(x, floor(2^32/p)+1) is exact.
QADIC_D uint32_t mod_small(uint32_t x, uint32_t p, uint32_t magic) {
    return x - p * __umulhi(x, magic);
}

// x mod p for any 32-bit x (p < 2^26): 64-bit magic floor(2^64/p)+1.
QADIC_D uint32_t mod_u32(uint32_t x, uint32_t p, uint64_t magic64) {
    uint64_t q = __umul64hi((uint64_t)x, magic64);
    return x - (uint32_t)q * p;
}

QADIC_HD uint32_t small_magic(uint32_t p) { return (uint32_t)(0xFFFFFFFFull / p) + 1u; }
QADIC_HD uint64_t wide_magic(uint32_t p) { return 0xFFFFFFFFFFFFFFFFull / p + 1ull; }

// Exact floor(r / p) for integer-valued 0 <= r < 2^53 via the RU reciprocal
// and a RN product (fdiv case 2).  `bound` is the first r that may need the
// multiply-back test; the branch is cold whenever r < bound.
QADIC_D double fdiv_floor(double r, double invp_up, double p, double bound) {
    double y = floor(__dmul_rn(r, invp_up));
    if (r >= bound) {
        if (__dmul_rn(p, y) > r) y -= 1.0;
    }
    return y;
}

// Compressed digits u_0..u_{nd} of r (r < 2^53, exact integer in a double).
template <int ND>
QADIC_D void redq_compress_f64(double r, double invp_up, double pd, double bound, uint32_t p,
                               int t, uint32_t (&u)[ND + 1]) {
    const uint64_t ri = (uint64_t)r;
    const uint64_t si = (uint64_t)fdiv_floor(r, invp_up, pd, bound);
#pragma unroll
    for (int i = 0; i <= ND; ++i) {
        const uint32_t rl = (uint32_t)(ri >> (i * t));
        const uint32_t sl = (uint32_t)(si >> (i * t));
        u[i] = rl - p * sl;
    }
}

// Runtime-digit-count variant (nd <= kMaxDigits-1).
QADIC_D void redq_compress_f64_rt(double r, double invp_up, double pd, double bound, uint32_t p,
                                  int t, int nd, uint32_t* u) {
    const uint64_t ri = (uint64_t)r;
    const uint64_t si = (uint64_t)fdiv_floor(r, invp_up, pd, bound);
#pragma unroll
    for (int i = 0; i < kMaxDigits; ++i) {
        if (i <= nd) u[i] = (uint32_t)(ri >> (i * t)) - p * (uint32_t)(si >> (i * t));
    }
}

// Parameters of one GF(p^k) field as the kernels see it (by value).
struct FieldConst {
    uint32_t p, k, t, bb;      // prime, degree, radix exponent, bits per digit in L/H index
    uint32_t nd;               // 2k-2 : top digit of a product word
    uint32_t corr;             // (-q) mod p : correction multiplier (src/redq.py:308-315)
    uint32_t magic;            // small_magic(p)
    double invp_up;            // RU(1/p)
    double bound;              // fdiv case-2 bound B
    uint8_t xpow[kMaxDigits][kMaxK];   // X^i mod f, i <= 2k-2
    const uint32_t* l_table;   // device: 2^(bb*k) entries, k coefficient bytes each
    const uint32_t* h_table;
};

QADIC_D uint32_t add_coeff_bytes(uint32_t a, uint32_t b, uint32_t p, int k) {
    uint32_t out = 0;
#pragma unroll
    for (int l = 0; l < kMaxK; ++l) {
        if (l < k) {
            uint32_t s = ((a >> (8 * l)) & 0xFF) + ((b >> (8 * l)) & 0xFF);
            if (s >= p) s -= p;
            out |= s << (8 * l);
        }
    }
    return out;
}

}  // namespace qadic

// ---------------------------------------------------------------------------
// host-side error plumbing shared by every translation unit
// ---------------------------------------------------------------------------
namespace qadic {
void set_error(int code, const char* fmt, ...);
int check_launch(const char* what, int launched = 0);
}  // namespace qadic

#define QADIC_REQUIRE(cond, code, ...)            \
    do {                                          \
        if (!(cond)) {                            \
            ::qadic::set_error(code, __VA_ARGS__); \
            return code;                          \
        }                                         \
    } while (0)
