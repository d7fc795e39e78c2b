// HBM-bound batched kernels of the hot path:
//
//  * cfg1  polymul_batch : one packed FP64 product per pair of short
//    polynomials, then REDQ (compression + correction) -> 2k-1 residues.
//    Reference: polymul.polymul_fqt for one-word operands
//    (src/polymul.py:274-313 -> _wordconv_reduce :175-216 with na = nb = 1).
//  * cfg2  gf_dot_batch  : GF(p^k) dot products with all products accumulated
//    unreduced in FP64, then REDQ and the L/H correction+fold tables staged
//    in shared memory.  Reference: GFqField.fgdp (src/gfext.py:268-309).
//
// Both read uint8 coefficients with 128-bit loads and never touch the
// packed words in HBM: DQT packing happens in registers.
#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

// exact double of an integer w < 2^52 without the FP64 conversion unit
QADIC_D double u52_to_f64(uint64_t w) {
    return __longlong_as_double((long long)(0x4330000000000000ull | w)) - 4503599627370496.0;
}

QADIC_D uint32_t pack4(uint32_t bytes, int t) {
    return (bytes & 0xFF) | (((bytes >> 8) & 0xFF) << t) | (((bytes >> 16) & 0xFF) << (2 * t)) |
           ((bytes >> 24) << (3 * t));
}

struct PolyConst {
    uint32_t p, t, corr, magic;
    double invp_up, bound;
};

// ---- cfg1 fast path: k = 4 (degree-3 operands), 4 pairs per thread ----------
constexpr int PM_THREADS = 256;
constexpr int PM_PAIRS = 4 * PM_THREADS;  // pairs per block

__global__ void __launch_bounds__(PM_THREADS) polymul_k4_kernel(const uint8_t* __restrict__ a,
                                                                const uint8_t* __restrict__ b, int64_t n,
                                                                PolyConst c, uint8_t* __restrict__ out) {
    __shared__ __align__(16) uint8_t sout[PM_PAIRS * 7];
    const int64_t base = (int64_t)blockIdx.x * PM_PAIRS;
    const int64_t my = base + 4 * threadIdx.x;
    uint32_t av[4] = {0, 0, 0, 0}, bv[4] = {0, 0, 0, 0};
    if (my + 4 <= n) {
        const uint4 va = __ldg(reinterpret_cast<const uint4*>(a + my * 4));
        const uint4 vb = __ldg(reinterpret_cast<const uint4*>(b + my * 4));
        av[0] = va.x; av[1] = va.y; av[2] = va.z; av[3] = va.w;
        bv[0] = vb.x; bv[1] = vb.y; bv[2] = vb.z; bv[3] = vb.w;
    } else {
        for (int i = 0; i < 4; ++i)
            if (my + i < n) {
                av[i] = *reinterpret_cast<const uint32_t*>(a + (my + i) * 4);
                bv[i] = *reinterpret_cast<const uint32_t*>(b + (my + i) * 4);
            }
    }
    const double pd = (double)c.p;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double r = u52_to_f64(pack4(av[i], c.t)) * u52_to_f64(pack4(bv[i], c.t));
        uint32_t u[7];
        redq_compress_f64<6>(r, c.invp_up, pd, c.bound, c.p, c.t, u);
        uint8_t* o = sout + (4 * threadIdx.x + i) * 7;
#pragma unroll
        for (int j = 0; j < 6; ++j) o[j] = (uint8_t)mod_small(u[j] + c.corr * u[j + 1], c.p, c.magic);
        o[6] = (uint8_t)u[6];
    }
    __syncthreads();
    const int64_t npairs = (n - base) < PM_PAIRS ? (n - base) : PM_PAIRS;
    const int64_t nbytes = npairs * 7;
    uint8_t* gout = out + base * 7;
    if (nbytes == PM_PAIRS * 7) {
        const uint4* s4 = reinterpret_cast<const uint4*>(sout);
        uint4* g4 = reinterpret_cast<uint4*>(gout);
        for (int i = threadIdx.x; i < PM_PAIRS * 7 / 16; i += PM_THREADS) g4[i] = s4[i];
    } else {
        for (int64_t i = threadIdx.x; i < nbytes; i += PM_THREADS) gout[i] = sout[i];
    }
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
constexpr int GD_THREADS = 256;
constexpr int GD_GROUP = 8;  // lanes per dot product
constexpr int GD_SMEM_TABLE = 4096;

template <int K, bool VEC, bool SMEM_TABLES>
__global__ void __launch_bounds__(GD_THREADS) gf_dot_kernel(const uint8_t* __restrict__ v1,
                                                            const uint8_t* __restrict__ v2, int64_t batch,
                                                            int64_t len, FieldConst f,
                                                            uint8_t* __restrict__ out) {
    __shared__ uint32_t s_l[SMEM_TABLES ? GD_SMEM_TABLE : 1];
    __shared__ uint32_t s_h[SMEM_TABLES ? GD_SMEM_TABLE : 1];
    const uint32_t* ltab = f.l_table;
    const uint32_t* htab = f.h_table;
    if (SMEM_TABLES) {
        const int size = 1 << (f.bb * K);
        for (int i = threadIdx.x; i < size; i += GD_THREADS) {
            s_l[i] = f.l_table[i];
            s_h[i] = f.h_table[i];
        }
        __syncthreads();
        ltab = s_l;
        htab = s_h;
    }
    const int lane = threadIdx.x % GD_GROUP;
    const int64_t dot = ((int64_t)blockIdx.x * GD_THREADS + threadIdx.x) / GD_GROUP;
    const bool live = dot < batch;
    const int t = (int)f.t;
    double acc = 0.0;
    if (live) {
        const int64_t row_bytes = len * K;
        const uint8_t* r1 = v1 + dot * row_bytes;
        const uint8_t* r2 = v2 + dot * row_bytes;
        if (VEC) {  // 16-byte chunks hold 16/K whole elements (K | 16)
            const int64_t nchunks = row_bytes / 16;
            for (int64_t ch = lane; ch < nchunks; ch += GD_GROUP) {
                const uint4 x = __ldg(reinterpret_cast<const uint4*>(r1) + ch);
                const uint4 y = __ldg(reinterpret_cast<const uint4*>(r2) + ch);
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int e = 0; e < 4 / K; ++e) {
                        uint64_t wx = 0, wy = 0;
#pragma unroll
                        for (int l = 0; l < K; ++l) {
                            wx |= (uint64_t)((xs[q] >> (8 * (e * K + l))) & 0xFF) << (l * t);
                            wy |= (uint64_t)((ys[q] >> (8 * (e * K + l))) & 0xFF) << (l * t);
                        }
                        acc = fma(u52_to_f64(wx), u52_to_f64(wy), acc);
                    }
                }
            }
        } else {
            for (int64_t e = lane; e < len; e += GD_GROUP) {
                uint64_t wx = 0, wy = 0;
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    wx |= (uint64_t)r1[e * K + l] << (l * t);
                    wy |= (uint64_t)r2[e * K + l] << (l * t);
                }
                acc = fma(u52_to_f64(wx), u52_to_f64(wy), acc);
            }
        }
    }
#pragma unroll
    for (int off = GD_GROUP / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (!live || lane != 0) return;
    constexpr int ND = 2 * K - 2;
    uint32_t u[ND + 1];
    redq_compress_f64<ND>(acc, f.invp_up, (double)f.p, f.bound, f.p, t, u);
    uint32_t li = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        li |= u[i] << (f.bb * i);
        hi |= u[K - 1 + i] << (f.bb * i);
    }
    const uint32_t res = add_coeff_bytes(ltab[li], htab[hi], f.p, K);
#pragma unroll
    for (int l = 0; l < K; ++l) out[dot * K + l] = (uint8_t)(res >> (8 * l));
}

template <int K>
static void launch_gf_dot(const uint8_t* v1, const uint8_t* v2, int64_t batch, int64_t len, const FieldConst& f,
                          uint8_t* out, cudaStream_t s) {
    const bool vec = (16 % K == 0) && ((len * K) % 16 == 0) && ((uintptr_t)v1 % 16 == 0) &&
                     ((uintptr_t)v2 % 16 == 0);
    const bool smem = (1 << (f.bb * K)) <= GD_SMEM_TABLE;
    const unsigned blocks = (unsigned)((batch * GD_GROUP + GD_THREADS - 1) / GD_THREADS);
    if (vec && smem) gf_dot_kernel<K, (16 % K == 0), true><<<blocks, GD_THREADS, 0, s>>>(v1, v2, batch, len, f, out);
    else if (vec) gf_dot_kernel<K, (16 % K == 0), false><<<blocks, GD_THREADS, 0, s>>>(v1, v2, batch, len, f, out);
    else if (smem) gf_dot_kernel<K, false, true><<<blocks, GD_THREADS, 0, s>>>(v1, v2, batch, len, f, out);
    else gf_dot_kernel<K, false, false><<<blocks, GD_THREADS, 0, s>>>(v1, v2, batch, len, f, out);
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

int qadic_polymul_batch_u8(const uint8_t* a, const uint8_t* b, int64_t n, int32_t k, int64_t p, int32_t t,
                           uint8_t* out, void* stream) {
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
    c.invp_up = host_reciprocal_up(p);
    c.bound = host_case2_bound();
    cudaStream_t s = (cudaStream_t)stream;
    const bool aligned = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)out % 16 == 0);
    if (k == 4 && aligned && 3 * t + 8 <= 32) {  // pack4 keeps words in 32 bits
        QADIC_TIMED("polymul_k4", s,
                    polymul_k4_kernel<<<(unsigned)((n + PM_PAIRS - 1) / PM_PAIRS), PM_THREADS, 0, s>>>(a, b, n, c, out));
    } else {
        QADIC_TIMED("polymul_generic", s,
                    polymul_generic_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n, k, c, out));
    }
    return check_launch("polymul_batch_u8");
}

int qadic_gf_dot_batch_u8(const qadic_field_desc* fd, const uint8_t* v1, const uint8_t* v2, int64_t batch,
                          int64_t len, uint8_t* out, void* stream) {
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
    switch (f.k) {
        case 1: launch_gf_dot<1>(v1, v2, batch, len, f, out, s); break;
        case 2: launch_gf_dot<2>(v1, v2, batch, len, f, out, s); break;
        case 3: launch_gf_dot<3>(v1, v2, batch, len, f, out, s); break;
        default: launch_gf_dot<4>(v1, v2, batch, len, f, out, s); break;
    }
    prof_end(pi, s);
    return check_launch("gf_dot_batch_u8");
}

}  // extern "C"
