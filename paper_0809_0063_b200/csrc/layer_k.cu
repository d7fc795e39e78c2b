// Layer K of the qadic operator API on B200: the five reference kernels
// (src/_kernels/_speed.pyx) with identical integer semantics, plus the bulk
// REDQ reduction (src/redq.py:318-343), the DQT row packers
// (src/cmm.py:72-85, 130-145) and the handle <-> coefficient gathers
// (src/gfext.py:136-146).
//
// These are exact-semantics primitives (uint64 wrap-around GEMM, any-width
// REDQ); the throughput engines for the configs live in engine_tc.cu,
// engine_f64.cu and batched.cu, behind the operation-level API where the
// parameters prove the digit bounds.
#include <algorithm>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

bool tc_u64_ok(int64_t m, int64_t k, int64_t n, const void* a);
int tc_matmul_u64(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t m, int64_t k, int64_t n,
                  cudaStream_t s);

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

// Vectorised REDQ for D = d (compile time): each thread takes two consecutive
// words (one 16-byte load); a warp's 64(D+1) digits are staged in shared memory
// and stored as lane-consecutive 16-byte vectors, the repacked words as one
// 16-byte store per thread; grid-stride over a one-wave grid.
// The correction mu_i = (u_i + c*u_{i+1}) mod p is a lookup in the tabulated
// correction (redq.py:194-300 with one-digit blocks) staged in shared memory
// (p*p bytes, p <= 127) whenever both digits are reduced (u < p, always so for
// in-range words); anything else takes the exact uint64 path of _speed.pyx.
constexpr int RQ_THREADS = 256;
constexpr int RQ_TAB = 127 * 127;

template <int D>
__device__ __forceinline__ void redq_word(uint64_t ri, uint64_t p, int t, double invp_up, double bound, uint64_t corr,
                                          int mode, const uint8_t* tab, uint64_t (&out)[D + 1], uint64_t& word) {
    const uint64_t s = div_p(ri, p, invp_up, bound);
    // u_i = floor(r / 2^(it)) mod p lies in [0, p): 32-bit wrap-around arithmetic
    // on the low words is exact (one funnel shift per operand + one IMAD with -p)
    const uint32_t negp = 0u - (uint32_t)p;
    uint64_t u[D + 1];
#pragma unroll
    for (int i = 0; i <= D; ++i) u[i] = (uint32_t)(ri >> (i * t)) + negp * (uint32_t)(s >> (i * t));
    word = 0;
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        uint64_t o = u[i];
        if (mode >= 1 && i < D) {
            if (tab != nullptr && u[i] < p && u[i + 1] < p) o = tab[u[i] * p + u[i + 1]];
            else o = (u[i] + corr * u[i + 1]) % p;
        }
        out[i] = o;
        word += o << (i * t);
    }
}

template <int D>
__global__ void __launch_bounds__(RQ_THREADS) redq_vec_kernel(const uint64_t* __restrict__ r, int64_t n, uint64_t p,
                                                              int t, double invp_up, double bound, uint64_t corr,
                                                              int mode, uint64_t* __restrict__ digits,
                                                              uint64_t* __restrict__ packed) {
    __shared__ uint8_t stab[RQ_TAB];
    const bool use_tab = mode >= 1 && p * p <= (uint64_t)RQ_TAB;
    if (use_tab) {
        for (int i = threadIdx.x; i < (int)(p * p); i += RQ_THREADS)
            stab[i] = (uint8_t)(((uint64_t)(i / (int)p) + corr * (uint64_t)(i % (int)p)) % p);
        __syncthreads();
    }
    const uint8_t* tab = use_tab ? stab : nullptr;
    // digits of a warp's 64 words are one contiguous run: stage them in shared
    // memory and store the run with lane-consecutive 16-byte vectors
    __shared__ __align__(16) uint64_t stage[RQ_THREADS / 32][64 * (D + 1)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t pairs = n / 2;
    const int64_t stride = (int64_t)gridDim.x * RQ_THREADS;
    // the next iteration's pair of words is loaded before this one is reduced (two loads in
    // flight per thread: the kernel's stalls were the load latency, ncu long scoreboard)
    ulonglong2 xn = make_ulonglong2(0, 0);
    {
        const int64_t qf = (int64_t)blockIdx.x * RQ_THREADS + threadIdx.x;
        if (qf < pairs) xn = __ldcs(reinterpret_cast<const ulonglong2*>(r) + qf);
    }
    for (int64_t q0 = (int64_t)blockIdx.x * RQ_THREADS; q0 < pairs; q0 += stride) {
        const int64_t q = q0 + threadIdx.x;
        const int64_t qw = q0 + 32 * wid;  // first pair of this warp
        const bool live = q < pairs;
        uint64_t o0[D + 1], o1[D + 1], w0 = 0, w1 = 0;
        const ulonglong2 x = xn;
        if (q + stride < pairs) xn = __ldcs(reinterpret_cast<const ulonglong2*>(r) + q + stride);
        if (live) {
            redq_word<D>(x.x, p, t, invp_up, bound, corr, mode, tab, o0, w0);
            redq_word<D>(x.y, p, t, invp_up, bound, corr, mode, tab, o1, w1);
        }
        if (digits) {
            uint64_t* st = stage[wid];
            if (live) {
#pragma unroll
                for (int i = 0; i <= D; ++i) {
                    st[2 * lane * (D + 1) + i] = o0[i];
                    st[(2 * lane + 1) * (D + 1) + i] = o1[i];
                }
            }
            __syncwarp();
            const int64_t npairs = pairs - qw < 32 ? pairs - qw : 32;  // pairs of this warp in range
            const int nvec = (int)(npairs > 0 ? npairs * (D + 1) : 0);  // 16-byte vectors
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(digits + 2 * qw * (D + 1));
            for (int v = lane; v < nvec; v += 32)
                __stcs(dst + v, *reinterpret_cast<const ulonglong2*>(st + 2 * v));
            __syncwarp();
        }
        if (packed && live) __stcs(reinterpret_cast<ulonglong2*>(packed) + q, make_ulonglong2(w0, w1));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail word
        uint64_t o[D + 1], w;
        redq_word<D>(r[n - 1], p, t, invp_up, bound, corr, mode, tab, o, w);
        if (digits)
            for (int i = 0; i <= D; ++i) digits[(n - 1) * (D + 1) + i] = o[i];
        if (packed) packed[n - 1] = w;
    }
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

// Tiled pack / unpack: a block owns PK_WORDS consecutive words of one row.
// The row's uint8 segment moves between HBM and shared memory as 16-byte chunks
// (aligned to the global address, so any row offset works); each thread packs
// or unpacks PK_WPT consecutive words and writes / reads them as 16-byte vectors.
constexpr int PK_THREADS = 256, PK_WPT = 8, PK_WORDS = PK_WPT * PK_THREADS;
#ifndef QADIC_PK_ST256
#define QADIC_PK_ST256 1  // 0: the byte-wise generic path only (measurement / fallback build)
#endif

template <int k>
__global__ void __launch_bounds__(PK_THREADS) pack_rows_tile_kernel(const uint8_t* __restrict__ m, int64_t rows,
                                                                     int64_t cols, int t, int reverse,
                                                                     uint64_t* __restrict__ words,
                                                                     int64_t tiles_per_row) {
    constexpr int BUF = PK_WORDS * 8 + 32;
    __shared__ __align__(16) uint8_t buf[2][BUF];  // the next tile streams in (cp.async) during this one
    const int64_t width = (cols + k - 1) / k;
    const uint8_t* mend = m + rows * cols;
    const int64_t ntiles = rows * tiles_per_row;
    struct Geo {
        int64_t r, g0, nbytes;
        int nw, lead;
    };
    auto geo = [&](int64_t tile) {
        Geo g;
        g.r = tile / tiles_per_row;
        g.g0 = (tile % tiles_per_row) * PK_WORDS;
        g.nw = (int)(width - g.g0 < PK_WORDS ? width - g.g0 : PK_WORDS);
        const int64_t c0 = g.g0 * k;
        g.nbytes = (cols - c0 < (int64_t)g.nw * k) ? cols - c0 : (int64_t)g.nw * k;
        g.lead = (int)(reinterpret_cast<uintptr_t>(m + g.r * cols + c0) & 15);
        return g;
    };
    auto stage = [&](int64_t tile, int bi) {
        const Geo g = geo(tile);
        const uint8_t* base = m + g.r * cols + g.g0 * k - g.lead;
        const int nchunks = (int)((g.lead + g.nbytes + 15) / 16);
        for (int i = threadIdx.x; i < nchunks; i += PK_THREADS) {
            const uint8_t* ch = base + 16 * i;
            if (ch >= m && ch + 16 <= mend) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(buf[bi] + 16 * i)),
                             "l"(ch));
            } else {
                for (int q = 0; q < 16; ++q) buf[bi][16 * i + q] = (ch + q >= m && ch + q < mend) ? ch[q] : 0;
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    if ((int64_t)blockIdx.x < ntiles) stage(blockIdx.x, 0);
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int bi = it & 1;
        if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, bi ^ 1);
        else asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const Geo g = geo(tile);
        uint64_t* rowp = words + g.r * width + g.g0;
        if (QADIC_PK_ST256) {
            // Each thread packs up to 2 groups of 4 consecutive words from 4k staged bytes read
            // as k+1 aligned u32 (stride 3k/4 words across lanes: conflict-free for odd k) and
            // funnel-shifted into place -- ~5 integer ops per digit instead of a byte load with
            // bounds tests -- and writes each group with ONE 32-byte store (st.global.v4.b64,
            // sm_100: a full sector per lane, 1 KB contiguous per warp instruction; two 16-byte
            // stores per lane wrote half sectors).  Groups start at the first 32-byte-aligned
            // word of the row segment, so any row offset works; every whole group of a partial
            // tile (a row's last tile: a third of cfg4's) takes this path too, and only the
            // words before the first / after the last whole group (at most 7) are packed byte
            // by byte.
            const int whole_words = (int)(g.nbytes / k) < g.nw ? (int)(g.nbytes / k) : g.nw;
            const int woff = (int)((32 - (reinterpret_cast<uintptr_t>(rowp) & 31)) & 31) >> 3;
            const int ngroups = whole_words > woff ? (whole_words - woff) / 4 : 0;
#pragma unroll
            for (int h = 0; h < PK_WPT / 4; ++h) {
                const int gi = threadIdx.x + PK_THREADS * h;
                if (gi >= ngroups) continue;
                const int b0 = g.lead + (woff + gi * 4) * k;  // first byte of the group in buf
                const uint32_t* src = reinterpret_cast<const uint32_t*>(buf[bi] + (b0 & ~3));
                const int fs = 8 * (b0 & 3);
                uint32_t v[k + 1], x[k];
#pragma unroll
                for (int i = 0; i <= k; ++i) v[i] = src[i];
#pragma unroll
                for (int i = 0; i < k; ++i) x[i] = __funnelshift_r(v[i], v[i + 1], fs);
                uint64_t out4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint64_t wd = 0;
#pragma unroll
                    for (int j = 0; j < k; ++j) {
                        const int q = i * k + j;  // byte of the group (compile-time)
                        const uint32_t b = (x[q >> 2] >> (8 * (q & 3))) & 0xffu;
                        wd |= (uint64_t)b << ((reverse ? (k - 1 - j) : j) * t);
                    }
                    out4[i] = wd;
                }
                asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(rowp + woff + 4 * gi), "l"(out4[0]),
                             "l"(out4[1]), "l"(out4[2]), "l"(out4[3])
                             : "memory");
            }
            // ragged ends: words [0, woff) and [woff + 4 ngroups, nw)
            const int nhead = woff < g.nw ? woff : g.nw;
            const int ntail = g.nw - (ngroups ? woff + 4 * ngroups : nhead);
            if ((int)threadIdx.x < nhead + ntail) {
                const int w = (int)threadIdx.x < nhead ? (int)threadIdx.x : g.nw - ntail + ((int)threadIdx.x - nhead);
                uint64_t wd = 0;
                for (int j = 0; j < k; ++j) {
                    const int64_t off = (int64_t)w * k + j;
                    if (off < g.nbytes) wd += (uint64_t)buf[bi][g.lead + off] << ((reverse ? (k - 1 - j) : j) * t);
                }
                rowp[w] = wd;
            }
            __syncthreads();  // this buffer is refilled two tiles later
            continue;
        }
        uint64_t wv[PK_WPT];
#pragma unroll
        for (int h = 0; h < PK_WPT; ++h) {
            const int w = 2 * threadIdx.x + (h & 1) + 2 * PK_THREADS * (h >> 1);  // lane-consecutive pairs
            wv[h] = 0;
            if (w < g.nw) {
                const bool whole = (int64_t)w * k + k <= g.nbytes;
#pragma unroll
                for (int j = 0; j < k; ++j) {
                    const int64_t off = (int64_t)w * k + j;
                    if (whole || off < g.nbytes) {
                        const int e = reverse ? (k - 1 - j) : j;
                        wv[h] += (uint64_t)buf[bi][g.lead + off] << (e * t);
                    }
                }
            }
        }
#pragma unroll
        for (int h = 0; h < PK_WPT; h += 2) {
            const int w = 2 * threadIdx.x + 2 * PK_THREADS * (h >> 1);
            if (w + 1 < g.nw && (reinterpret_cast<uintptr_t>(rowp + w) & 15) == 0) {
                __stcs(reinterpret_cast<ulonglong2*>(rowp + w), make_ulonglong2(wv[h], wv[h + 1]));
            } else {
                if (w < g.nw) rowp[w] = wv[h];
                if (w + 1 < g.nw) rowp[w + 1] = wv[h + 1];
            }
        }
        __syncthreads();  // this buffer is refilled two tiles later
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <int k>
__global__ void __launch_bounds__(PK_THREADS) unpack_rows_tile_kernel(const uint64_t* __restrict__ words,
                                                                       int64_t rows, int64_t cols, int t,
                                                                       int reverse, uint8_t* __restrict__ out,
                                                                       int64_t tiles_per_row) {
    __shared__ __align__(16) uint8_t buf[PK_WORDS * 8 + 32];
    const int64_t width = (cols + k - 1) / k;
    const uint64_t mask = t >= 64 ? ~0ull : ((1ull << t) - 1);
    for (int64_t tile = blockIdx.x; tile < rows * tiles_per_row; tile += gridDim.x) {
        const int64_t r = tile / tiles_per_row, g0 = (tile % tiles_per_row) * PK_WORDS;
        const int nw = (int)(width - g0 < PK_WORDS ? width - g0 : PK_WORDS);
        const int64_t c0 = g0 * k;
        const int64_t nbytes = (cols - c0 < (int64_t)nw * k) ? cols - c0 : (int64_t)nw * k;
        uint8_t* dst = out + r * cols + c0;
        const int lead = (int)(reinterpret_cast<uintptr_t>(dst) & 15);  // buf[lead + x] <-> dst[x]
        const uint64_t* roww = words + r * width + g0;
        if (nw == PK_WORDS && nbytes == (int64_t)PK_WORDS * k && (reinterpret_cast<uintptr_t>(roww) & 15) == 0) {
            // full tile (mirror of pack's fast path): 4 consecutive words per group,
            // their 4k digit bytes assembled in k registers and written as aligned
            // u32 at buf[4k*gi]; the copy-out funnel-shifts 5 aligned u32 per 16-byte
            // chunk to the destination's alignment
            uint32_t* b32 = reinterpret_cast<uint32_t*>(buf);
#pragma unroll
            for (int h = 0; h < PK_WPT / 4; ++h) {
                const int gi = threadIdx.x + PK_THREADS * h;
                const ulonglong2 w01 = __ldcs(reinterpret_cast<const ulonglong2*>(roww + 4 * gi));
                const ulonglong2 w23 = __ldcs(reinterpret_cast<const ulonglong2*>(roww + 4 * gi + 2));
                const uint64_t wd[4] = {w01.x, w01.y, w23.x, w23.y};
                uint32_t x[k];
#pragma unroll
                for (int i = 0; i < k; ++i) x[i] = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < k; ++j) {
                        const int q = i * k + j;  // byte of the group (compile-time)
                        const uint32_t d = (uint32_t)((wd[i] >> ((reverse ? (k - 1 - j) : j) * t)) & mask) & 0xffu;
                        x[q >> 2] |= d << (8 * (q & 3));
                    }
#pragma unroll
                for (int i = 0; i < k; ++i) b32[k * gi + i] = x[i];
            }
            __syncthreads();
            const int nchunks = (lead + PK_WORDS * k + 15) / 16;
            uint8_t* base = dst - lead;
            for (int i = threadIdx.x; i < nchunks; i += PK_THREADS) {
                const int o = 16 * i - lead;  // buf offset of the chunk's first byte
                if (o >= 0 && o + 16 <= PK_WORDS * k) {
                    const uint32_t* src = b32 + (o >> 2);
                    const int fs = 8 * (o & 3);
                    uint32_t v[5];
#pragma unroll
                    for (int j = 0; j < 5; ++j) v[j] = src[j];
                    __stcs(reinterpret_cast<uint4*>(base + 16 * i),
                           make_uint4(__funnelshift_r(v[0], v[1], fs), __funnelshift_r(v[1], v[2], fs),
                                      __funnelshift_r(v[2], v[3], fs), __funnelshift_r(v[3], v[4], fs)));
                } else {
                    for (int b = 0; b < 16; ++b)
                        if (o + b >= 0 && o + b < PK_WORDS * k) base[16 * i + b] = buf[o + b];
                }
            }
            __syncthreads();
            continue;
        }
        uint64_t wv[PK_WPT];
#pragma unroll
        for (int h = 0; h < PK_WPT; h += 2) {  // lane-consecutive 16-byte pairs
            const int w = 2 * threadIdx.x + 2 * PK_THREADS * (h >> 1);
            if (w + 1 < nw && (reinterpret_cast<uintptr_t>(roww + w) & 15) == 0) {
                const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(roww + w));
                wv[h] = x.x;
                wv[h + 1] = x.y;
            } else {
                wv[h] = w < nw ? roww[w] : 0;
                wv[h + 1] = w + 1 < nw ? roww[w + 1] : 0;
            }
        }
#pragma unroll
        for (int h = 0; h < PK_WPT; ++h) {
            const int w = 2 * threadIdx.x + (h & 1) + 2 * PK_THREADS * (h >> 1);
            if (w < nw) {
                const bool whole = (int64_t)w * k + k <= nbytes;
#pragma unroll
                for (int j = 0; j < k; ++j) {
                    const int64_t off = (int64_t)w * k + j;
                    const int e = reverse ? (k - 1 - j) : j;
                    if (whole || off < nbytes) buf[lead + off] = (uint8_t)((wv[h] >> (e * t)) & mask);
                }
            }
        }
        __syncthreads();
        const int nchunks = (int)((lead + nbytes + 15) / 16);
        uint8_t* base = dst - lead;
        for (int i = threadIdx.x; i < nchunks; i += PK_THREADS) {
            const int lo = 16 * i, hi = lo + 16;
            if (lo >= lead && hi <= lead + nbytes) {
                __stcs(reinterpret_cast<uint4*>(base + lo), *reinterpret_cast<const uint4*>(buf + lo));
            } else {
                for (int b = lo; b < hi; ++b)
                    if (b >= lead && b < lead + nbytes) base[b] = buf[b];
            }
        }
        __syncthreads();
    }
}

// one wave of resident blocks (grid-stride over the tiles)
template <typename F>
static int grid_for_tiles(F kern, int64_t tiles) {
    const int sms = num_sms_cached();
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PK_THREADS, 0);
    static const int blocks_env = getenv("QADIC_PK_BLOCKS") ? atoi(getenv("QADIC_PK_BLOCKS")) : 0;  // measurement switch
    if (blocks_env > 0 && blocks_env < occ) occ = blocks_env;
    if (occ < 1) occ = 1;
    return (int)std::min<int64_t>(tiles, (int64_t)sms * occ);
}

template <int K>
static void launch_pack_tiles(const uint8_t* m, int64_t rows, int64_t cols, int t, int reverse, uint64_t* words,
                              cudaStream_t s) {
    const int64_t width = (cols + K - 1) / K, tpr = (width + PK_WORDS - 1) / PK_WORDS;
    pack_rows_tile_kernel<K><<<grid_for_tiles(pack_rows_tile_kernel<K>, rows * tpr), PK_THREADS, 0, s>>>(
        m, rows, cols, t, reverse, words, tpr);
}

template <int K>
static void launch_unpack_tiles(const uint64_t* words, int64_t rows, int64_t cols, int t, int reverse, uint8_t* out,
                                cudaStream_t s) {
    const int64_t width = (cols + K - 1) / K, tpr = (width + PK_WORDS - 1) / PK_WORDS;
    unpack_rows_tile_kernel<K><<<grid_for_tiles(unpack_rows_tile_kernel<K>, rows * tpr), PK_THREADS, 0, s>>>(
        words, rows, cols, t, reverse, out, tpr);
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
    if (tc_u64_ok(m, k, n, a) && !(getenv("QADIC_U64_SIMT") && atoi(getenv("QADIC_U64_SIMT")) != 0))
        return tc_matmul_u64(a, b, c, m, k, n, s);  // INT8 tensor cores on byte planes
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
    cudaStream_t s = (cudaStream_t)stream;
    const bool aligned = ((uintptr_t)r % 16 == 0) && (!digits || (uintptr_t)digits % 16 == 0) &&
                         (!packed || (uintptr_t)packed % 16 == 0);
    if (aligned && d >= 1 && d <= 6 && p < (1ll << 31)) {  // digits in [0, p) fit the 32-bit arithmetic
        const int sms = num_sms_cached();
        const int64_t pairs = (n + 1) / 2;
        const double inv = host_reciprocal_up(p), bnd = host_case2_bound();
        const uint64_t pp = (uint64_t)p;
        // one wave of 4 blocks per SM (grid-stride loop).  Measured at 2^26 words, d = 2 (cfg3's
        // accumulators), blocks per SM -> ms: 1 0.700, 2 0.443, 3 0.384, 4 0.364, 5 0.400,
        // 6 0.439, 8 (a partial second round) 0.378: beyond 4 the extra concurrent write
        // streams cost more DRAM efficiency than their latency hiding returns.
        // QADIC_RQ_BLOCKS=n: n blocks per SM (measurement switch)
        static const int blocks_env = getenv("QADIC_RQ_BLOCKS") ? atoi(getenv("QADIC_RQ_BLOCKS")) : 0;
        switch (d) {
#define QADIC_RQ(DD)                                                                                           \
    case DD: {                                                                                                 \
        int occ = 0;                                                                                           \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, redq_vec_kernel<DD>, RQ_THREADS, 0);               \
        if (occ > 4) occ = 4;                                                                                  \
        if (blocks_env > 0) occ = blocks_env;                                                                  \
        if (occ < 1) occ = 1;                                                                                  \
        const int grid = (int)std::min<int64_t>((pairs + RQ_THREADS - 1) / RQ_THREADS, (int64_t)sms * occ);    \
        redq_vec_kernel<DD><<<grid, RQ_THREADS, 0, s>>>(r, n, pp, t, inv, bnd, corr, mode, digits, packed);     \
        break;                                                                                                 \
    }
            QADIC_RQ(1) QADIC_RQ(2) QADIC_RQ(3) QADIC_RQ(4) QADIC_RQ(5) QADIC_RQ(6)
#undef QADIC_RQ
        }
        return check_launch(what, 1);
    }
    redq_words_kernel<<<blocks_for(n, 256), 256, 0, s>>>(r, n, (uint64_t)p, t, d, host_reciprocal_up(p),
                                                         host_case2_bound(), corr, mode, digits, packed);
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
    const int64_t width = (cols + k - 1) / k, total = rows * width;
    if (total == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (k <= 8) {
        switch (k) {
            case 1: launch_pack_tiles<1>(m, rows, cols, t, reverse, words, s); break;
            case 2: launch_pack_tiles<2>(m, rows, cols, t, reverse, words, s); break;
            case 3: launch_pack_tiles<3>(m, rows, cols, t, reverse, words, s); break;
            case 4: launch_pack_tiles<4>(m, rows, cols, t, reverse, words, s); break;
            case 5: launch_pack_tiles<5>(m, rows, cols, t, reverse, words, s); break;
            case 6: launch_pack_tiles<6>(m, rows, cols, t, reverse, words, s); break;
            case 7: launch_pack_tiles<7>(m, rows, cols, t, reverse, words, s); break;
            default: launch_pack_tiles<8>(m, rows, cols, t, reverse, words, s); break;
        }
    } else {
        pack_rows_kernel<<<blocks_for(total, 256), 256, 0, s>>>(m, rows, cols, k, t, reverse, words);
    }
    return check_launch("pack_rows_u8", 1);
}

int qadic_unpack_rows_u8(const uint64_t* words, int64_t rows, int64_t cols, int32_t k, int32_t t,
                         int32_t reverse, uint8_t* out, void* stream) {
    QADIC_REQUIRE(rows >= 0 && cols >= 0 && k >= 1 && t >= 1 && t <= 8 * 8, QADIC_ERR_VALUE, "bad unpack geometry");
    if (rows * cols == 0) return QADIC_OK;
    if (k <= 8) {
        cudaStream_t s = (cudaStream_t)stream;
        switch (k) {
            case 1: launch_unpack_tiles<1>(words, rows, cols, t, reverse, out, s); break;
            case 2: launch_unpack_tiles<2>(words, rows, cols, t, reverse, out, s); break;
            case 3: launch_unpack_tiles<3>(words, rows, cols, t, reverse, out, s); break;
            case 4: launch_unpack_tiles<4>(words, rows, cols, t, reverse, out, s); break;
            case 5: launch_unpack_tiles<5>(words, rows, cols, t, reverse, out, s); break;
            case 6: launch_unpack_tiles<6>(words, rows, cols, t, reverse, out, s); break;
            case 7: launch_unpack_tiles<7>(words, rows, cols, t, reverse, out, s); break;
            default: launch_unpack_tiles<8>(words, rows, cols, t, reverse, out, s); break;
        }
        return check_launch("unpack_rows_u8", 1);
    }
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
