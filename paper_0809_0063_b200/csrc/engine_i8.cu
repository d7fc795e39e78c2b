// Engine I8: exact GF(p^k) / F_p matrix products on the 5th-gen tensor cores.
//
// Coefficient-plane formulation of the paper's delayed reduction
// (PAPER.md:216-223 applied to GFqField.matmul, src/gfext.py:311-345, and
// cmm.right_cmm, src/cmm.py:244-276):
//
//   C[m, (j,l)] = sum_{kk,i} A[m, (kk,i)] * Bx[(j,l), (kk,i)]   (mod p)
//   Bx[(j,l), (kk,i)] = coefficient l of  X^i * b[kk,j](X)  mod (f, p)
//
// i.e. every B entry is expanded once into its k x k multiplication matrix
// over F_p with the X^k fold already applied (the "companion" rows
// X^i mod f, src/gfext.py:200-205, reduced into [0, p)).  A needs no
// transformation: the row-major uint8[M, K, k] coefficient tensor IS the
// K-major A operand.  All products are nonnegative 8-bit integers and the
// int32 TMEM accumulator holds the whole delayed sum exactly while
// K*k*(p-1)^2 < 2^31 (cfg3: 65,536; cfg5: 884,736), so the epilogue is a
// single mod p per output coefficient.
//
// GEMM: persistent, warp-specialised tcgen05 kernel.
//   warp 0  TMA producer (128B-swizzled K-major tiles, 4-stage mbarrier ring)
//   warp 1  UMMA issuer  (tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32)
//   warp 2  TMEM allocator (512 columns = 2 accumulator buffers of 256)
//   warps 4-7 epilogue   (tcgen05.ld -> mod p -> uint8 stores), overlapping
//            the next tile's MMAs through the double-buffered accumulator.
#include <cuda.h>

#include "qadic_common.cuh"
#include "qadic_internal.h"
#include "sm100_ptx.cuh"

namespace qadic {

int make_field_const(const qadic_field_desc* d, FieldConst* f);

namespace i8 {

constexpr int BM = 128, BN = 256, BK = 128;  // BK in bytes (= int8 elements)
constexpr int UMMA_K = 32;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int ACC_COLS = BN;           // one fp32/s32 column per output column
constexpr int TMEM_COLS = 2 * ACC_COLS;
constexpr int THREADS = 256;
constexpr int GROUP_M = 16;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
    int64_t M, N, Kb;       // output rows, output cols, inner bytes
    int64_t ldc;            // output row pitch (bytes)
    uint32_t p;
    uint64_t magic64;
    int m_tiles, n_tiles, num_kb;
    uint8_t* c;
};

__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int& mt, int& nt) {
    const int per_group = GROUP_M * n_tiles;
    const int group = tile / per_group;
    const int first_m = group * GROUP_M;
    const int gm = min(m_tiles - first_m, GROUP_M);
    const int r = tile % per_group;
    mt = first_m + r % gm;
    nt = r / gm;
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_u8_modp_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        Params prm) {
    using namespace sm100;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tmem_full = empty_bar + STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int num_tiles = prm.m_tiles * prm.n_tiles;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmap_a);
        tma_prefetch(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 128);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int mt, nt;
                tile_coords(tile, prm.m_tiles, prm.n_tiles, mt, nt);
                for (int kb = 0; kb < prm.num_kb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    uint8_t* sb = sa + A_BYTES;
                    mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
                    tma_load_2d(sa, &tmap_a, &full_bar[stage], kb * BK, mt * BM);
                    tma_load_2d(sb, &tmap_b, &full_bar[stage], kb * BK, nt * BN);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== UMMA issuer =====
        constexpr uint32_t idesc = idesc_u8_s32(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + acc * ACC_COLS;
            for (int kb = 0; kb < prm.num_kb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sa = smem_addr(smem + stage * STAGE_BYTES);
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        umma_i8(tmem_d, smem_desc_k_sw128(sa + k * UMMA_K), smem_desc_k_sw128(sb + k * UMMA_K),
                                idesc, (kb | k) != 0);
                    }
                    umma_commit(&empty_bar[stage]);
                    if (kb == prm.num_kb - 1) umma_commit(&tmem_full[acc]);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> mod p -> uint8 =====
        const int ew = warp - 4;  // TMEM lane quarter this warp may access
        int local = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            int mt, nt;
            tile_coords(tile, prm.m_tiles, prm.n_tiles, mt, nt);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tmem_full[acc], acc_phase);
            tc_fence_after();
            const int64_t row = (int64_t)mt * BM + ew * 32 + lane;
            const bool row_ok = row < prm.M;
            uint8_t* crow = prm.c + row * prm.ldc;
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * ACC_COLS + ch * 32, v);
                tmem_ld_wait();
                const int64_t col0 = (int64_t)nt * BN + ch * 32;
                if (!row_ok || col0 >= prm.N) continue;
                uint32_t w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    w[q] = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) w[q] |= mod_u32(v[4 * q + e], prm.p, prm.magic64) << (8 * e);
                }
                if (col0 + 32 <= prm.N && ((reinterpret_cast<uintptr_t>(crow + col0) & 15) == 0)) {
                    uint4* dst = reinterpret_cast<uint4*>(crow + col0);
                    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                } else {
                    for (int e = 0; e < 32 && col0 + e < prm.N; ++e) crow[col0 + e] = (uint8_t)(w[e / 4] >> (8 * (e % 4)));
                }
            }
            tc_fence_before();
            mbar_arrive(&tmem_empty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// B expansion: Bx[(j,l), kk*k + i] = coeff_l( X^i * b[kk,j] mod f ) mod p.
// For k = 1 with xpow = {{1}} this is a plain transpose (right_cmm's B).
// 64 x 64 (kk, j) tile through shared memory: coalesced reads of b rows,
// coalesced 4-byte writes of Bx rows.
// ---------------------------------------------------------------------------
constexpr int EX_T = 64;

__global__ void __launch_bounds__(256) expand_b_kernel(const uint8_t* __restrict__ b, int64_t K, int64_t N,
                                                       FieldConst f, uint8_t* __restrict__ bx, int64_t ldb) {
    __shared__ uint8_t sb[EX_T][EX_T * kMaxK + 4];
    const int k = (int)f.k;
    const int64_t kk0 = (int64_t)blockIdx.x * EX_T, j0 = (int64_t)blockIdx.y * EX_T;
    const int rowbytes = EX_T * k;
    for (int i = threadIdx.x; i < EX_T * rowbytes; i += blockDim.x) {
        const int r = i / rowbytes, c = i % rowbytes;
        const int64_t gk = kk0 + r, gj = j0 + c / k;
        sb[r][c] = (gk < K && gj < N) ? b[gk * N * k + j0 * k + c] : 0;
    }
    __syncthreads();
    // output rows (j, l) for j in tile; columns kk*k + i for kk in tile
    const int words_per_row = rowbytes / 4;  // rowbytes = 64k, divisible by 4
    const int64_t colbase = kk0 * k;
    for (int w = threadIdx.x; w < EX_T * k * words_per_row; w += blockDim.x) {
        const int orow = w / words_per_row, wq = w % words_per_row;
        const int jl = orow / k, l = orow % k;
        const int64_t gj = j0 + jl;
        if (gj >= N) continue;
        uint32_t word = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = wq * 4 + e;        // byte within the output row segment
            const int kl = c / k, i = c % k;  // kk (local) and X^i
            uint32_t acc = 0;
            for (int s = 0; s < k; ++s) acc += (uint32_t)sb[kl][jl * k + s] * f.xpow[s + i][l];
            word |= mod_small(acc, f.p, f.magic) << (8 * e);
        }
        const int64_t col = colbase + wq * 4;
        uint8_t* dst = bx + (gj * k + l) * ldb + col;
        if (col + 4 <= ldb) *reinterpret_cast<uint32_t*>(dst) = word;
        else
            for (int e = 0; e < 4 && col + e < ldb; ++e) dst[e] = (uint8_t)(word >> (8 * e));
    }
}

// Table-driven expansion (fields with p^K <= XT_CODES): every element code
// maps to its K x K block, staged in shared memory as K rows of K bytes
// (T[code*K + l] = bytes i=0..K-1 of output row l).  Tile = 64 kk x 128 j:
// b rows are read with 16-byte loads, codes are stored j-major so that an
// output row segment of 16 consecutive kk (16K bytes, K 16-byte stores) is
// one contiguous smem read.  Grid-stride over tiles amortises the table.
constexpr int XT_KK = 64, XT_J = 64, XT_CODES = 1024;

template <int K>
__global__ void __launch_bounds__(256) expand_b_table_kernel(const uint8_t* __restrict__ b, int64_t Kd, int64_t N,
                                                             FieldConst f, uint8_t* __restrict__ bx, int64_t ldb,
                                                             int tiles_kk, int tiles_j) {
    __shared__ uint32_t tab[XT_CODES * K];
    __shared__ __align__(16) uint8_t raw[XT_KK][XT_J * K + 16];
    __shared__ __align__(16) uint16_t code[XT_J][XT_KK + 8];
    const uint32_t p = f.p;
    int ncodes = 1;
    for (int s = 0; s < K; ++s) ncodes *= (int)p;
    // block table: T[c, l] packs coeff_l(X^i * c(X) mod f), i = 0..K-1
    for (int e = threadIdx.x; e < ncodes * K; e += blockDim.x) {
        const int c = e / K, l = e % K;
        uint32_t dig[K];
        int r = c;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            dig[s] = (uint32_t)(r % (int)p);
            r /= (int)p;
        }
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            uint32_t acc = 0;
#pragma unroll
            for (int s = 0; s < K; ++s) acc += dig[s] * f.xpow[s + i][l];
            w |= mod_small(acc, p, f.magic) << (8 * i);
        }
        tab[e] = w;
    }
    const bool vec_rows = ((N * K) % 16 == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t kk0 = (tile % tiles_kk) * XT_KK, j0 = (tile / tiles_kk) * XT_J;
        __syncthreads();  // previous tile's smem fully consumed (and table ready)
        // phase 1: raw coefficient tile
        constexpr int ROWB = XT_J * K;
        if (vec_rows && j0 + XT_J <= N) {
            for (int i = threadIdx.x; i < XT_KK * (ROWB / 16); i += blockDim.x) {
                const int r = i / (ROWB / 16), q = i % (ROWB / 16);
                const int64_t gk = kk0 + r;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (gk < Kd) v = __ldg(reinterpret_cast<const uint4*>(b + gk * N * K + j0 * K) + q);
                *reinterpret_cast<uint4*>(&raw[r][q * 16]) = v;
            }
        } else {
            for (int i = threadIdx.x; i < XT_KK * ROWB; i += blockDim.x) {
                const int r = i / ROWB, c = i % ROWB;
                const int64_t gk = kk0 + r, gj = j0 + c / K;
                raw[r][c] = (gk < Kd && gj < N) ? b[gk * N * K + j0 * K + c] : 0;
            }
        }
        __syncthreads();
        // phase 2: element codes, transposed to j-major
        for (int i = threadIdx.x; i < XT_KK * XT_J; i += blockDim.x) {
            const int r = i / XT_J, jl = i % XT_J;
            uint32_t cd = 0;
#pragma unroll
            for (int s = K - 1; s >= 0; --s) cd = cd * p + raw[r][jl * K + s];
            code[jl][r] = (uint16_t)cd;
        }
        __syncthreads();
        // phase 3: output rows (j, l), 16 kk per work item -> K 16-byte stores
        for (int i = threadIdx.x; i < XT_J * K * (XT_KK / 16); i += blockDim.x) {
            const int ch = i % (XT_KK / 16), row = i / (XT_KK / 16);
            const int jl = row / K, l = row % K;
            const int64_t gj = j0 + jl;
            if (gj >= N) continue;
            uint32_t w[4 * K];
#pragma unroll
            for (int q = 0; q < 4 * K; ++q) w[q] = 0;
            const uint16_t* cr = &code[jl][ch * 16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const uint32_t v = tab[cr[e] * K + l];
#pragma unroll
                for (int ii = 0; ii < K; ++ii) {
                    const int pos = e * K + ii;
                    w[pos / 4] |= ((v >> (8 * ii)) & 0xFF) << (8 * (pos % 4));
                }
            }
            const int64_t col = (kk0 + ch * 16) * K;
            uint8_t* dst = bx + (gj * K + l) * ldb + col;
            if (col + 16 * K <= ldb) {
#pragma unroll
                for (int q = 0; q < K; ++q)
                    reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            } else {
                for (int e = 0; e < 16 * K && col + e < ldb; ++e) dst[e] = (uint8_t)(w[e / 4] >> (8 * (e % 4)));
            }
        }
    }
}

// rows of width `width` bytes copied into a pitched, zero-padded buffer
__global__ void pad_rows_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t width, uint8_t* __restrict__ dst,
                                int64_t ld) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * ld) return;
    const int64_t r = i / ld, c = i % ld;
    dst[i] = c < width ? src[r * width + c] : 0;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

static int make_tmap(CUtensorMap* map, const void* base, int64_t inner_bytes, int64_t rows, int64_t ld,
                     uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    QADIC_REQUIRE(fn != nullptr, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)inner_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QADIC_REQUIRE(r == CUDA_SUCCESS, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return QADIC_OK;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct Layout {
    int64_t Kb;      // inner bytes (K * k)
    int64_t lda, ldb;
    bool pad_a;
    size_t bx_bytes, a_bytes;
};

static Layout plan(const uint8_t* a, int64_t m, int64_t kdim, int64_t n, int k) {
    Layout L;
    L.Kb = kdim * k;
    L.ldb = round_up(L.Kb, 16);
    L.pad_a = (L.Kb % 16 != 0) || ((reinterpret_cast<uintptr_t>(a) & 15) != 0);
    L.lda = L.pad_a ? L.ldb : L.Kb;
    L.bx_bytes = (size_t)round_up(n * k * L.ldb, 1024);
    L.a_bytes = L.pad_a ? (size_t)round_up(m * L.lda, 1024) : 0;
    return L;
}

// C[m, n*k] = A[m, Kb] (x) expand(B)  (mod p)
static int run(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
               void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    const int k = (int)f.k;
    Layout L = plan(a, m, kdim, n, k);
    QADIC_REQUIRE(ws != nullptr && ws_bytes >= L.bx_bytes + L.a_bytes, QADIC_ERR_VALUE,
                  "workspace too small (%zu < %zu)", ws_bytes, L.bx_bytes + L.a_bytes);
    uint8_t* bx = static_cast<uint8_t*>(ws);
    const uint8_t* a_op = a;
    if (L.pad_a) {
        uint8_t* ap = bx + L.bx_bytes;
        const int64_t tot = m * L.lda;
        QADIC_TIMED("i8 pad A", s, pad_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, m, L.Kb, ap, L.lda));
        int rc = check_launch("i8 pad A");
        if (rc) return rc;
        a_op = ap;
    }
    {
        int ncodes = 1;
        for (int s2 = 0; s2 < k; ++s2) ncodes *= (int)f.p;
        if (ncodes <= XT_CODES) {
            const int tk = (int)((kdim + XT_KK - 1) / XT_KK), tj = (int)((n + XT_J - 1) / XT_J);
            const int64_t tiles = (int64_t)tk * tj;
            const int grid = (int)(tiles < 4 * num_sms() ? tiles : 4 * num_sms());
            switch (k) {
                case 1: QADIC_TIMED("i8 expand B", s, expand_b_table_kernel<1><<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb, tk, tj)); break;
                case 2: QADIC_TIMED("i8 expand B", s, expand_b_table_kernel<2><<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb, tk, tj)); break;
                case 3: QADIC_TIMED("i8 expand B", s, expand_b_table_kernel<3><<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb, tk, tj)); break;
                default: QADIC_TIMED("i8 expand B", s, expand_b_table_kernel<4><<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb, tk, tj)); break;
            }
        } else {
            dim3 grid((unsigned)((kdim + EX_T - 1) / EX_T), (unsigned)((n + EX_T - 1) / EX_T));
            QADIC_REQUIRE(grid.y <= 65535, QADIC_ERR_UNSUPPORTED, "n too large");
            QADIC_TIMED("i8 expand B", s, expand_b_kernel<<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb));
        }
        int rc = check_launch("i8 expand B");
        if (rc) return rc;
    }
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, a_op, L.Kb, m, L.lda, BM);
    if (rc) return rc;
    rc = make_tmap(&tb, bx, L.Kb, n * k, L.ldb, BN);
    if (rc) return rc;
    Params prm;
    prm.M = m;
    prm.N = n * k;
    prm.Kb = L.Kb;
    prm.ldc = n * k;
    prm.p = f.p;
    prm.magic64 = wide_magic(f.p);
    prm.m_tiles = (int)((m + BM - 1) / BM);
    prm.n_tiles = (int)((prm.N + BN - 1) / BN);
    prm.num_kb = (int)((L.Kb + BK - 1) / BK);
    prm.c = c;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_u8_modp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
        attr = true;
    }
    const int tiles = prm.m_tiles * prm.n_tiles;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    QADIC_TIMED("i8 gemm", s, gemm_u8_modp_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(ta, tb, prm));
    return check_launch("i8 gemm");
}

}  // namespace i8

size_t i8_workspace(int64_t m, int64_t kdim, int64_t n, int k) {
    // worst case: A needs padding
    const int64_t Kb = kdim * k;
    const int64_t ld = i8::round_up(Kb, 16);
    return (size_t)i8::round_up(n * k * ld, 1024) + (size_t)i8::round_up(m * ld, 1024);
}

int i8_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                 void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    QADIC_REQUIRE((__int128)kdim * f.k * (f.p - 1) * (f.p - 1) < ((__int128)1 << 31), QADIC_ERR_PARAMS,
                  "inner dimension %lld overflows the int32 plane accumulator", (long long)kdim);
    return i8::run(f, a, b, m, kdim, n, ws, ws_bytes, c, s);
}

int i8_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                 size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    QADIC_REQUIRE((__int128)kdim * (p - 1) * (p - 1) < ((__int128)1 << 31), QADIC_ERR_PARAMS,
                  "inner dimension %lld overflows the int32 accumulator", (long long)kdim);
    FieldConst f = {};
    f.p = p;
    f.k = 1;
    f.t = 8;
    f.magic = small_magic(p);
    f.xpow[0][0] = 1;
    return i8::run(f, a, b, m, kdim, n, ws, ws_bytes, c, s);
}

}  // namespace qadic
