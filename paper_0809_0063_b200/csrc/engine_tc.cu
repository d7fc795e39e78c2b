// Tensor-core engines (tcgen05) for exact GF(p^k) / F_p matrix products.
//
// Coefficient-plane formulation of the paper's delayed reduction
// (PAPER.md:216-223 applied to GFqField.matmul, src/gfext.py:311-345, and
// cmm.right_cmm, src/cmm.py:244-276).  Two decompositions:
//
// * Expanded form (I8, FP4):
//     C[m, (j,l)] = sum_{kk,i} A[m, (kk,i)] * Bx[(j,l), (kk,i)]   (mod p)
//     Bx[(j,l), (kk,i)] = coefficient l of  X^i * b[kk,j](X)  mod (f, p)
//   every B entry expanded once into its k x k multiplication matrix over F_p
//   with the X^k fold applied (rows X^i mod f, src/gfext.py:200-205): one GEMM
//   of M x (N k) x (K k).
// * Evaluation planes (FP4K, the default for p <= 7): S = 2k-1 Toom-Cook points
//   over F_p (Karatsuba k(k+1)/2 when 2k-1 > p+1); plane s of A and of B is an
//   F_p-linear combination of the coefficients (a plane-table lookup per element
//   code), the S plane products are independent F_p GEMMs of M x N x K, and
//   C_l = sum_s W[l][s] D_s mod p recombines them (separate SWAR pass, or in the
//   GEMM epilogue for S <= 3).
//
// The delayed sum is exact in the accumulator, so no intermediate reduction:
//   KIND_I8  tcgen05.mma.kind::i8, residues 0..p-1, s32 accumulate; exact while
//            K*k*(p-1)^2 < 2^31 (any p <= 127).
//   KIND_F4  tcgen05.mma.kind::mxf4.block_scale (E2M1, two per byte) on residue
//            representatives that E2M1 holds exactly (half-integer codes under
//            2^1 block scales, see e2m1_lut); the fp32 accumulator is exact while
//            K * max|v|^2 < 2^24.  Twice the int8 MMA rate, half the bytes.
//
// Kernel roles (gemm_modp_kernel): warp 0 TMA producer (128B-swizzled K-major
// tiles, up to 8-stage mbarrier ring), warp 1 single-thread MMA issuer (M=256
// over a CTA pair with cta_group::2, N=240), warp 2 TMEM allocator, warps 4-7
// (4-11 when fused) epilogue (tcgen05.ld -> mod p -> residues) overlapping the
// next tile through two TMEM accumulators.
#include <cuda.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <utility>

#include "qadic_common.cuh"
#include "qadic_internal.h"
#include "sm100_ptx.cuh"

namespace qadic {

int make_field_const(const qadic_field_desc* d, FieldConst* f);

namespace tc {

enum Kind { KIND_I8 = 0, KIND_F4 = 1 };

constexpr int BM = 128, BK = 128;  // BK in bytes per stage (128 int8 / 256 fp4 elements)
constexpr int STAGES = 4;
constexpr int THREADS = 256;        // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-7 epilogue
constexpr int THREADS_FUSED = 384;  // fused combine: 8 epilogue warps (4-11)
constexpr int GROUP_M = 16;
#ifndef QADIC_MAX_STAGES
#define QADIC_MAX_STAGES 8
#endif

template <int KIND>
struct Cfg;
template <>
struct Cfg<KIND_I8> {
    static constexpr int BN = 256;
    static constexpr int SF_COL = -1;  // no scale factors
};
template <>
struct Cfg<KIND_F4> {
    static constexpr int BN = 240;      // 2 x 240 accumulator columns + 32 scale-factor columns = 512
    static constexpr int SF_COL = 480;
};

// Geometry per operand kind and CTA grouping.  PAIR = cta_group::2: two CTAs
// of a cluster share one M=256 MMA; each loads its own 128 A rows and half of
// the BN B rows, so the per-SM operand traffic (TMA writes + MMA reads of
// shared memory) drops by a third at the same MMA rate.
// FUSE_K > 0: the epilogue applies the plane combination C_l = sum_s W[l][s] D_s
// itself, accumulating the S plane results of one output tile in registers
// (8 epilogue warps, byte lanes).
// MC: two CTA pairs per cluster (4 CTAs) work on vertically adjacent tiles of
// the same B columns; each pair TMA-loads half of the B tile and multicasts it
// to both pairs, so L2 -> SM operand traffic drops by a quarter.  The B slot is
// then 2 x 64 rows (slices land at 8-row swizzle-atom boundaries).
template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
struct Geo {
    static constexpr int BN = Cfg<KIND>::BN;
    static constexpr int B_ROWS = PAIR ? BN / 2 : BN;  // B rows this CTA's MMA half reads
    static constexpr int B_BOX = MC ? 64 : B_ROWS;      // rows per B TMA box
    static constexpr int B_SLOT = MC ? 2 * B_BOX : B_ROWS;
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = B_SLOT * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int ACC_BYTES = 0;
    // as many stages as 227 KB of shared memory holds (deeper prefetch hides
    // the L2 misses at tile boundaries of short-K plane products)
    static constexpr int FIT = (232448 - 1280 - ACC_BYTES) / STAGE_BYTES;
    static constexpr int STAGES_N = PAIR ? (FIT > QADIC_MAX_STAGES ? QADIC_MAX_STAGES : FIT) : STAGES;
    static constexpr size_t SMEM = (size_t)STAGES_N * STAGE_BYTES + ACC_BYTES + 1024 + 256;
    static constexpr int TILE_M = PAIR ? 2 * BM : BM;
};

// SWAR variant (S*(p-1)^2 < 256): every byte lane of the weighted plane sum
// stays below 256, so the sum, the reduction mod p and the interleave into
// coefficient-minor order all run on 4 lanes per instruction:
//   x mod p = x - p * floor(x / p),  floor(x / p) = (x * lm) >> ls per 16-bit lane
//   (host-checked exact for every lane value that can occur), then PRMT places
//   the K coefficient words of 4 columns into K output words.
struct LaneDiv {
    uint32_t m, sh, qmask;  // qmask: per 16-bit lane, bits that can hold the quotient
};

__device__ __forceinline__ uint32_t lanes_mod_div(uint32_t x, uint32_t p, LaneDiv d) {
    const uint32_t e = x & 0x00FF00FFu, o = (x >> 8) & 0x00FF00FFu;
    const uint32_t qe = ((e * d.m) >> d.sh) & d.qmask, qo = ((o * d.m) >> d.sh) & d.qmask;
    return x - (qe | (qo << 8)) * p;
}

struct Params {
    int64_t M, N;        // output rows / cols of one plane (cols = n * k for the expanded form)
    int64_t ldc;         // output row pitch (bytes)
    int64_t c_plane;     // output plane stride (bytes)
    uint32_t p;
    uint32_t offset;     // multiple of p added before the unsigned mod (centred kinds)
    uint64_t magic64;
    int epi_mod64;       // QADIC_EPI_MOD64=1: the unfused epilogue keeps the 64-bit form (measurement switch)
    uint32_t magic32;    // nonzero: accumulator + offset < 2^32 / p, so x mod p = x - p * umulhi(x, magic32) (2 instructions)
    int m_tiles, n_tiles, num_kb;
    int n_full;          // column tiles of full width BN (n_tiles - 1 when N % BN != 0)
    int planes;          // independent plane products, stacked along the A / B rows
    int nibble_out;      // 0: uint8 residues; 1: residues packed two per byte
    uint8_t* c;
    uint8_t W[4][8];     // FUSE_K: combination weights (mod p), C_l = sum_s W[l][s] D_s
    uint32_t sf;         // 4 x UE8M0 block scale bytes (0x7F7F7F7F: every scale 2^0)
    uint32_t lane_m, lane_sh, lane_qmask;  // FUSE_K: per-16-bit-lane division by p (LaneDiv)
    int group_m;                           // FUSE_K: m tiles per raster group
    int diag_noload;     // diagnostics only (QADIC_DIAG_NOLOAD): stages after the first pass skip the TMA
    // exact uint64 GEMM through byte planes (KIND_I8): C64 = (acc64 ? C64 : 0) + (u32 D << shift)
    uint64_t* c64;
    int shift, acc64;
    // segmented K (uint64 byte planes): K'' block kb belongs to segment kb / seg_kpb,
    // i = seg_i_lo + segment; A is read at byte offset i * seg_kp + (kb % seg_kpb) * BK
    // of its row, B at row offset (seg_s - i) * N.  seg_kpb = 0: contiguous K.
    int seg_kpb, seg_i_lo, seg_s, seg_kp;
    // uint64 byte planes with the significant-byte counts resolved on the device:
    // seg_dev[0] / [1] = bytes of A / B that can be nonzero; the launch derives its
    // shift's segments (seg_i_lo, num_kb) from them and exits when it has none
    const int* seg_dev;
    // plane_inner: all byte shifts of one output tile run back to back on one CTA
    // (pair) in a single launch -- shift s = plane index, its segments
    // seg_lo[s] .. seg_lo[s] + seg_cnt[s] - 1, C accumulated in program order
    int plane_inner;
    int seg_lo[8], seg_cnt[8];
    // column-tile range of this launch: tiles n_tile0 .. n_tile0 + n_tiles - 1
    int n_tile0;
    // launched as the programmatic dependent of a concurrent GEMM launch: wait for
    // that grid to complete before exiting, so stream order still covers both
    int pdl_tail;
    // uint8 epilogue: store column n of row m at c[n * ldc + m + n * diag_shift] (0: row-major)
    int64_t diag_shift;
    // A operand as 16 phase-shifted copies read through one 4-D tensor map {K bytes,
    // rows at a 16-byte stride, phase, plane} (the Toeplitz operand of the long-product
    // GEMM without materialising it): a 128-row tile is one box of 16 phases x 8 rows,
    // smem row 8 phi + r holding GEMM row 16 r + phi of the tile; the epilogue maps TMEM lanes
    // back and stores GEMM row x at M - 1 - x (rows are the Toeplitz rows reversed)
    int a_phase;
    // Convolution mode (the batched long products, conv_tc): a work unit is the output
    // block y = y0 + i + v TL (i < 128: TMEM lane, v: column) of one pair; its K loop runs
    // over the Toeplitz row blocks w (rows y0 + w TL .. +127, A = the phase map at row
    // (conv_x0 - y0 - w TL - 127) / 16) against the b blocks shifted by w (B = a 3-D map
    // {TL, V, batch} at row v0 - w: out-of-range blocks load as zeros), so the overlap-add
    // of the block products happens in the TMEM accumulator and the epilogue writes the
    // final coefficients mod p.  m tile = y0 / 128, planes = pairs.
    int conv, conv_tl, conv_x0, conv_kpw;  // kpw: K blocks per Toeplitz row block (TL / BK)
    int conv_brows;                        // rows of the B box (the column tile, <= BN)
    int conv_tn;                           // column tile width (<= BN, a multiple of 16)
    // split-K over the Toeplitz row blocks (small batches): m tile = split * conv_rows + y0
    // tile; split j runs row blocks [j conv_wc, min(conv_w, (j+1) conv_wc)) and, when
    // conv_part is set, writes raw int32 sums to conv_part[j][plane][y] (y < conv_ytot)
    // for conv_reduce_kernel
    int conv_rows, conv_wc, conv_w;
    int32_t* conv_part;
    int64_t conv_ytot;
    int64_t conv_ncoef;
    unsigned int* conv_flag;               // bit 1: a nonzero coefficient at or past ncoef
};

// tile index -> (plane, m tile, n tile).  Unfused: planes outermost.  Fused:
// the planes of one output tile are consecutive so the epilogue can combine them.
template <int FUSE_K>
__device__ __forceinline__ void decode_tile(int tile, const Params& prm, int& pl, int& mt, int& nt);

__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int& mt, int& nt,
                                            int group_m = GROUP_M) {
    const int per_group = group_m * n_tiles;
    const int group = tile / per_group;
    const int first_m = group * group_m;
    const int gm = min(m_tiles - first_m, group_m);
    const int r = tile % per_group;
    mt = first_m + r % gm;
    nt = r / gm;
}

// MMA width of column tile nt: BN, or the last tile's remainder rounded up to
// 16 (the instruction's N granularity) -- a narrow tail costs its own width,
// not a full BN (cfg5: N = 8192 = 34 x 240 + 32)
template <int BN>
__device__ __forceinline__ int tile_n(const Params& prm, int nt) {
    const int64_t rem = prm.N - (int64_t)nt * BN;
    return rem >= BN ? BN : (int)((rem + 15) / 16 * 16);
}

template <int FUSE_K>
__device__ __forceinline__ void decode_tile(int tile, const Params& prm, int& pl, int& mt, int& nt) {
    if (FUSE_K || prm.plane_inner) {
        pl = tile % prm.planes;
        tile_coords(tile / prm.planes, prm.m_tiles, prm.n_tiles, mt, nt, prm.group_m);
    } else {
        // full-width tiles first (plane-major, grouped raster), then the narrow
        // tail tiles of every plane: the round-robin assignment then hands the
        // cheap tails to the CTAs that got one full tile fewer
        const int full_tiles = prm.m_tiles * prm.n_full;
        const int F = full_tiles * prm.planes;
        if (tile < F) {
            pl = tile / full_tiles;
            tile_coords(tile % full_tiles, prm.m_tiles, prm.n_full, mt, nt, prm.group_m);
        } else {
            const int i = tile - F;
            pl = i / prm.m_tiles;
            mt = i % prm.m_tiles;
            nt = prm.n_tiles - 1;
        }
    }
}

// convolution mode: a unit's y0 tile, first Toeplitz row block and K blocks
__device__ __forceinline__ void conv_unit(const Params& prm, int mt, int& my, int& w_lo, int& nkb) {
    const int split = mt / prm.conv_rows;
    my = mt - split * prm.conv_rows;
    w_lo = split * prm.conv_wc;
    const int w_hi = min(prm.conv_w, w_lo + prm.conv_wc);
    nkb = (w_hi - w_lo) * prm.conv_kpw;
}

template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
__global__ void __launch_bounds__(FUSE_K ? THREADS_FUSED : THREADS, 1)
    gemm_modp_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ Params prm_in) {
    using namespace sm100;
    using G = Geo<KIND, PAIR, FUSE_K, MC>;
    static_assert(!MC || (PAIR && FUSE_K == 0), "multicast needs the CTA-pair, unfused kernel");
    // the convolution / Toeplitz long-product modes run on the int8 kind only: compiled out of the
    // FP4 instantiations (the headline kernel), whose code then holds only what it executes
    constexpr bool CONVK = KIND == KIND_I8 && FUSE_K == 0;
    // MC: work units cover two m tiles (one per pair of the cluster)
    Params prm = prm_in;
    if (KIND == KIND_I8 && prm.seg_dev != nullptr) {
        const int nba = prm.seg_dev[0], nbb = prm.seg_dev[1], sp = prm.seg_s;
        const int i_lo = sp - (nbb - 1) > 0 ? sp - (nbb - 1) : 0, i_hi = sp < nba - 1 ? sp : nba - 1;
        if (i_hi < i_lo) return;  // every byte product of this shift is zero: C unchanged
        prm.seg_i_lo = i_lo;
        prm.num_kb = (i_hi - i_lo + 1) * prm.seg_kpb;
    }
    if (MC) {
        prm.m_tiles = (prm_in.m_tiles + 1) / 2;
        pdl_trigger();  // the concurrent tail launch may take the SMs no 4-CTA cluster fits on
    }
    constexpr int BN = G::BN;
    constexpr int NST = G::STAGES_N;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + NST * G::STAGE_BYTES);
    uint64_t* empty_bar = full_bar + NST;
    uint64_t* tmem_full = empty_bar + NST;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    constexpr int CL = MC ? 4 : (PAIR ? 2 : 1);  // CTAs per cluster
    const uint32_t crank = PAIR ? cluster_ctarank() : 0;
    const uint32_t rank = crank & 1;                // rank within the CTA pair
    const uint32_t pidx = MC ? (crank >> 1) : 0;    // pair within the cluster
    const uint32_t pair_leader = crank & ~1u;       // cluster rank of this pair's leader
    const bool leader = rank == 0;
    const int group_id = blockIdx.x / CL;
    const int num_groups = gridDim.x / CL;
    // work units: one tile of one plane; fused, one output tile with all its
    // planes processed back to back by the same CTA (group)
    const int plane_tiles = prm.m_tiles * prm.n_tiles;
    const bool inner = FUSE_K || prm.plane_inner;
    const int per_unit = inner ? prm.planes : 1;
    const int units = inner ? plane_tiles : plane_tiles * prm.planes;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmap_a);
        tma_prefetch(&tmap_b);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], MC ? 2 : 1);  // MC: both pairs' MMAs free the stage
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            // one arrival per epilogue warp (of both CTAs)
            mbar_init(&tmem_empty[a], (FUSE_K ? 8 : 4) * (PAIR ? 2 : 1));
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        if (PAIR) tmem_alloc_pair<512>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    if (PAIR) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (KIND == KIND_F4 && warp >= 4 && warp < 8) {
        tmem_fill_sf(tmem_base + ((uint32_t)((warp - 4) * 32) << 16) + Cfg<KIND>::SF_COL, prm.sf);
        tc_fence_before();
    }
    if (PAIR) cluster_sync();
    else __syncthreads();
    tc_fence_after();

    if (warp == 0) {
        // ===== TMA producer (both CTAs of a pair load their own halves) =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = group_id; u < units; u += num_groups)
            for (int sp = 0; sp < per_unit; ++sp) {
                const int tile = u * per_unit + sp;
                int pl, mt, nt;
                decode_tile<FUSE_K>(tile, prm, pl, mt, nt);
                if (MC) mt = 2 * mt + (int)pidx;
                nt += prm.n_tile0;
                const int pstack = prm.plane_inner ? 0 : pl;  // planes stacked along the operand rows
                const int arow = (int)(pstack * prm.M) + mt * G::TILE_M + (int)rank * BM;
                // the pair splits the tile's (possibly narrowed, see tile_n) columns in halves
                const int brow = (int)(pstack * prm.N) + nt * BN + (int)rank * (tile_n<BN>(prm, nt) / 2);
                int nkb = prm.plane_inner ? prm.seg_cnt[pl] * prm.seg_kpb : prm.num_kb;
                int cmy = 0, cwlo = 0;
                if (CONVK && prm.conv) conv_unit(prm, mt, cmy, cwlo, nkb);
                const int seg_lo = prm.plane_inner ? prm.seg_lo[pl] : prm.seg_i_lo;
                const int seg_s = prm.plane_inner ? pl : prm.seg_s;
                // MC: CTA (pair i, rank r) loads slice i of half r and multicasts it to both pairs
                const uint16_t mc_mask = (uint16_t)((1u << crank) | (1u << (crank ^ 2u)));
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * G::STAGE_BYTES;
                    uint8_t* sb = sa + G::A_BYTES;
                    int ak = kb * BK, bk = kb * BK, boff = 0;
                    if (prm.seg_kpb) {  // byte-plane segments of the uint64 GEMM
                        const int seg = kb / prm.seg_kpb, kin = kb - seg * prm.seg_kpb, i = seg_lo + seg;
                        ak = i * prm.seg_kp + kin * BK;
                        bk = kin * BK;
                        boff = (seg_s - i) * (int)prm.N;
                    }
                    if (CONVK && PAIR && !MC && prm.conv) {  // convolution mode on a CTA pair: rows y0 = rank * 128
                        const uint32_t lbar = map_to_rank(&full_bar[stage], 0);
                        if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * (G::A_BYTES + prm.conv_brows * BK));
                        const int wk = kb / prm.conv_kpw, kin = (kb - wk * prm.conv_kpw) * BK, w = cwlo + wk;
                        const int r0 = (prm.conv_x0 - cmy * G::TILE_M - (int)rank * BM - w * prm.conv_tl - 127) / 16;
                        tma_load_4d_pair(sa, &tmap_a, lbar, kin, r0, 0, pl);  // 16 phases x 8 rows
                        tma_load_3d_pair(sb, &tmap_b, lbar, kin, nt * prm.conv_tn + (int)rank * prm.conv_brows - w, pl);
                    } else if (CONVK && !PAIR && !MC && prm.conv) {  // convolution mode: Toeplitz block w, b blocks shifted by w
                        mbar_arrive_expect_tx(&full_bar[stage], G::A_BYTES + prm.conv_brows * BK);
                        const int wk = kb / prm.conv_kpw, kin = (kb - wk * prm.conv_kpw) * BK, w = cwlo + wk;
                        const int r0 = (prm.conv_x0 - cmy * G::TILE_M - w * prm.conv_tl - 127) / 16;
                        tma_load_4d(sa, &tmap_a, &full_bar[stage], kin, r0, 0, pl);  // 16 phases x 8 rows
                        tma_load_3d(sb, &tmap_b, &full_bar[stage], kin, nt * prm.conv_tn - w, pl);
                    } else if (CONVK && !PAIR && !MC && prm.a_phase) {  // Toeplitz operand: 16 phase boxes + B
                        mbar_arrive_expect_tx(&full_bar[stage], G::STAGE_BYTES);
                        const int r0 = (mt * G::TILE_M) / 16;
                        tma_load_4d(sa, &tmap_a, &full_bar[stage], ak, r0, 0, pl);  // 16 phases x 8 rows
                        tma_load_2d(sb, &tmap_b, &full_bar[stage], bk, brow + boff);
                    } else if (prm.diag_noload && (u != group_id || kb >= NST)) {  // wrong results: power probe
                        if (!PAIR || leader) mbar_arrive(&full_bar[stage]);
                    } else if (MC) {
                        const uint32_t lbar = map_to_rank(&full_bar[stage], pair_leader);
                        if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * G::STAGE_BYTES);
                        tma_load_2d_pair(sa, &tmap_a, lbar, ak, arow);
                        tma_load_2d_pair_mc(sb + pidx * G::B_BOX * BK, &tmap_b, lbar, bk,
                                            brow + boff + (int)pidx * G::B_BOX, mc_mask);
                    } else if (PAIR) {
                        const uint32_t lbar = map_to_rank(&full_bar[stage], 0);
                        if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * G::STAGE_BYTES);
                        tma_load_2d_pair(sa, &tmap_a, lbar, ak, arow);
                        tma_load_2d_pair(sb, &tmap_b, lbar, bk, brow + boff);
                    } else {
                        mbar_arrive_expect_tx(&full_bar[stage], G::STAGE_BYTES);
                        tma_load_2d(sa, &tmap_a, &full_bar[stage], ak, arow);
                        tma_load_2d(sb, &tmap_b, &full_bar[stage], bk, brow + boff);
                    }
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ===== MMA issuer (pair leader only): 4 MMAs of 32 bytes per stage =====
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int u = group_id; u < units; u += num_groups)
        for (int sp = 0; sp < per_unit; ++sp, ++local) {
            int pl, mt, nt;
            decode_tile<FUSE_K>(u * per_unit + sp, prm, pl, mt, nt);
            nt += prm.n_tile0;
            int nkb = prm.plane_inner ? prm.seg_cnt[pl] * prm.seg_kpb : prm.num_kb;
            if (CONVK && prm.conv) {
                int cmy, cwlo;
                conv_unit(prm, mt, cmy, cwlo, nkb);
            }
            const uint32_t nn = (CONVK && prm.conv) ? (uint32_t)prm.conv_tn : (uint32_t)tile_n<BN>(prm, nt);
            const uint32_t idesc = KIND == KIND_I8 ? idesc_u8_s32(G::TILE_M, nn) : idesc_mxf4(G::TILE_M, nn);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + acc * BN;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sa = smem_addr(smem + stage * G::STAGE_BYTES);
                    const uint32_t sb = sa + G::A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k) {
                        const uint64_t ad = smem_desc_k_sw128(sa + k * 32), bd = smem_desc_k_sw128(sb + k * 32);
                        const uint32_t accum = (kb | k) != 0;
                        const uint32_t sf = tmem_base + (Cfg<KIND>::SF_COL > 0 ? Cfg<KIND>::SF_COL : 0);
                        if (KIND == KIND_I8) {
                            if (PAIR) umma_i8_pair(tmem_d, ad, bd, idesc, accum);
                            else umma_i8(tmem_d, ad, bd, idesc, accum);
                        } else {
                            if (PAIR) umma_mxf4_pair(tmem_d, ad, bd, idesc, accum, sf, sf);
                            else umma_mxf4(tmem_d, ad, bd, idesc, accum, sf, sf);
                        }
                    }
                    if (PAIR) {
                        umma_commit_pair(&empty_bar[stage], MC ? 0xF : 0x3);
                        if (kb == nkb - 1) umma_commit_pair(&tmem_full[acc], (uint16_t)(0x3u << (2 * pidx)));
                    } else {
                        umma_commit(&empty_bar[stage]);
                        if (kb == nkb - 1) umma_commit(&tmem_full[acc]);
                    }
                }
                __syncwarp();
                if (++stage == NST) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> mod p -> uint8 =====
        const int ew = warp - 4;   // TMEM lane quarter this warp may access (unfused: 4 warps)
        const int ew4 = warp & 3;  // fused (8 warps): warps 4+q and 8+q share lane quarter q
        const uint32_t empty_addr0 = PAIR ? map_to_rank(&tmem_empty[0], pair_leader) : 0;
        const uint32_t empty_addr1 = PAIR ? map_to_rank(&tmem_empty[1], pair_leader) : 0;
        int local = 0;
        // fused: this thread's byte-lane plane sums, 16 columns x FUSE_K bytes per chunk
        uint32_t facc[FUSE_K ? (BN / 16 + 1) / 2 : 1][FUSE_K ? 4 * FUSE_K : 1];
        (void)facc;
        for (int u = group_id; u < units; u += num_groups)
        for (int sp = 0; sp < per_unit; ++sp, ++local) {
            const int tile = u * per_unit + sp;
            int pl, mt, nt;
            decode_tile<FUSE_K>(tile, prm, pl, mt, nt);
            if (MC) mt = 2 * mt + (int)pidx;
            nt += prm.n_tile0;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tmem_full[acc], acc_phase);
            tc_fence_after();
            int64_t row = (int64_t)mt * G::TILE_M + (int)rank * BM + (FUSE_K ? ew4 : ew) * 32 + lane;
            bool row_ok = row < prm.M;
            if (CONVK && !PAIR && prm.a_phase) {  // smem / TMEM row l = 8 phi + r holds GEMM row 16 r + phi
                const int l = ew * 32 + lane;
                const int64_t x = (int64_t)mt * G::TILE_M + 16 * (l % 8) + l / 8;
                row_ok = x < prm.M;
                row = prm.M - 1 - x;
            }
            if constexpr (FUSE_K > 0) {
                // plane pl of this tile: acc[(col, l)] += W[l][pl] * (D_pl[row, col] mod p)
                // on byte lanes held in registers (S * (p-1)^2 < 256: no carries).
                // 8 epilogue warps: lane quarter q = warp & 3, 16-column chunks of
                // parity h; the last plane reduces mod p and writes the coefficients.
                constexpr int NCH = BN / 16, MYCH = (NCH + 1) / 2, W4 = 4 * FUSE_K;
                const int h = (warp - 4) >> 2;
                uint32_t mult[FUSE_K][4];  // W[l][pl] placed in byte lane j
#pragma unroll
                for (int l = 0; l < FUSE_K; ++l)
#pragma unroll
                    for (int j = 0; j < 4; ++j) mult[l][j] = (uint32_t)prm.W[l][pl] << (8 * j);
                if (sp == 0) {
#pragma unroll
                    for (int i = 0; i < MYCH; ++i)
#pragma unroll
                        for (int q = 0; q < W4; ++q) facc[i][q] = 0;
                }
                const int nch = tile_n<BN>(prm, nt) / 16;
                // (run_kara always sets magic32 for the fused kernel's fields: p <= 7; the offset add is
                // compiled out for non-negative representatives, cfg3's case)
                const uint32_t fm32 = prm.magic32, fnp = 0u - prm.p, foff = prm.offset;
                auto fchunks = [&](auto has_off) {
#pragma unroll
                    for (int i = 0; i < MYCH; ++i) {
                        const int ch = 2 * i + h;
                        if (ch < NCH && ch < nch) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew4 * 32) << 16) + acc * BN + ch * 16, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                uint32_t x = (uint32_t)__float2int_rn(__uint_as_float(v[c]));
                                if (decltype(has_off)::value) x += foff;
                                const uint32_t r = __umulhi(x, fm32) * fnp + x;
#pragma unroll
                                for (int l = 0; l < FUSE_K; ++l) {
                                    const int pos = c * FUSE_K + l;
                                    facc[i][pos >> 2] += r * mult[l][pos & 3];
                                }
                            }
                        }
                    }
                };
                if (foff) fchunks(std::true_type{});
                else fchunks(std::false_type{});
                // TMEM fully read: hand the accumulator back to the MMA warp first
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_cluster(acc ? empty_addr1 : empty_addr0);
                    else mbar_arrive(&tmem_empty[acc]);
                }
                if (pl == prm.planes - 1 && row_ok) {
                    const LaneDiv ldv = {prm.lane_m, prm.lane_sh, prm.lane_qmask};
#pragma unroll
                    for (int i = 0; i < MYCH; ++i) {
                        const int ch = 2 * i + h;
                        const int64_t col0 = (int64_t)nt * BN + ch * 16;
                        if (ch >= NCH || col0 >= prm.N) continue;
                        uint32_t o[W4];
#pragma unroll
                        for (int q = 0; q < W4; ++q) o[q] = lanes_mod_div(facc[i][q], prm.p, ldv);
                        uint8_t* dst = prm.c + row * prm.ldc + col0 * FUSE_K;
                        if (col0 + 16 <= prm.N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
                            for (int q = 0; q < FUSE_K; ++q)
                                reinterpret_cast<uint4*>(dst)[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
                        } else {
                            const int64_t nb = (prm.N - col0 < 16 ? prm.N - col0 : 16) * FUSE_K;
#pragma unroll
                            for (int e = 0; e < W4 * 4; ++e)  // unrolled: o[] stays in registers
                                if (e < nb) dst[e] = (uint8_t)(o[e >> 2] >> (8 * (e & 3)));
                        }
                    }
                }
                continue;
            }
            if (CONVK && prm.conv) {
                // TMEM lane l = smem row 8 phi + r = tile row i = 127 - 16 r - phi: coefficient
                // y = y0 + i + v TL of pair pl, column c = block v (y0 = the CTA's 128 rows)
                const int l = ew * 32 + lane;
                int cmy, cwlo, cnkb;
                conv_unit(prm, mt, cmy, cwlo, cnkb);
                const int64_t ybase = (int64_t)cmy * G::TILE_M + (int)rank * BM + 127 - 16 * (l % 8) - l / 8;
                uint8_t* orow = prm.c + (int64_t)pl * prm.ldc;
                int32_t* prow = prm.conv_part ? prm.conv_part + ((int64_t)(mt / prm.conv_rows) * prm.planes + pl) * prm.conv_ytot
                                              : nullptr;
                const int nch = prm.conv_tn / 16;
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + ch * 16, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int64_t col = (int64_t)nt * prm.conv_tn + ch * 16 + e;
                        if (col >= prm.N) continue;
                        const int64_t y = ybase + col * prm.conv_tl;
                        if (prow) {  // split-K partial: raw int32 sum
                            if (y < prm.conv_ytot) prow[y] = (int32_t)v[e];
                            continue;
                        }
                        const uint32_t r = mod_u32(v[e], prm.p, prm.magic64);
                        if (y < prm.conv_ncoef) orow[y] = (uint8_t)r;
                        else if (r) atomicOr(prm.conv_flag, 2u);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_cluster(acc ? empty_addr1 : empty_addr0);
                    else mbar_arrive(&tmem_empty[acc]);
                }
                continue;
            }
            uint8_t* crow = prm.c + pl * prm.c_plane + row * prm.ldc;
            const int nch = tile_n<BN>(prm, nt) / 16;  // accumulator columns the MMA wrote
            // Whole tile in range, nibble planes, 32-bit reciprocal: the plane GEMM's common case without
            // the per-chunk range / alignment tests (the epilogue runs under the MMA, but every
            // instruction it issues is power the capped tensor clock does not get)
            if (prm.nibble_out && prm.magic32 && !prm.epi_mod64 && !prm.diag_shift &&
                __all_sync(0xffffffffu, row_ok) && (int64_t)nt * BN + nch * 16 <= prm.N &&
                ((reinterpret_cast<uintptr_t>(crow + ((int64_t)nt * BN) / 2)) & 7) == 0) {
                uint2* dst = reinterpret_cast<uint2*>(crow + ((int64_t)nt * BN) / 2);
                const uint32_t m32 = prm.magic32, np = 0u - prm.p, off = prm.offset;
                const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
                auto chunks = [&](auto has_off) {  // per element: F2I (+ offset), IMAD.HI, IMAD, IMAD (Horner pack)
#pragma unroll 1
                    for (int ch = 0; ch < nch; ++ch) {
                        uint32_t v[16];
                        tmem_ld_32x32b_x16(tbase + ch * 16, v);
                        tmem_ld_wait();
                        uint32_t w[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint32_t acc_w = 0;
#pragma unroll
                            for (int e = 7; e >= 0; --e) {
                                uint32_t x = KIND == KIND_I8 ? v[8 * h + e]
                                                             : (uint32_t)__float2int_rn(__uint_as_float(v[8 * h + e]));
                                if (decltype(has_off)::value) x += off;
                                acc_w = acc_w * 16u + (__umulhi(x, m32) * np + x);
                            }
                            w[h] = acc_w;
                        }
                        dst[ch] = make_uint2(w[0], w[1]);
                    }
                };
                if (off) chunks(std::true_type{});
                else chunks(std::false_type{});
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR) mbar_arrive_cluster(acc ? empty_addr1 : empty_addr0);
                    else mbar_arrive(&tmem_empty[acc]);
                }
                continue;
            }
#pragma unroll 1
            for (int ch = 0; ch < nch; ++ch) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + ch * 16, v);
                tmem_ld_wait();
                const int64_t col0 = (int64_t)nt * BN + ch * 16;
                if (!row_ok || col0 >= prm.N) continue;
                if (KIND == KIND_I8 && prm.c64 != nullptr) {  // byte-plane uint64 GEMM (mod 2^64)
                    const int shift = prm.plane_inner ? 8 * pl : prm.shift;
                    const bool acc64 = prm.plane_inner ? (pl > 0 || prm.acc64) : prm.acc64 != 0;
                    uint64_t* crow64 = prm.c64 + row * prm.ldc + col0;
                    const int ncol = (int)(prm.N - col0 < 16 ? prm.N - col0 : 16);
                    if (ncol == 16 && ((reinterpret_cast<uintptr_t>(crow64) & 15) == 0)) {
#pragma unroll
                        for (int e = 0; e < 16; e += 2) {
                            ulonglong2 o = make_ulonglong2((uint64_t)v[e] << shift, (uint64_t)v[e + 1] << shift);
                            if (acc64) {
                                const ulonglong2 old = *reinterpret_cast<const ulonglong2*>(crow64 + e);
                                o.x += old.x;
                                o.y += old.y;
                            }
                            *reinterpret_cast<ulonglong2*>(crow64 + e) = o;
                        }
                    } else {
                        for (int e = 0; e < ncol; ++e) {
                            const uint64_t o = (uint64_t)v[e] << shift;
                            crow64[e] = acc64 ? crow64[e] + o : o;
                        }
                    }
                    continue;
                }
                uint32_t r[16];
                if (prm.magic32 && !prm.epi_mod64) {  // (a real branch: both forms predicated per element cost issue slots)
                    const uint32_t m32 = prm.magic32, np = 0u - prm.p;  // x - p q as one IMAD with -p
                    const int off = (int)prm.offset;
                    if (KIND == KIND_I8) {  // non-negative int32 sums (the host sets magic32 only then)
#pragma unroll
                        for (int e = 0; e < 16; ++e) r[e] = __umulhi(v[e], m32) * np + v[e];
                    } else if (off == 0) {  // non-negative representatives: F2I, IMAD.HI, IMAD per element
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const uint32_t x = (uint32_t)__float2int_rn(__uint_as_float(v[e]));
                            r[e] = __umulhi(x, m32) * np + x;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const uint32_t x = (uint32_t)(__float2int_rn(__uint_as_float(v[e])) + off);
                            r[e] = __umulhi(x, m32) * np + x;
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        uint32_t x;
                        if (KIND == KIND_I8) x = v[e];
                        else x = (uint32_t)(__float2int_rn(__uint_as_float(v[e])) + (int)prm.offset);
                        r[e] = mod_u32(x, prm.p, prm.magic64);
                    }
                }
                if (prm.nibble_out) {  // residues < 16: two per byte, 8 bytes per 16 columns
                    uint32_t w0 = r[7], w1 = r[15];  // Horner: one multiply-add per nibble
#pragma unroll
                    for (int e = 6; e >= 0; --e) {
                        w0 = w0 * 16u + r[e];
                        w1 = w1 * 16u + r[8 + e];
                    }
                    uint8_t* dst = crow + col0 / 2;
                    if (col0 + 16 <= prm.N && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
                        *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
                    } else {
                        for (int e = 0; e < 16 && col0 + e < prm.N; e += 2) {
                            const uint32_t hi = (col0 + e + 1 < prm.N) ? r[e + 1] : 0;
                            dst[e / 2] = (uint8_t)(r[e] | (hi << 4));
                        }
                    }
                } else if (CONVK && prm.diag_shift) {
                    // diagonal-shifted transpose (Toeplitz products): column v of row x lands at
                    // c[v][x + v * diag_shift] -- a warp's 32 rows write 32 consecutive bytes per column
                    uint8_t* cpl = prm.c + pl * prm.c_plane;
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (col0 + e < prm.N) cpl[(col0 + e) * prm.ldc + row + (col0 + e) * prm.diag_shift] = (uint8_t)r[e];
                } else {
                    uint32_t w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        w[q] = r[4 * q] | (r[4 * q + 1] << 8) | (r[4 * q + 2] << 16) | (r[4 * q + 3] << 24);
                    if (col0 + 16 <= prm.N && ((reinterpret_cast<uintptr_t>(crow + col0) & 15) == 0)) {
                        *reinterpret_cast<uint4*>(crow + col0) = make_uint4(w[0], w[1], w[2], w[3]);
                    } else {
                        for (int e = 0; e < 16 && col0 + e < prm.N; ++e) crow[col0 + e] = (uint8_t)r[e];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) mbar_arrive_cluster(acc ? empty_addr1 : empty_addr0);
                else mbar_arrive(&tmem_empty[acc]);
            }
        }
    }
    tc_fence_before();
    if (PAIR) cluster_sync();
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair<512>(tmem_base);
        else tmem_dealloc<512>(tmem_base);
    }
    if (prm.pdl_tail) pdl_wait();
}

// ---------------------------------------------------------------------------
// Operand preparation.
// I8: Bx bytes = residues.  F4: Bx / A nibbles = E2M1 codes of centred residues.
// Table-driven expansion (fields with p^K <= XT_CODES): every element code maps
// to its K x K block, staged in shared memory as K rows (T[code*K + l] = the K
// output values of row l, bytes for I8 / nibbles for F4).  Tile = 64 kk x 64 j;
// b rows are read with 16-byte loads, codes stored j-major so that one work item
// (an output row segment of 16K bytes) reads contiguous smem and issues K
// 16-byte stores.  Grid-stride over tiles amortises the table build.
// ---------------------------------------------------------------------------
constexpr int XT_KK = 64, XT_J = 64, XT_CODES = 1024;

template <int K, int KIND>
__global__ void __launch_bounds__(256) expand_b_table_kernel(const uint8_t* __restrict__ b, int64_t Kd, int64_t N,
                                                             FieldConst f, uint32_t nib_lut, uint8_t* __restrict__ bx,
                                                             int64_t ldb, int tiles_kk, int tiles_j) {
    constexpr int ELEM_PER_ITEM = KIND == KIND_I8 ? 16 : 32;  // kk per work item (16K output bytes)
    __shared__ uint32_t tab[XT_CODES * K];
    __shared__ __align__(16) uint8_t raw[XT_KK][XT_J * K + 16];
    __shared__ __align__(16) uint16_t code[XT_J][XT_KK + 8];
    const uint32_t p = f.p;
    int ncodes = 1;
    for (int s = 0; s < K; ++s) ncodes *= (int)p;
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
            const uint32_t res = mod_small(acc, p, f.magic);
            if (KIND == KIND_I8) w |= res << (8 * i);
            else w |= ((nib_lut >> (4 * res)) & 0xF) << (4 * i);
        }
        tab[e] = w;
    }
    const bool vec_rows = ((N * K) % 16 == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t kk0 = (tile % tiles_kk) * XT_KK, j0 = (tile / tiles_kk) * XT_J;
        __syncthreads();
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
        for (int i = threadIdx.x; i < XT_KK * XT_J; i += blockDim.x) {
            const int r = i / XT_J, jl = i % XT_J;
            uint32_t cd = 0;
#pragma unroll
            for (int s = K - 1; s >= 0; --s) cd = cd * p + raw[r][jl * K + s];
            code[jl][r] = (uint16_t)cd;
        }
        __syncthreads();
        constexpr int CHUNKS = XT_KK / ELEM_PER_ITEM;
        for (int i = threadIdx.x; i < XT_J * K * CHUNKS; i += blockDim.x) {
            const int ch = i % CHUNKS, row = i / CHUNKS;
            const int jl = row / K, l = row % K;
            const int64_t gj = j0 + jl;
            if (gj >= N) continue;
            uint32_t w[4 * K];
#pragma unroll
            for (int q = 0; q < 4 * K; ++q) w[q] = 0;
            const uint16_t* cr = &code[jl][ch * ELEM_PER_ITEM];
#pragma unroll
            for (int e = 0; e < ELEM_PER_ITEM; ++e) {
                const uint32_t v = tab[cr[e] * K + l];
#pragma unroll
                for (int ii = 0; ii < K; ++ii) {
                    const int pos = e * K + ii;
                    if (KIND == KIND_I8) w[pos / 4] |= ((v >> (8 * ii)) & 0xFF) << (8 * (pos % 4));
                    else w[pos / 8] |= ((v >> (4 * ii)) & 0xF) << (4 * (pos % 8));
                }
            }
            const int64_t col = (kk0 + ch * ELEM_PER_ITEM) * K / (KIND == KIND_I8 ? 1 : 2);  // bytes
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

// Generic arithmetic expansion for large fields (p^K > XT_CODES), INT8 only.
constexpr int EX_T = 64;
__global__ void __launch_bounds__(256) expand_b_generic_kernel(const uint8_t* __restrict__ b, int64_t K, int64_t N,
                                                               FieldConst f, uint8_t* __restrict__ bx, int64_t ldb) {
    __shared__ uint8_t sb[EX_T][EX_T * kMaxK + 4];
    __shared__ uint8_t xp[kMaxDigits][kMaxK];
    const int k = (int)f.k;
    if (threadIdx.x < kMaxDigits * kMaxK) xp[threadIdx.x / kMaxK][threadIdx.x % kMaxK] = f.xpow[threadIdx.x / kMaxK][threadIdx.x % kMaxK];
    const int64_t kk0 = (int64_t)blockIdx.x * EX_T, j0 = (int64_t)blockIdx.y * EX_T;
    const int rowbytes = EX_T * k;
    for (int i = threadIdx.x; i < EX_T * rowbytes; i += blockDim.x) {
        const int r = i / rowbytes, c = i % rowbytes;
        const int64_t gk = kk0 + r, gj = j0 + c / k;
        sb[r][c] = (gk < K && gj < N) ? b[gk * N * k + j0 * k + c] : 0;
    }
    __syncthreads();
    const int words_per_row = rowbytes / 4;
    const int64_t colbase = kk0 * k;
    for (int w = threadIdx.x; w < EX_T * k * words_per_row; w += blockDim.x) {
        const int orow = w / words_per_row, wq = w % words_per_row;
        const int jl = orow / k, l = orow % k;
        const int64_t gj = j0 + jl;
        if (gj >= N) continue;
        uint32_t word = 0;
        for (int e = 0; e < 4; ++e) {
            const int c = wq * 4 + e;
            const int kl = c / k, i = c % k;
            uint32_t acc = 0;
            for (int s = 0; s < k; ++s) acc += (uint32_t)sb[kl][jl * k + s] * xp[s + i][l];
            word |= mod_small(acc, f.p, f.magic) << (8 * e);
        }
        const int64_t col = colbase + wq * 4;
        uint8_t* dst = bx + (gj * k + l) * ldb + col;
        if (col + 4 <= ldb) *reinterpret_cast<uint32_t*>(dst) = word;
        else
            for (int e = 0; e < 4 && col + e < ldb; ++e) dst[e] = (uint8_t)(word >> (8 * e));
    }
}

// rows of width `width` bytes copied into a pitched, zero-padded buffer (I8 A)
__global__ void pad_rows_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t width, uint8_t* __restrict__ dst,
                                int64_t ld) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * ld) return;
    const int64_t r = i / ld, c = i % ld;
    dst[i] = c < width ? src[r * width + c] : 0;
}

// A residues -> packed E2M1 nibbles of the centred residues, pitched rows (F4 A).
// Each thread: 32 residues (2 x 16B loads when aligned) -> 16 bytes out.
__global__ void pack_a_f4_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t width, uint32_t nib_lut,
                                 uint8_t* __restrict__ dst, int64_t ld) {
    const int64_t per_row = ld / 16;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * per_row) return;
    const int64_t r = i / per_row, q = i % per_row;
    const int64_t c0 = q * 32;  // first residue of this 16-byte chunk
    const uint8_t* s = src + r * width;
    uint32_t out[4] = {0, 0, 0, 0};
    if (c0 + 32 <= width && ((reinterpret_cast<uintptr_t>(s + c0) & 15) == 0)) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(s + c0));
        const uint4 y = __ldg(reinterpret_cast<const uint4*>(s + c0) + 1);
        const uint32_t in[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const uint32_t res = (in[e / 4] >> (8 * (e % 4))) & 0xFF;
            out[e / 8] |= ((nib_lut >> (4 * res)) & 0xF) << (4 * (e % 8));
        }
    } else {
        for (int e = 0; e < 32; ++e) {
            if (c0 + e < width) {
                const uint32_t res = s[c0 + e];
                out[e / 8] |= ((nib_lut >> (4 * res)) & 0xF) << (4 * (e % 8));
            }
        }
    }
    *reinterpret_cast<uint4*>(dst + r * ld + q * 16) = make_uint4(out[0], out[1], out[2], out[3]);
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

static int num_sms() { return num_sms_cached(); }

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static bool getenv_flag(const char* name) {
    const char* e = getenv(name);
    return e && e[0] && e[0] != '0';
}

// CTA-pair (cta_group::2) GEMM unless QADIC_TC_PAIR=0
static bool pair_mode() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("QADIC_TC_PAIR");
        mode = (e && e[0] == '0') ? 0 : 1;
    }
    return mode == 1;
}

// B-tile multicast across two CTA pairs for the unfused fp4k GEMM (QADIC_MCAST=1)
static bool mcast_mode() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("QADIC_MCAST");
        mode = (e && e[0] == '1') ? 1 : 0;
    }
    return mode == 1;
}

// E2M1 nibble codes of the centred residues 0..p-1 (p <= 7), packed 4 bits each
// E2M1 codes of the residue representatives (4-bit code of residue r at nibble r).
// Every operand value is a half-integer code under block scales 2^1 on both
// operands, so each product is (x/2)(y/2) * 4 = x*y exactly; the representable
// integers are +-{0, 1, 2, 3, 4, 6, 8, 12}.  Preferred: the smallest NON-NEGATIVE
// representative of each residue (p = 7: 0, 1, 2, 3, 4, 12, 6) -- no sign bits,
// fewer operand bit toggles, and the power-capped GEMM clocks higher (cfg5 GEMM
// 0.749 vs 0.782 ms centred; cfg3 0.446 vs 0.474) -- while K * max_v^2 stays below
// 2^24 (exact fp32 sums); else the centred residues (|v| <= 3).
// QADIC_E2M1_CENTRED=1 forces centred, QADIC_E2M1_INT=1 the integer codes with
// unit scales (both for measurements).
static bool e2m1_half() {
    static const bool on = !(getenv("QADIC_E2M1_INT") && atoi(getenv("QADIC_E2M1_INT")) != 0);
    return on;
}
static uint32_t e2m1_scale_word() { return e2m1_half() ? 0x80808080u : 0x7F7F7F7Fu; }
static int nonneg_rep(uint32_t r, uint32_t p) {  // smallest representable v >= 0 with v = r mod p, or -1
    static const int vals[8] = {0, 1, 2, 3, 4, 6, 8, 12};
    for (int v : vals)
        if ((uint32_t)v % p == r) return v;
    return -1;
}
static uint32_t e2m1_lut(uint32_t p, int64_t kdim) {
    static const bool force_centred = getenv("QADIC_E2M1_CENTRED") && atoi(getenv("QADIC_E2M1_CENTRED")) != 0;
    int maxv = 0;
    bool nonneg = e2m1_half() && !force_centred;
    for (uint32_t r = 0; r < p && nonneg; ++r) {
        const int v = nonneg_rep(r, p);
        if (v < 0) nonneg = false;
        else if (v > maxv) maxv = v;
    }
    if (nonneg && (__int128)kdim * maxv * maxv >= ((__int128)1 << 24)) nonneg = false;
    static const uint32_t pos_int[4] = {0x0, 0x2, 0x4, 0x5};   // 0, 1, 2, 3
    static const uint32_t pos_half[4] = {0x0, 0x1, 0x2, 0x3};  // 0, 0.5, 1, 1.5
    uint32_t lut = 0;
    for (uint32_t r = 0; r < p; ++r) {
        uint32_t code;
        if (nonneg) {
            static const int vals[8] = {0, 1, 2, 3, 4, 6, 8, 12};
            const int v = nonneg_rep(r, p);
            code = 0;
            for (uint32_t c = 0; c < 8; ++c)
                if (vals[c] == v) code = c;  // half codes 0..7 = 0, 0.5, 1, 1.5, 2, 3, 4, 6
        } else {
            const uint32_t* pos = e2m1_half() ? pos_half : pos_int;
            const int v = (2 * r <= p - 1) ? (int)r : (int)r - (int)p;
            code = v >= 0 ? pos[v] : (0x8u | pos[-v]);
        }
        lut |= code << (4 * r);
    }
    return lut;
}

struct Layout {
    int64_t Kb;      // inner elements (K * k)
    int64_t inner;   // inner bytes of the operand tensors
    int64_t lda, ldb;
    bool prep_a;     // A needs a prepass (padding for I8, conversion for F4)
    size_t bx_bytes, a_bytes;
};

static Layout plan(int kind, const uint8_t* a, int64_t m, int64_t kdim, int64_t n, int k) {
    Layout L;
    L.Kb = kdim * k;
    L.inner = kind == KIND_I8 ? L.Kb : (L.Kb + 1) / 2;
    L.ldb = round_up(L.inner, 16);
    L.prep_a = kind == KIND_F4 || (L.Kb % 16 != 0) || ((reinterpret_cast<uintptr_t>(a) & 15) != 0);
    L.lda = L.prep_a ? L.ldb : L.Kb;
    L.bx_bytes = (size_t)round_up(n * k * L.ldb, 1024);
    L.a_bytes = L.prep_a ? (size_t)round_up(m * L.lda, 1024) : 0;
    return L;
}

template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
static cudaLaunchConfig_t gemm_config(cudaStream_t s) {
    using G = Geo<KIND, PAIR, FUSE_K, MC>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_modp_kernel<KIND, PAIR, FUSE_K, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)G::SMEM);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(FUSE_K ? THREADS_FUSED : THREADS);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = s;
    return cfg;
}

// Co-resident clusters of the persistent GEMM (GPC shapes leave some SMs out
// of 4-CTA clusters: 33 x 4 of 148 on B200; a second wave would double the time).
template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
static int gemm_max_clusters() {
    static int max_clusters = 0;
    if (!max_clusters) {
        const int per = MC ? 4 : (PAIR ? 2 : 1);
        cudaLaunchConfig_t cfg = gemm_config<KIND, PAIR, FUSE_K, MC>(nullptr);
        cfg.gridDim = dim3((unsigned)(num_sms() / per * per));
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = per;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&max_clusters, (void*)gemm_modp_kernel<KIND, PAIR, FUSE_K, MC>, &cfg) !=
                cudaSuccess ||
            max_clusters < 1)
            max_clusters = num_sms() / per;
        cudaGetLastError();
        if (getenv_flag("QADIC_VERBOSE"))
            fprintf(stderr, "[qadic] gemm<%d,%d,%d,%d>: %d co-resident clusters of %d CTAs (%d SMs)\n", KIND,
                    (int)PAIR, FUSE_K, (int)MC, max_clusters, per, num_sms());
    }
    return max_clusters;
}

// One persistent GEMM launch.  max_clusters > 0 caps the grid (the tail launch
// of a split runs on the SMs the 4-CTA clusters leave free); pdl_secondary
// launches it as the programmatic dependent of the launch just before it.
template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
static cudaError_t launch_gemm_raw(const CUtensorMap& ta, const CUtensorMap& tb, const Params& prm, cudaStream_t s,
                                   int max_clusters = 0, bool pdl_secondary = false) {
    const int per = MC ? 4 : (PAIR ? 2 : 1);  // CTAs per cluster
    // cluster work units of the launch: tiles of every plane (plane-inner / fused
    // launches walk the planes of one tile inside a unit)
    const int64_t per_plane = (int64_t)(MC ? (prm.m_tiles + 1) / 2 : prm.m_tiles) * prm.n_tiles;
    const int64_t units = (FUSE_K || prm.plane_inner) ? per_plane : per_plane * (prm.planes > 0 ? prm.planes : 1);
    int grid = gemm_max_clusters<KIND, PAIR, FUSE_K, MC>();
    if (max_clusters > 0 && max_clusters < grid) grid = max_clusters;
    if (units < grid) grid = (int)units;
    cudaLaunchConfig_t cfg = gemm_config<KIND, PAIR, FUSE_K, MC>(s);
    cfg.gridDim = dim3((unsigned)(grid * per));
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = per;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = pdl_secondary ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, gemm_modp_kernel<KIND, PAIR, FUSE_K, MC>, ta, tb, prm);
}

template <int KIND, bool PAIR, int FUSE_K = 0, bool MC = false>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, Params prm, cudaStream_t s,
                       const char* label = nullptr) {
    const char* name = label ? label : (KIND == KIND_I8 ? "i8 gemm" : "fp4 gemm");
    // diagnostics: QADIC_DIAG_GEMM_CLUSTERS caps the persistent grid (SM-count scaling probe)
    static const int cap = getenv("QADIC_DIAG_GEMM_CLUSTERS") ? atoi(getenv("QADIC_DIAG_GEMM_CLUSTERS")) : 0;
    QADIC_TIMED(name, s, (launch_gemm_raw<KIND, PAIR, FUSE_K, MC>(ta, tb, prm, s, cap)));
    return check_launch(name);
}

template <int K, int KIND>
static void launch_expand_table(const uint8_t* b, int64_t kdim, int64_t n, const FieldConst& f, uint32_t lut,
                                uint8_t* bx, int64_t ldb, cudaStream_t s) {
    const int tk = (int)((kdim + XT_KK - 1) / XT_KK), tj = (int)((n + XT_J - 1) / XT_J);
    const int64_t tiles = (int64_t)tk * tj;
    const int grid = (int)(tiles < 4 * num_sms() ? tiles : 4 * num_sms());
    QADIC_TIMED("expand B", s,
                (expand_b_table_kernel<K, KIND><<<grid, 256, 0, s>>>(b, kdim, n, f, lut, bx, ldb, tk, tj)));
}

template <int KIND>
static void expand_dispatch(int k, const uint8_t* b, int64_t kdim, int64_t n, const FieldConst& f, uint32_t lut,
                            uint8_t* bx, int64_t ldb, cudaStream_t s) {
    switch (k) {
        case 1: launch_expand_table<1, KIND>(b, kdim, n, f, lut, bx, ldb, s); break;
        case 2: launch_expand_table<2, KIND>(b, kdim, n, f, lut, bx, ldb, s); break;
        case 3: launch_expand_table<3, KIND>(b, kdim, n, f, lut, bx, ldb, s); break;
        default: launch_expand_table<4, KIND>(b, kdim, n, f, lut, bx, ldb, s); break;
    }
}

// C[m, n*k] = A[m, K*k] (x) expand(B)  (mod p)
static int run(int kind, const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
               void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    const int k = (int)f.k;
    Layout L = plan(kind, a, m, kdim, n, k);
    QADIC_REQUIRE(ws != nullptr && ws_bytes >= L.bx_bytes + L.a_bytes, QADIC_ERR_VALUE,
                  "workspace too small (%zu < %zu)", ws_bytes, L.bx_bytes + L.a_bytes);
    const uint32_t lut = kind == KIND_F4 ? e2m1_lut(f.p, kdim * k) : 0;
    uint8_t* bx = static_cast<uint8_t*>(ws);
    const uint8_t* a_op = a;
    if (L.prep_a) {
        uint8_t* ap = bx + L.bx_bytes;
        if (kind == KIND_F4) {
            const int64_t tot = m * (L.lda / 16);
            QADIC_TIMED("fp4 pack A", s,
                        pack_a_f4_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, m, L.Kb, lut, ap, L.lda));
        } else {
            const int64_t tot = m * L.lda;
            QADIC_TIMED("i8 pad A", s,
                        pad_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, m, L.Kb, ap, L.lda));
        }
        int rc = check_launch("tc prepare A");
        if (rc) return rc;
        a_op = ap;
    }
    int ncodes = 1;
    for (int s2 = 0; s2 < k; ++s2) ncodes *= (int)f.p;
    if (ncodes <= XT_CODES) {
        if (kind == KIND_I8) expand_dispatch<KIND_I8>(k, b, kdim, n, f, lut, bx, L.ldb, s);
        else expand_dispatch<KIND_F4>(k, b, kdim, n, f, lut, bx, L.ldb, s);
    } else {
        QADIC_REQUIRE(kind == KIND_I8, QADIC_ERR_UNSUPPORTED, "fp4 engine needs p^k <= %d", XT_CODES);
        dim3 grid((unsigned)((kdim + EX_T - 1) / EX_T), (unsigned)((n + EX_T - 1) / EX_T));
        QADIC_REQUIRE(grid.y <= 65535, QADIC_ERR_UNSUPPORTED, "n too large");
        QADIC_TIMED("expand B", s, expand_b_generic_kernel<<<grid, 256, 0, s>>>(b, kdim, n, f, bx, L.ldb));
    }
    int rc = check_launch("tc expand B");
    if (rc) return rc;
    const int BN = kind == KIND_I8 ? Cfg<KIND_I8>::BN : Cfg<KIND_F4>::BN;
    const bool pair = pair_mode();
    CUtensorMap ta, tb;
    rc = make_tmap(&ta, a_op, L.inner, m, L.lda, BM);
    if (rc) return rc;
    rc = make_tmap(&tb, bx, L.inner, n * k, L.ldb, pair ? BN / 2 : BN);
    if (rc) return rc;
    Params prm = {};
    prm.sf = e2m1_scale_word();
    prm.group_m = getenv("QADIC_GROUP_M") ? atoi(getenv("QADIC_GROUP_M")) : GROUP_M;
    if (prm.group_m < 1) prm.group_m = 1;
    prm.diag_noload = getenv_flag("QADIC_DIAG_NOLOAD");
    prm.M = m;
    prm.N = n * k;
    prm.ldc = n * k;
    prm.p = f.p;
    prm.offset = f.p * ((1u << 25) / f.p + 1);  // > |centred sum| (< 2^24), multiple of p
    prm.magic64 = wide_magic(f.p);
    // the light epilogue (32-bit reciprocal) where x * p < 2^32: F4 sums + offset < 2^26 (p <= 7), I8 sums
    // of non-negative residue bytes <= K k (p-1)^2
    if (kind == KIND_F4 ? ((uint64_t)f.p << 26) < (1ull << 32)
                        : (__int128)kdim * k * (f.p - 1) * (f.p - 1) * f.p < ((__int128)1 << 32))
        prm.magic32 = small_magic(f.p);
    prm.epi_mod64 = getenv_flag("QADIC_EPI_MOD64");
    prm.m_tiles = (int)((m + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM));
    prm.n_tiles = (int)((prm.N + BN - 1) / BN);
    prm.n_full = (int)(prm.N / BN);
    prm.num_kb = (int)((L.inner + BK - 1) / BK);
    prm.c = c;
    prm.c_plane = 0;
    prm.planes = 1;
    prm.nibble_out = 0;
    if (pair) return kind == KIND_I8 ? launch_gemm<KIND_I8, true>(ta, tb, prm, s) : launch_gemm<KIND_F4, true>(ta, tb, prm, s);
    return kind == KIND_I8 ? launch_gemm<KIND_I8, false>(ta, tb, prm, s) : launch_gemm<KIND_F4, false>(ta, tb, prm, s);
}

// ---------------------------------------------------------------------------
// Karatsuba planes (FP4 kind).  The S = k(k+1)/2 plane products
//     D_i = A_i B_i,    D_ij = (A_i + A_j)(B_i + B_j)   (i < j)
// of coefficient planes (operand sums reduced mod p, centred, E2M1) give all
// product coefficients P_t = sum_{i<j, i+j=t} (D_ij - D_i - D_j) + [t even] D_{t/2};
// with the field fold C_l = sum_t xpow[t][l] P_t this is ONE mod-p linear map
// C_l = sum_s W[l][s] D_s, applied by the combine kernel.  Every plane product
// is an ordinary M x N x K GEMM (inner dimension K, not K*k), so cfg5 (k = 3)
// runs 6 plane GEMMs where the expanded form runs 9: 1/3 fewer MACs.
// ---------------------------------------------------------------------------
// plane s: s < k -> single coefficient s; then the pairs (i, j), i < j, in
// lexicographic order (k <= 4).  Branch-only so unrolled indices fold.
__host__ __device__ constexpr int combo_first(int k, int s) {
    return s < k ? s : (k == 2 ? 0 : k == 3 ? (s <= 4 ? 0 : 1) : (s <= 6 ? 0 : s <= 8 ? 1 : 2));
}
__host__ __device__ constexpr int combo_second(int k, int s) {
    return s < k ? s
                 : (k == 2 ? 1
                           : k == 3 ? (s == 3 ? 1 : 2)
                                    : (s == 4 ? 1 : s == 5 ? 2 : s == 6 ? 3 : s == 7 ? 2 : 3));
}

constexpr int KMAX_S = 8;  // planes per product handled by the nibble transpose

// The plane products of one field: D_s = (sum_i E[s][i] a_i)(sum_i E[s][i] b_i)
// (all mod p), and C_l = sum_s W[l][s] D_s (mod p).
//   Toom-Cook over F_p when 2k-1 <= p+1: evaluation at 2k-1 distinct points of
//     F_p u {inf}, W = (X^t mod f) o Vandermonde^-1  -> S = 2k-1 planes
//     (cfg5, GF(7^3): 5 plane GEMMs where the expanded form does 9 products);
//   otherwise Karatsuba: D_i = a_i b_i, D_ij = (a_i + a_j)(b_i + b_j)
//     -> S = k(k+1)/2 planes (GF(3^3): 6).
struct PlaneSpec {
    int S;
    uint8_t E[KMAX_S][kMaxK];
    uint8_t W[kMaxK][KMAX_S];
};

static int64_t pmod(int64_t x, int64_t p) { return ((x % p) + p) % p; }
static int64_t ipow_mod(int64_t x, int e, int64_t p) {
    int64_t r = 1;
    for (int i = 0; i < e; ++i) r = r * x % p;
    return r;
}

// inverse of an n x n matrix over F_p (n <= 8); false if singular
static bool inv_mod_p(int n, int64_t (*a)[KMAX_S], int64_t (*out)[KMAX_S], int64_t p) {
    int64_t m[KMAX_S][2 * KMAX_S];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < 2 * n; ++j) m[i][j] = j < n ? pmod(a[i][j], p) : (j - n == i);
    for (int c = 0; c < n; ++c) {
        int piv = -1;
        for (int r = c; r < n; ++r)
            if (m[r][c]) { piv = r; break; }
        if (piv < 0) return false;
        for (int j = 0; j < 2 * n; ++j) { const int64_t t = m[c][j]; m[c][j] = m[piv][j]; m[piv][j] = t; }
        int64_t iv = 1;
        for (int64_t e = p - 2, b = m[c][c]; e; e >>= 1, b = b * b % p)
            if (e & 1) iv = iv * b % p;
        for (int j = 0; j < 2 * n; ++j) m[c][j] = m[c][j] * iv % p;
        for (int r = 0; r < n; ++r)
            if (r != c && m[r][c]) {
                const int64_t fct = m[r][c];
                for (int j = 0; j < 2 * n; ++j) m[r][j] = pmod(m[r][j] - fct * m[c][j], p);
            }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) out[i][j] = m[i][n + j];
    return true;
}

static bool plan_planes(const FieldConst& f, PlaneSpec* ps) {
    const int k = (int)f.k;
    const int64_t p = f.p;
    const int n = 2 * k - 1;
    *ps = PlaneSpec{};
    if (n <= p + 1) {  // Toom-Cook: points inf, 0, 1, -1, 2, -2, ...
        int64_t pts[KMAX_S];
        bool inf[KMAX_S] = {};
        int cnt = 0;
        inf[cnt++] = true;
        const int64_t cand[] = {0, 1, -1, 2, -2, 3, -3};
        for (int64_t c : cand) {
            if (cnt == n) break;
            const int64_t v = pmod(c, p);
            bool dup = false;
            for (int i = 1; i < cnt; ++i) dup |= (!inf[i] && pts[i] == v);
            if (!dup) pts[cnt++] = v;
        }
        if (cnt != n) return false;
        int64_t V[KMAX_S][KMAX_S] = {}, Vi[KMAX_S][KMAX_S] = {};
        for (int s = 0; s < n; ++s) {
            for (int i = 0; i < k; ++i) ps->E[s][i] = (uint8_t)(inf[s] ? (i == k - 1) : ipow_mod(pts[s], i, p));
            for (int t = 0; t < n; ++t) V[s][t] = inf[s] ? (t == n - 1) : ipow_mod(pts[s], t, p);
        }
        if (!inv_mod_p(n, V, Vi, p)) return false;
        for (int l = 0; l < k; ++l)
            for (int s = 0; s < n; ++s) {
                int64_t acc = 0;
                for (int t = 0; t < n; ++t) acc += (int64_t)f.xpow[t][l] * Vi[t][s];
                ps->W[l][s] = (uint8_t)pmod(acc, p);
            }
        ps->S = n;
        return true;
    }
    const int S = k * (k + 1) / 2;
    if (S > KMAX_S) return false;
    for (int s = 0; s < S; ++s) {
        const int i = combo_first(k, s), j = combo_second(k, s);
        ps->E[s][i] = 1;
        ps->E[s][j] = 1;
        for (int l = 0; l < k; ++l) {
            int64_t acc = 0;
            if (i == j) {
                acc += f.xpow[2 * i][l];
                for (int o = 0; o < k; ++o)
                    if (o != i) acc -= f.xpow[i + o][l];
            } else {
                acc += f.xpow[i + j][l];
            }
            ps->W[l][s] = (uint8_t)pmod(acc, p);
        }
    }
    ps->S = S;
    return true;
}

// T[code] = E2M1 nibble of plane s of the element with this code, at bit 4s

// The plane table built inside the B-plane kernels (each block into its own
// shared memory; block 0 also publishes it for the A-plane kernel that follows
// on the stream) -- saves the separate table launch.
__device__ __forceinline__ void build_plane_table(uint32_t* tab, uint32_t p, int k, int S, const PlaneSpec& ps,
                                                  uint32_t lut, uint32_t* __restrict__ gout) {
    int ncodes = 1;
    for (int i = 0; i < k; ++i) ncodes *= (int)p;
    for (int c = threadIdx.x; c < ncodes; c += blockDim.x) {
        int r = c;
        uint32_t dig[kMaxK] = {};
        for (int i = 0; i < k; ++i) {
            dig[i] = (uint32_t)(r % (int)p);
            r /= (int)p;
        }
        uint32_t w = 0;
        for (int s = 0; s < S; ++s) {
            uint32_t v = 0;
            for (int i = 0; i < k; ++i) v += ps.E[s][i] * dig[i];
            w |= ((lut >> (4 * (v % p))) & 0xF) << (4 * s);
        }
        tab[c] = w;
        if (blockIdx.x == 0) gout[c] = w;
    }
}

// 4 byte lanes (values < 16) -> 16-bit field of 4 nibbles
__device__ __forceinline__ uint32_t bytes_to_nibbles(uint32_t v) {
    const uint32_t x = v | (v >> 4);
    return __byte_perm(x, 0, 0x0020) & 0xFFFFu;
}
// k = 1 (a single plane): 4 residues (< 8) -> 4 E2M1 nibbles by one PRMT table lookup
__device__ __forceinline__ uint32_t residues_to_e2m1(uint32_t v, uint32_t lut_lo, uint32_t lut_hi) {
    return bytes_to_nibbles(__byte_perm(lut_lo, lut_hi, bytes_to_nibbles(v)));
}
__device__ __forceinline__ void byte_lut_from_table(const uint32_t* tab, uint32_t p, uint32_t& lo, uint32_t& hi) {
    lo = hi = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        lo |= ((uint32_t)v < p ? (tab[v] & 0xF) : 0u) << (8 * v);
        hi |= ((uint32_t)(v + 4) < p ? (tab[v + 4] & 0xF) : 0u) << (8 * v);
    }
}

// 8 x 8 transpose of 4-bit cells: on return nibble e of x[s] = old nibble s of x[e]
// 8 words x 8 nibbles -> transposed (word s = nibble s of the 8 inputs):
// 16-bit and 8-bit stages are byte permutes, the 4-bit stage two SHF+LOP3 pairs.
__device__ __forceinline__ void transpose8_nibbles(uint32_t (&x)[8]) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t a = x[r], b = x[r + 4];
        x[r] = __byte_perm(a, b, 0x5410);
        x[r + 4] = __byte_perm(a, b, 0x7632);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
        if ((r & 2) == 0) {
            const uint32_t a = x[r], b = x[r + 2];
            x[r] = __byte_perm(a, b, 0x6240);
            x[r + 2] = __byte_perm(a, b, 0x7351);
        }
#pragma unroll
    for (int r = 0; r < 8; r += 2) {
        const uint32_t a = x[r], b = x[r + 1];
        x[r] = (a & 0x0F0F0F0Fu) | ((b << 4) & 0xF0F0F0F0u);
        x[r + 1] = ((a >> 4) & 0x0F0F0F0Fu) | (b & 0xF0F0F0F0u);
    }
}

// Element codes sum_i p^i b_i of K-byte elements packed back to back in 32-bit
// words, by byte dot products: an element at byte offset o of word w is
// dp4a(w, A[o]) (+ dp4a(w+1, B[o]) when it straddles), A/B holding p^i in the
// element's byte slots.  K = 4 (word aligned) keeps p^3 (up to 343) out of the
// byte weights: dp4a(w, [1, p, p^2, 0]) + p^3 * (w >> 24).
template <int K>
struct CodeCoef {
    uint32_t a[4], b[4], p3;
};
template <int K>
__device__ __forceinline__ CodeCoef<K> make_code_coef(uint32_t p) {
    CodeCoef<K> c;
    uint32_t pw[4] = {1, p, p * p, p * p * p};
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        c.a[o] = c.b[o] = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (K == 4 && i == 3) continue;
            if (o + i < 4) c.a[o] |= pw[i] << (8 * (o + i));
            else c.b[o] |= pw[i] << (8 * (o + i - 4));
        }
    }
    c.p3 = pw[3];
    return c;
}
template <int K, int E, int NW>
__device__ __forceinline__ uint32_t elem_code(const uint32_t (&w)[NW], const CodeCoef<K>& c) {
    constexpr int off = E * K, wi = off >> 2, o = off & 3;
    uint32_t code = __dp4a(w[wi], c.a[o], 0u);
    if constexpr (K == 4) code += c.p3 * (w[wi] >> 24);
    if constexpr (o + K > 4 && K != 4) code = __dp4a(w[wi + 1], c.b[o], code);
    return code;
}
template <int K, int NW, int... Es>
__device__ __forceinline__ void elem_codes_seq(const uint32_t (&w)[NW], const CodeCoef<K>& c, uint32_t* out,
                                               std::integer_sequence<int, Es...>) {
    ((out[Es] = elem_code<K, Es>(w, c)), ...);
}
// codes of the NE = 4 * NW / K elements held in w[]
template <int K, int NW>
__device__ __forceinline__ void elem_codes(const uint32_t (&w)[NW], const CodeCoef<K>& c, uint32_t* out) {
    elem_codes_seq<K, NW>(w, c, out, std::make_integer_sequence<int, 4 * NW / K>{});
}

constexpr int PT_CODES = 1024;

// Rows [R, Kd, K] of residues -> S planes [S][R][ld] of packed E2M1 nibbles.
// Thread: one row, 32 consecutive kk.  Per element one shared-memory table
// lookup yields all S plane nibbles; an 8x8 nibble transpose turns 8
// elements' lookups into the 8 plane words.
// resident blocks per SM asked of the compiler: 6 (40 registers, 16 B of spills) measured 0.0457 vs
// 0.0494 ms at cfg3 and 0.067 vs 0.068 at cfg5 against the unconstrained 48 registers / 5 blocks; 7-8
// (32 registers, 148 B of spills) 0.098 ms
#ifndef QADIC_PA_MINB
#define QADIC_PA_MINB 6
#endif
template <int K>
__global__ void __launch_bounds__(256, (K <= 3 ? QADIC_PA_MINB : 5)) planes_kernel(const uint8_t* __restrict__ src, int64_t R, int64_t Kd, uint32_t p,
                                                     const uint32_t* __restrict__ gtab, int S,
                                                     uint8_t* __restrict__ out, int64_t ld, int64_t plane_stride) {

    __shared__ uint32_t tab[PT_CODES];
    const int64_t chunks = ld / 16;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = idx < R * chunks;
    const int64_t r = live ? idx / chunks : 0, q = live ? idx % chunks : 0;
    const int64_t kk0 = q * 32;
    const uint8_t* row = src + (r * Kd + kk0) * K;
    // the row's loads go out first; the plane table is staged while they are in flight
    uint32_t in[8 * K];
    if (live && kk0 + 32 <= Kd && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
        for (int v = 0; v < 2 * K; ++v) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(row) + v);
            in[4 * v] = x.x; in[4 * v + 1] = x.y; in[4 * v + 2] = x.z; in[4 * v + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int v = 0; v < 8 * K; ++v) in[v] = 0;
        if (live)
#pragma unroll
            for (int e = 0; e < 32 * K; ++e)
                if (kk0 + e / K < Kd) in[e >> 2] |= (uint32_t)row[e] << (8 * (e & 3));
    }
    int ncodes = 1;
    for (int i = 0; i < K; ++i) ncodes *= (int)p;
    for (int i = threadIdx.x; i < ncodes; i += blockDim.x) tab[i] = gtab[i];
    __syncthreads();
    if (!live) return;
    if constexpr (K == 1) {  // one plane: 4 residues per PRMT lookup
        uint32_t lo, hi;
        byte_lut_from_table(tab, p, lo, hi);
        uint32_t o[4];
#pragma unroll
        for (int g = 0; g < 4; ++g)
            o[g] = residues_to_e2m1(in[2 * g], lo, hi) | (residues_to_e2m1(in[2 * g + 1], lo, hi) << 16);
        *reinterpret_cast<uint4*>(out + r * ld + q * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        return;
    }
    uint32_t w[KMAX_S][4];
    uint32_t code[32];
    elem_codes<K, 8 * K>(in, make_code_coef<K>(p), code);
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // 8 elements per group
        uint32_t x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = tab[code[8 * g + e]];
        transpose8_nibbles(x);
#pragma unroll
        for (int s = 0; s < KMAX_S; ++s) w[s][g] = x[s];
    }
    uint8_t* dst = out + r * ld + q * 16;
#pragma unroll
    for (int s = 0; s < KMAX_S; ++s)
        if (s < S) *reinterpret_cast<uint4*>(dst + s * plane_stride) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

// B [Kd, N, K] -> S transposed planes [S][N][ld], two passes per 256 kk x 32 j tile:
//  1. a warp reads 4 B-row segments per instruction (a lane = 4 consecutive
//     elements = K aligned 32-bit words), forms the 4 element codes (sum_i p^i b_i,
//     byte dot products) and stores them (8 bytes) into a [kk][j] uint16 tile
//     whose 4-column chunks are XOR-swizzled by kk/32, so that pass 2 reads it
//     without bank conflicts;
//  2. lane = (32-kk chunk, j): plane-table lookup of 8 codes per plane word,
//     8x8 nibble transpose, S 16-byte stores -- every store instruction writes
//     4 rows x 128 contiguous bytes of each plane (whole lines, no partial sectors).
// planes_b3_kernel feeds pass 1 by TMA; planes_b2_kernel (unaligned B) by lane loads.
constexpr int P2_KK = 256, P2_J = 32;
#ifndef QADIC_P2_NBUF
#define QADIC_P2_NBUF 2
#endif
constexpr int P2_NBUF = QADIC_P2_NBUF;  // TMA input buffers of planes_b3_kernel (NBUF - 1 tiles in flight;
                                        // 3 and 4 measured slower: fewer resident blocks)

// pass 2 of the B-plane kernels: lane = (32-kk chunk, column) of the code tile
template <int K>
__device__ __forceinline__ void planes_b_pass2(const uint16_t (*codes)[P2_J], const uint32_t* tab, uint32_t lo,
                                               uint32_t hi, int64_t j0, int64_t kk0, int64_t N, int64_t ld,
                                               int64_t plane_stride, int S, uint8_t* __restrict__ out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kc = lane & 7, jl = 4 * warp + (lane >> 3);
    const int64_t gj = j0 + jl;
    const int64_t col = (kk0 + kc * 32) / 2;
    const int cidx = 4 * ((jl >> 2) ^ kc) + (jl & 3);  // swizzled column in rows 32kc .. 32kc+31
    if (gj < N && col + 16 <= ld) {
        if constexpr (K == 1) {
            uint32_t o[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t c[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) c[e] = codes[kc * 32 + 8 * g + e][cidx];
                const uint32_t v0 = __byte_perm(c[0] | (c[1] << 16), c[2] | (c[3] << 16), 0x6420);
                const uint32_t v1 = __byte_perm(c[4] | (c[5] << 16), c[6] | (c[7] << 16), 0x6420);
                o[g] = residues_to_e2m1(v0, lo, hi) | (residues_to_e2m1(v1, lo, hi) << 16);
            }
            *reinterpret_cast<uint4*>(out + gj * ld + col) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
            uint32_t w[KMAX_S][4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t x[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) x[e] = tab[codes[kc * 32 + 8 * g + e][cidx]];
                transpose8_nibbles(x);
#pragma unroll
                for (int s = 0; s < KMAX_S; ++s) w[s][g] = x[s];
            }
            uint8_t* dst = out + gj * ld + col;
#pragma unroll
            for (int s = 0; s < KMAX_S; ++s)
                if (s < S)
                    *reinterpret_cast<uint4*>(dst + s * plane_stride) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
        }
    }
}

template <int K>
__global__ void __launch_bounds__(256) planes_b2_kernel(const uint8_t* __restrict__ b, int64_t Kd, int64_t N,
                                                        uint32_t p, uint32_t* __restrict__ gtab, PlaneSpec ps, uint32_t lut, int S,
                                                        uint8_t* __restrict__ out, int64_t ld, int64_t plane_stride,
                                                        int tiles_kk, int tiles_j) {

    __shared__ __align__(16) uint16_t codes[P2_KK][P2_J];
    __shared__ uint32_t tab[PT_CODES];
    build_plane_table(tab, p, K, S, ps, lut, gtab);
    const CodeCoef<K> cc = make_code_coef<K>(p);
    const bool vec = ((N * K) % 4 == 0) && ((reinterpret_cast<uintptr_t>(b) & 3) == 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r4 = lane >> 3, c8 = lane & 7;  // pass 1: row of the warp's 4, 4-element chunk
    uint32_t lo = 0, hi = 0;
    if (K == 1) {
        __syncthreads();
        byte_lut_from_table(tab, p, lo, hi);
    }
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t kk0 = (t % tiles_kk) * P2_KK, j0 = (t / tiles_kk) * P2_J;
        // ---- pass 1: codes ----
        const int64_t jj = j0 + 4 * c8;
        constexpr int ROUNDS = P2_KK / 32;  // 8 warps x 4 rows per round
        uint32_t wv[ROUNDS][K];
        if (vec && kk0 + P2_KK <= Kd && j0 + P2_J <= N) {  // whole tile in range: all loads in flight at once
            const uint32_t* src = reinterpret_cast<const uint32_t*>(b + ((kk0 + 4 * warp + r4) * N + jj) * K);
            const int64_t rstride = 8 * N * K;  // 32 rows, in 32-bit words
#pragma unroll
            for (int r = 0; r < ROUNDS; ++r)
#pragma unroll
                for (int i = 0; i < K; ++i) wv[r][i] = __ldg(src + r * rstride + i);
        } else
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int64_t gk = kk0 + 32 * r + 4 * warp + r4;
            const uint8_t* src = b + (gk * N + jj) * K;
            if (vec && gk < Kd && jj + 4 <= N) {
#pragma unroll
                for (int i = 0; i < K; ++i) wv[r][i] = __ldg(reinterpret_cast<const uint32_t*>(src) + i);
            } else {
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    uint32_t w = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = (4 * i + q) / K;  // element within the 4
                        if (gk < Kd && jj + e < N) w |= (uint32_t)src[4 * i + q] << (8 * q);
                    }
                    wv[r][i] = w;
                }
            }
        }
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            uint32_t cd[4];
            elem_codes<K, K>(wv[r], cc, cd);
            const int row = 32 * r + 4 * warp + r4;  // row >> 5 == r
            *reinterpret_cast<uint2*>(&codes[row][4 * (c8 ^ (r & 7))]) =
                make_uint2(__byte_perm(cd[0], cd[1], 0x5410), __byte_perm(cd[2], cd[3], 0x5410));
        }
        __syncthreads();
        // ---- pass 2: planes ----
        planes_b_pass2<K>(codes, tab, lo, hi, j0, kk0, N, ld, plane_stride, S, out);
        __syncthreads();  // the code tile is rewritten by the next tile's pass 1
    }
}

// TMA-fed variant of planes_b2_kernel: the 256 kk x (32 j * K bytes) input box
// of the next tile streams into shared memory (cp.async.bulk.tensor, zero fill
// outside B) while the current tile is converted, so the strided B rows are
// fetched by the copy engine in whole sectors instead of 4-byte lane loads.
#ifndef QADIC_P2_MINB
#define QADIC_P2_MINB 1
#endif
template <int K>
__global__ void __launch_bounds__(256, QADIC_P2_MINB) planes_b3_kernel(const __grid_constant__ CUtensorMap tmap, int64_t Kd,
                                                        int64_t N, uint32_t p, uint32_t* __restrict__ gtab, PlaneSpec ps, uint32_t lut,
                                                        int S, uint8_t* __restrict__ out, int64_t ld,
                                                        int64_t plane_stride, int tiles_kk, int tiles_j, int jmajor) {

    using namespace sm100;
    constexpr int ROWB = P2_J * K;  // bytes per box row
    extern __shared__ __align__(128) uint8_t dsm3[];
    uint8_t* inb = dsm3;                                                     // 2 x [P2_KK][ROWB]
    constexpr int NB = P2_NBUF;
    uint16_t (*codes)[P2_J] = reinterpret_cast<uint16_t (*)[P2_J]>(dsm3 + NB * P2_KK * ROWB);
    uint32_t* tab = reinterpret_cast<uint32_t*>(dsm3 + NB * P2_KK * ROWB + P2_KK * P2_J * 2);
    __shared__ __align__(8) uint64_t bar[NB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r4 = lane >> 3, c8 = lane & 7;
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    // tile t -> (kk0, j0): kk fastest (concurrent blocks write adjacent plane columns of
    // the same rows) or, jmajor, j fastest (concurrent blocks read adjacent 96-byte
    // segments of the same B rows)
    auto tile_of = [&](int64_t t, int64_t& kk0, int64_t& j0) {
        if (jmajor) {
            kk0 = (t / tiles_j) * P2_KK;
            j0 = (t % tiles_j) * P2_J;
        } else {
            kk0 = (t % tiles_kk) * P2_KK;
            j0 = (t / tiles_kk) * P2_J;
        }
    };
    auto issue = [&](int64_t t, int buf) {
        int64_t kk0, j0;
        tile_of(t, kk0, j0);
        mbar_arrive_expect_tx(&bar[buf], P2_KK * ROWB);
        tma_load_2d(inb + buf * P2_KK * ROWB, &tmap, &bar[buf], (int32_t)(j0 * K), (int32_t)kk0);
    };
    // the first tiles' loads go out before the plane table is built (the other
    // threads wait on the barriers only after the __syncthreads below)
    if (threadIdx.x == 0) {
        tma_prefetch(&tmap);
        for (int i = 0; i < NB; ++i) mbar_init(&bar[i], 1);
        fence_barrier_init();
        for (int i = 0; i < (NB > 1 ? NB - 1 : 1); ++i)
            if ((int64_t)blockIdx.x + (int64_t)i * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)i * gridDim.x, i);
    }
    build_plane_table(tab, p, K, S, ps, lut, gtab);
    const CodeCoef<K> cc = make_code_coef<K>(p);
    __syncthreads();
    uint32_t lo = 0, hi = 0;
    if (K == 1) byte_lut_from_table(tab, p, lo, hi);
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int buf = it % NB;
        // the other buffer was last read in the previous iteration's pass 1 (fenced by its barrier)
        // NB - 1 tiles in flight; the buffer refilled here was last read in the previous
        // iteration's pass 1 (fenced by its barriers)
        const int64_t tn = t + (int64_t)(NB > 1 ? NB - 1 : 1) * gridDim.x;
        if (NB > 1 && threadIdx.x == 0 && tn < ntiles) issue(tn, (it + NB - 1) % NB);
        mbar_wait(&bar[buf], (uint32_t)((it / NB) & 1));
        int64_t kk0, j0;
        tile_of(t, kk0, j0);
        const uint8_t* tb = inb + buf * P2_KK * ROWB;
#pragma unroll
        for (int r = 0; r < P2_KK / 32; ++r) {
            const int row = 32 * r + 4 * warp + r4;
            uint32_t w[K];
#pragma unroll
            for (int i = 0; i < K; ++i) w[i] = reinterpret_cast<const uint32_t*>(tb + row * ROWB + 4 * K * c8)[i];
            uint32_t cd[4];
            elem_codes<K, K>(w, cc, cd);
            *reinterpret_cast<uint2*>(&codes[row][4 * (c8 ^ (r & 7))]) =
                make_uint2(__byte_perm(cd[0], cd[1], 0x5410), __byte_perm(cd[2], cd[3], 0x5410));
        }
        __syncthreads();
        // one input buffer: pass 1 has consumed it, the next tile streams in during pass 2
        if (NB == 1 && threadIdx.x == 0 && tn < ntiles) issue(tn, 0);
        planes_b_pass2<K>(codes, tab, lo, hi, j0, kk0, N, ld, plane_stride, S, out);
        __syncthreads();  // code tile rewritten next iteration
    }
}

// K = 1 (one plane, cfg4): B [Kd][N] residues -> E2M1 nibbles [N][ld], transposed.
// Tile 128 kk x 128 j: a thread reads four 16-byte row vectors (the next tile's are
// loaded during this tile's pass 2), scatters them j-major into shared memory
// (16-byte chunks XOR-swizzled by j / 16, so a warp's byte stores hit 8 distinct
// bank quads), then thread (j, g) turns 16 kk into 8 nibble bytes (one 16-byte
// shared read, four PRMT lookups).  The 16-byte-per-row segments of pass 1 are
// what the K = 1 tile of planes_b3 (32-byte rows) lacked.
constexpr int B1_KK = 128, B1_J = 128;
__global__ void __launch_bounds__(256) planes_b1_kernel(const uint8_t* __restrict__ b, int64_t Kd, int64_t N,
                                                        uint32_t p, uint32_t* __restrict__ gtab, PlaneSpec ps,
                                                        uint32_t lut, uint8_t* __restrict__ out, int64_t ld,
                                                        int tiles_kk, int tiles_j) {
    __shared__ uint32_t tab[PT_CODES];
    __shared__ __align__(16) uint8_t res[B1_J][B1_KK];
    const bool vec = (N % 16 == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    uint4 w[4];
    auto load = [&](int64_t t) {
        const int64_t kk0 = (t % tiles_kk) * B1_KK, j0 = (t / tiles_kk) * B1_J;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = threadIdx.x + 256 * q, row = c >> 3, cc = c & 7;
            const int64_t gk = kk0 + row, gj = j0 + 16 * cc;
            if (vec && gk < Kd && gj + 16 <= N) {
                w[q] = __ldg(reinterpret_cast<const uint4*>(b + gk * N + gj));
            } else {
                uint32_t x[4] = {0, 0, 0, 0};
                for (int e = 0; e < 16; ++e)
                    if (gk < Kd && gj + e < N) x[e >> 2] |= (uint32_t)b[gk * N + gj + e] << (8 * (e & 3));
                w[q] = make_uint4(x[0], x[1], x[2], x[3]);
            }
        }
    };
    if ((int64_t)blockIdx.x < ntiles) load(blockIdx.x);
    build_plane_table(tab, p, 1, 1, ps, lut, gtab);
    __syncthreads();
    uint32_t lo, hi;
    byte_lut_from_table(tab, p, lo, hi);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t kk0 = (t % tiles_kk) * B1_KK, j0 = (t / tiles_kk) * B1_J;
        __syncthreads();  // previous tile's residues consumed
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = threadIdx.x + 256 * q, row = c >> 3, cc = c & 7;
            const int col = ((((row >> 4) ^ cc) & 7) << 4) | (row & 15);  // swizzled kk position
            const uint32_t x[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
            for (int e = 0; e < 16; ++e) res[16 * cc + e][col] = (uint8_t)(x[e >> 2] >> (8 * (e & 3)));
        }
        __syncthreads();
        if (t + gridDim.x < ntiles) load(t + gridDim.x);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int item = threadIdx.x + 256 * q, j = item >> 3, g = item & 7;
            const int64_t gj = j0 + j, col = (kk0 + 16 * g) / 2;
            if (gj < N && col < ld) {
                const uint4 r = *reinterpret_cast<const uint4*>(&res[j][(g ^ ((j >> 4) & 7)) << 4]);
                const uint32_t o0 = residues_to_e2m1(r.x, lo, hi) | (residues_to_e2m1(r.y, lo, hi) << 16);
                const uint32_t o1 = residues_to_e2m1(r.z, lo, hi) | (residues_to_e2m1(r.w, lo, hi) << 16);
                *reinterpret_cast<uint2*>(out + gj * ld + col) = make_uint2(o0, o1);
            }
        }
    }
}

static int b3_jmajor() {
    static const int v = getenv("QADIC_B3_JMAJOR") ? atoi(getenv("QADIC_B3_JMAJOR")) : 1;  // measured 0.081 vs 0.083 ms (cfg5)
    return v;
}

template <int K>
constexpr size_t planes_b3_smem() {
    return (size_t)P2_NBUF * P2_KK * P2_J * K + (size_t)P2_KK * P2_J * 2 + PT_CODES * sizeof(uint32_t) + 128;
}

static int make_tmap_rows(CUtensorMap* map, const void* base, int64_t inner_bytes, int64_t rows, int64_t ld,
                          uint32_t box_inner, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    QADIC_REQUIRE(fn != nullptr, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)inner_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QADIC_REQUIRE(r == CUDA_SUCCESS, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return QADIC_OK;
}

// D planes [S][M][ldd] (nibbles, N columns) -> C [M][N][K] uint8 residues.
// Thread: one row, 32 consecutive columns.  The even and odd columns of a
// plane word are split into byte lanes (x & 0x0F0F0F0F, (x >> 4) & ...) and the
// weighted plane sum runs on 4 lanes at once (<= 6 terms of <= 36 per pass,
// < 256), then each lane is reduced mod p.
template <int K>
__global__ void __launch_bounds__(256) combine_kernel(const uint8_t* __restrict__ d, int64_t M, int64_t N, int64_t ldd,
                                                      int64_t plane_stride, int S, uint32_t p, uint32_t magic,
                                                      PlaneSpec ps, uint8_t* __restrict__ c) {
    const int64_t chunks = (N + 31) / 32;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= M * chunks) return;
    const int64_t m = idx / chunks, q = idx % chunks;
    const int64_t j0 = q * 32;
    uint32_t dv[KMAX_S][4];
#pragma unroll
    for (int s = 0; s < KMAX_S; ++s) {
        if (s < S) {
            const uint4 x = *reinterpret_cast<const uint4*>(d + s * plane_stride + m * ldd + j0 / 2);
            dv[s][0] = x.x; dv[s][1] = x.y; dv[s][2] = x.z; dv[s][3] = x.w;
        } else {
            dv[s][0] = dv[s][1] = dv[s][2] = dv[s][3] = 0;
        }
    }
    uint32_t o[8 * K];
#pragma unroll
    for (int v = 0; v < 8 * K; ++v) o[v] = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // one plane word = 8 columns
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // even / odd columns
#pragma unroll
            for (int l = 0; l < K; ++l) {
                uint32_t tot[4] = {0, 0, 0, 0};
#pragma unroll
                for (int s0 = 0; s0 < KMAX_S; s0 += 6) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int s = s0; s < KMAX_S && s < s0 + 6; ++s)
                        acc += ((dv[s][g] >> (4 * half)) & 0x0F0F0F0Fu) * ps.W[l][s];
#pragma unroll
                    for (int e = 0; e < 4; ++e) tot[e] += (acc >> (8 * e)) & 0xFF;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = 8 * g + 2 * e + half;  // column within the 32-column chunk
                    const int pos = col * K + l;
                    o[pos >> 2] |= mod_small(tot[e], p, magic) << (8 * (pos & 3));
                }
            }
        }
    }
    uint8_t* dst = c + (m * N + j0) * K;
    if (j0 + 32 <= N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int v = 0; v < 2 * K; ++v)
            reinterpret_cast<uint4*>(dst)[v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    } else {
#pragma unroll
        for (int e = 0; e < 32 * K; ++e)
            if (j0 + e / K < N) dst[e] = (uint8_t)(o[e >> 2] >> (8 * (e & 3)));
    }
}

// T[l] lanes = columns c0..c3 of coefficient l -> out[w] = bytes 4w..4w+3 of the
// coefficient-minor stream (column-major over l)
template <int K>
__device__ __forceinline__ void place_coeffs(const uint32_t* T, uint32_t* out) {
    if constexpr (K == 2) {
        out[0] = __byte_perm(T[0], T[1], 0x5140);
        out[1] = __byte_perm(T[0], T[1], 0x7362);
    } else if constexpr (K == 3) {
        out[0] = __byte_perm(__byte_perm(T[0], T[1], 0x1040), T[2], 0x3410);
        out[1] = __byte_perm(__byte_perm(T[1], T[0], 0x2601), T[2], 0x3250);
        out[2] = __byte_perm(__byte_perm(T[2], T[0], 0x3072), T[1], 0x3710);
    } else {
#pragma unroll
        for (int w = 0; w < K; ++w) {
            uint32_t r = 0;
#pragma unroll
            for (int bi = 0; bi < 4; ++bi) {
                const int b = 4 * w + bi, col = b / K, l = b % K;
                r |= ((T[l] >> (8 * col)) & 0xFFu) << (8 * bi);
            }
            out[w] = r;
        }
    }
}

// 5 resident blocks per SM (48 registers, no spills): 0.064 vs 0.070 ms at cfg5 for 4 blocks (63
// registers); 6 (40 registers) 0.067, 8 (32 registers, spills) 0.084 ms
#ifndef QADIC_COMBINE_MINB
#define QADIC_COMBINE_MINB 5
#endif
template <int K, int S>
__global__ void __launch_bounds__(256, (K <= 3 ? QADIC_COMBINE_MINB : 4)) combine_swar_kernel(const uint8_t* __restrict__ d, int64_t M, int64_t N,
                                                           int64_t ldd, int64_t plane_stride, uint32_t p,
                                                           LaneDiv ld, PlaneSpec ps, uint8_t* __restrict__ c, int st256) {

    const int64_t chunks = (N + 31) / 32;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = idx < M * chunks;
    if (__all_sync(0xffffffffu, !live)) return;
    if (!live) idx = M * chunks - 1;  // duplicate the last chunk (identical bytes, warp stays converged)
    const int64_t m = idx / chunks, q = idx % chunks;
    const int64_t j0 = q * 32;
    uint32_t dv[S][4];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint4 x = __ldcs(reinterpret_cast<const uint4*>(d + s * plane_stride + m * ldd + j0 / 2));
        dv[s][0] = x.x; dv[s][1] = x.y; dv[s][2] = x.z; dv[s][3] = x.w;
    }
    uint32_t o[8 * K];
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // one plane word = 8 columns (nibbles; even / odd columns -> byte lanes)
        uint32_t lo[K], hi[K];
#pragma unroll
        for (int l = 0; l < K; ++l) {
            uint32_t ev = 0, od = 0;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t w = ps.W[l][s];
                ev += (dv[s][g] & 0x0F0F0F0Fu) * w;
                od += ((dv[s][g] >> 4) & 0x0F0F0F0Fu) * w;
            }
            ev = lanes_mod_div(ev, p, ld);
            od = lanes_mod_div(od, p, ld);
            lo[l] = __byte_perm(ev, od, 0x5140);  // columns 0..3 of this word
            hi[l] = __byte_perm(ev, od, 0x7362);  // columns 4..7
        }
        place_coeffs<K>(lo, o + g * 2 * K);
        place_coeffs<K>(hi, o + g * 2 * K + K);
    }
    uint8_t* dst = c + (m * N + j0) * K;
    // a warp whose 32 chunks are whole and contiguous (same row) stages its
    // 32 x 32K output bytes in shared memory and stores them as lane-consecutive
    // 16-byte vectors (each thread's own 32K bytes would be a 32K-byte-strided,
    // partial-line store pattern)
    __shared__ __align__(16) uint32_t cstage[256 / 32][32 * 8 * K];
    const int lane = threadIdx.x & 31;
    const bool whole = live && j0 + 32 <= N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    const int64_t m_lane0 = __shfl_sync(0xffffffffu, m, 0);
    if (__all_sync(0xffffffffu, whole && m == m_lane0 && N % 32 == 0)) {
        uint32_t* st = cstage[threadIdx.x >> 5];
#pragma unroll
        for (int v = 0; v < 2 * K; ++v)
            *reinterpret_cast<uint4*>(st + lane * 8 * K + 4 * v) =
                make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
        __syncwarp();
        uint4* wdst = reinterpret_cast<uint4*>(dst - (int64_t)lane * 32 * K);  // the warp's first chunk
        if (st256 && (reinterpret_cast<uintptr_t>(wdst) & 31) == 0) {  // 32-byte stores: 1 KB per warp instruction
#pragma unroll
            for (int v = 0; v < K; ++v) {
                const uint4 x0 = *reinterpret_cast<const uint4*>(st + (v * 32 + lane) * 8);
                const uint4 x1 = *reinterpret_cast<const uint4*>(st + (v * 32 + lane) * 8 + 4);
                asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(wdst + 2 * (v * 32 + lane)),
                             "r"(x0.x), "r"(x0.y), "r"(x0.z), "r"(x0.w), "r"(x1.x), "r"(x1.y), "r"(x1.z), "r"(x1.w)
                             : "memory");
            }
        } else {
#pragma unroll
            for (int v = 0; v < 2 * K; ++v)
                __stcs(wdst + v * 32 + lane, *reinterpret_cast<const uint4*>(st + (v * 32 + lane) * 4));
        }
    } else if (!live) {
        return;
    } else if (j0 + 32 <= N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int v = 0; v < 2 * K; ++v)
            reinterpret_cast<uint4*>(dst)[v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    } else {
#pragma unroll
        for (int e = 0; e < 32 * K; ++e)
            if (j0 + e / K < N) dst[e] = (uint8_t)(o[e >> 2] >> (8 * (e & 3)));
    }
}

// exact per-16-bit-lane division by p for lane values <= xmax (false: none found)
static bool lane_div_plan(uint32_t p, uint32_t xmax, LaneDiv* d) {
    for (uint32_t sh = 4; sh <= 15; ++sh) {
        const uint32_t m = ((1u << sh) + p - 1) / p;  // ceil(2^sh / p)
        if ((uint64_t)xmax * m >= 65536) break;
        const uint32_t qmax = xmax / p;
        if (qmax >= (1u << (16 - sh))) continue;  // quotient must stay below the spill-in bits
        bool ok = true;
        for (uint32_t x = 0; x <= xmax && ok; ++x) ok = ((x * m) >> sh) == x / p;
        if (ok) {
            d->m = m;
            d->sh = sh;
            d->qmask = ((1u << (16 - sh)) - 1) * 0x00010001u;
            return true;
        }
    }
    return false;
}

struct KaraLayout {
    int S;
    int64_t ldk;   // bytes per plane row of A_s / B_s (packed K)
    int64_t ldd;   // bytes per plane row of D_s (packed N)
    size_t tab_bytes, a_bytes, b_bytes, d_bytes;
};

static KaraLayout kara_plan(int S, int64_t m, int64_t kdim, int64_t n, int k) {
    KaraLayout L;
    L.S = S;
    L.ldk = round_up((kdim + 1) / 2, 16);
    L.ldd = round_up((n + 1) / 2, 16);
    L.tab_bytes = PT_CODES * sizeof(uint32_t);
    L.a_bytes = (size_t)round_up(L.S * m * L.ldk, 1024);
    L.b_bytes = (size_t)round_up(L.S * n * L.ldk, 1024);
    L.d_bytes = k == 1 ? 0 : (size_t)round_up(L.S * m * L.ldd, 1024);
    return L;
}

// B planes (which also build the plane table: smem per block, global for the
// A kernel) then A planes, in stream order.  b == nullptr: the B planes and the
// table are already in the workspace (later row panels of a host call).
template <int K>
static void launch_planes(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p,
                          uint32_t* tab, const PlaneSpec& ps, uint32_t lut, const KaraLayout& L, uint8_t* as,
                          uint8_t* bs, cudaStream_t s) {
    if (b != nullptr) {
        const int tk = (int)((kdim + P2_KK - 1) / P2_KK), tj = (int)((n + P2_J - 1) / P2_J);
        const int64_t tiles = (int64_t)tk * tj;
        CUtensorMap tm;
        const bool use_tma = ((n * K) % 16 == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0) &&
                             make_tmap_rows(&tm, b, n * K, kdim, n * K, P2_J * K, P2_KK) == QADIC_OK;
        if (K == 1 && !getenv_flag("QADIC_B1_TMA")) {  // one plane: 16-byte row segments, see planes_b1_kernel
            const int t1k = (int)((L.ldk * 2 + B1_KK - 1) / B1_KK), t1j = (int)((n + B1_J - 1) / B1_J);
            const int64_t t1 = (int64_t)t1k * t1j;
            static int occ1 = 0;
            if (!occ1) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, planes_b1_kernel, 256, 0);
                if (occ1 < 1) occ1 = 1;
            }
            const int grid = (int)(t1 < (int64_t)occ1 * num_sms() ? t1 : (int64_t)occ1 * num_sms());
            QADIC_TIMED("fp4k planes B", s,
                        planes_b1_kernel<<<grid, 256, 0, s>>>(b, kdim, n, p, tab, ps, lut, bs, L.ldk, t1k, t1j));
        } else if (use_tma) {  // TMA-fed; the grid is exactly one wave of resident blocks
            static int occ = 0;
            if (!occ) {
                cudaFuncSetAttribute(planes_b3_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)planes_b3_smem<K>());
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, planes_b3_kernel<K>, 256, planes_b3_smem<K>());
                if (occ < 1) occ = 1;
            }
            const int grid = (int)(tiles < (int64_t)occ * num_sms() ? tiles : (int64_t)occ * num_sms());
            QADIC_TIMED("fp4k planes B", s,
                        planes_b3_kernel<K><<<grid, 256, planes_b3_smem<K>(), s>>>(tm, kdim, n, p, tab, ps, lut, L.S,
                                                                                  bs, L.ldk, n * L.ldk, tk, tj,
                                                                                  b3_jmajor()));
        } else {  // unaligned B: lane loads
            static int occ = 0;
            if (!occ) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, planes_b2_kernel<K>, 256, 0);
                if (occ < 1) occ = 1;
            }
            const int grid = (int)(tiles < (int64_t)occ * num_sms() ? tiles : (int64_t)occ * num_sms());
            QADIC_TIMED("fp4k planes B", s,
                        planes_b2_kernel<K><<<grid, 256, 0, s>>>(b, kdim, n, p, tab, ps, lut, L.S, bs, L.ldk,
                                                                  n * L.ldk, tk, tj));
        }
    }
    if (a == nullptr) return;  // A planes already in the workspace (column-panel sweep)
    const int64_t ta = m * (L.ldk / 16);
    // QADIC_PA_PAD=bytes: unused dynamic shared memory, caps the resident blocks per SM (measurement switch)
    static const int pa_pad = getenv("QADIC_PA_PAD") ? atoi(getenv("QADIC_PA_PAD")) : 0;
    if (pa_pad > 0) cudaFuncSetAttribute(planes_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, pa_pad);
    QADIC_TIMED("fp4k planes A", s,
                planes_kernel<K><<<(unsigned)((ta + 255) / 256), 256, pa_pad, s>>>(a, m, kdim, p, tab, L.S, as, L.ldk,
                                                                                     m * L.ldk));
}

template <int K>
static void launch_combine(const uint8_t* d, int64_t m, int64_t n, const KaraLayout& L, uint32_t p, uint32_t magic,
                           const PlaneSpec& ps, uint8_t* c, cudaStream_t s) {
    const int64_t tot = m * ((n + 31) / 32);
    LaneDiv ld;
    if ((uint32_t)L.S * (p - 1) * (p - 1) < 256 && lane_div_plan(p, (uint32_t)L.S * (p - 1) * (p - 1), &ld) &&
        !getenv_flag("QADIC_COMBINE_SCALAR")) {
        const unsigned blocks = (unsigned)((tot + 255) / 256);
        auto go = [&](auto kern) {
            static const int st256 = getenv("QADIC_COMBINE_ST256") ? atoi(getenv("QADIC_COMBINE_ST256")) : 0;
            static const int pad = getenv("QADIC_COMBINE_PAD") ? atoi(getenv("QADIC_COMBINE_PAD")) : 0;  // as QADIC_PA_PAD
            if (pad > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
            QADIC_TIMED("fp4k combine", s, kern<<<blocks, 256, pad, s>>>(d, m, n, L.ldd, m * L.ldd, p, ld, ps, c, st256));
        };
        // the plane counts plan_planes() produces: Toom 2K-1, Karatsuba K(K+1)/2
        constexpr int S_TOOM = 2 * K - 1, S_KARA = K * (K + 1) / 2 <= KMAX_S ? K * (K + 1) / 2 : 2 * K - 1;
        if (L.S == S_TOOM) { go(combine_swar_kernel<K, S_TOOM>); return; }
        if (L.S == S_KARA) { go(combine_swar_kernel<K, S_KARA>); return; }
    }
    QADIC_TIMED("fp4k combine", s,
                combine_kernel<K><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(d, m, n, L.ldd, m * L.ldd, L.S, p,
                                                                                 magic, ps, c));
}

// C[m, n, k] = A[m, K, k] B[K, n, k] over GF(p^k) through plane products.
// Workspace: [plane table | B planes | A planes | D planes]; the table and the B
// planes sit at offsets independent of m, so a row-panelled caller (the host
// pipeline) prepares them once and passes REUSE_B_READY for the later panels.
// REUSE_COL_PANEL swaps the layout to [table | A planes | B planes | D planes]
// (A at an n-independent offset) for a caller that sweeps column panels of B
// against one A (the multi-GPU row-block step); REUSE_A_READY then skips the A
// conversion on every panel after the first.
static int run_kara(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                    void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, int reuse) {
    const bool b_ready = reuse & REUSE_B_READY;
    const int k = (int)f.k;
    PlaneSpec ps;
    QADIC_REQUIRE(plan_planes(f, &ps), QADIC_ERR_UNSUPPORTED, "no plane decomposition with <= %d planes", KMAX_S);
    KaraLayout L = kara_plan(ps.S, m, kdim, n, k);
    const size_t need = L.tab_bytes + L.a_bytes + L.b_bytes + L.d_bytes;
    QADIC_REQUIRE(ws != nullptr && ws_bytes >= need, QADIC_ERR_VALUE, "workspace too small (%zu < %zu)", ws_bytes,
                  need);
    uint32_t* tab = static_cast<uint32_t*>(ws);
    uint8_t *bs, *as;
    if (reuse & REUSE_COL_PANEL) {
        as = static_cast<uint8_t*>(ws) + L.tab_bytes;
        bs = as + L.a_bytes;
    } else {
        bs = static_cast<uint8_t*>(ws) + L.tab_bytes;
        as = bs + L.b_bytes;
    }
    uint8_t* dd = static_cast<uint8_t*>(ws) + L.tab_bytes + L.a_bytes + L.b_bytes;
    int ncodes = 1;
    for (int i = 0; i < k; ++i) ncodes *= (int)f.p;
    QADIC_REQUIRE(ncodes <= PT_CODES, QADIC_ERR_UNSUPPORTED, "plane table needs p^k <= %d", PT_CODES);
    const uint8_t* bsrc = b_ready ? nullptr : b;
    const uint8_t* asrc = (reuse & REUSE_A_READY) ? nullptr : a;
    const uint32_t lut = e2m1_lut(f.p, kdim);
    switch (k) {
        case 1: launch_planes<1>(asrc, bsrc, m, kdim, n, f.p, tab, ps, lut, L, as, bs, s); break;
        case 2: launch_planes<2>(asrc, bsrc, m, kdim, n, f.p, tab, ps, lut, L, as, bs, s); break;
        case 3: launch_planes<3>(asrc, bsrc, m, kdim, n, f.p, tab, ps, lut, L, as, bs, s); break;
        default: launch_planes<4>(asrc, bsrc, m, kdim, n, f.p, tab, ps, lut, L, as, bs, s); break;
    }
    int rc = check_launch("fp4k planes");
    if (rc) return rc;
    const bool pair = pair_mode();
    constexpr int BN = Cfg<KIND_F4>::BN;
    CUtensorMap ta, tb;
    rc = make_tmap(&ta, as, (kdim + 1) / 2, L.S * m, L.ldk, BM);
    if (rc) return rc;
    rc = make_tmap(&tb, bs, (kdim + 1) / 2, L.S * n, L.ldk, pair ? BN / 2 : BN);
    if (rc) return rc;
    Params prm = {};
    prm.sf = e2m1_scale_word();
    prm.group_m = getenv("QADIC_GROUP_M") ? atoi(getenv("QADIC_GROUP_M")) : GROUP_M;
    if (prm.group_m < 1) prm.group_m = 1;
    prm.diag_noload = getenv_flag("QADIC_DIAG_NOLOAD");
    prm.M = m;
    prm.N = n;
    prm.p = f.p;
    prm.offset = f.p * ((1u << 25) / f.p + 1);
    {  // non-negative representatives (no sign bit in any code): the sums are >= 0, no offset to add
        bool nonneg = true;
        for (uint32_t r = 0; r < f.p; ++r) nonneg = nonneg && !((lut >> (4 * r)) & 8u);
        if (nonneg) prm.offset = 0;
    }
    prm.magic64 = wide_magic(f.p);
    // FP4 sums are exact integers |v| < 2^24 (the engine's guard), so x = v + offset < 2^26 and the
    // 32-bit reciprocal is exact while x * p < 2^32 (every plane-engine prime): the epilogue's mod p
    // drops from a 64-bit multiply-high to IMAD.HI + IMAD.  QADIC_EPI_MOD64=1: the 64-bit form
    prm.magic32 = small_magic(f.p);  // (p <= 7 here: x * p < 2^29)
    prm.epi_mod64 = getenv_flag("QADIC_EPI_MOD64");
    prm.m_tiles = (int)((m + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM));
    prm.n_tiles = (int)((n + BN - 1) / BN);
    prm.n_full = (int)(n / BN);
    prm.num_kb = (int)(((kdim + 1) / 2 + BK - 1) / BK);
    prm.planes = L.S;
    // Fused combine: the GEMM epilogue accumulates W[l][s] * (D_s mod p) per output
    // tile in registers on byte lanes (needs S*(p-1)^2 < 256, k in {2, 3} and the
    // CTA-pair kernel) and writes C directly -- no D planes, no combine pass.  Its
    // tiles run plane-inner, so the L2 must hold S planes of operands: measured a
    // win at S = 3 (cfg3: 0.570 vs 0.586 ms) and a loss at S = 5 (cfg5: 1.047 vs
    // 1.012 ms; DRAM reads 1.6 vs 0.6 GB, tensor pipe 88 vs 94% active), hence the
    // default S <= 3; QADIC_FUSE_COMBINE=0/1 forces it off/on.
    const char* fuse_env = getenv("QADIC_FUSE_COMBINE");
    const bool want_fuse = fuse_env ? atoi(fuse_env) != 0 : L.S <= 3;
    LaneDiv ldv = {};
    const bool fuse = pair && (k == 2 || k == 3) && (int64_t)L.S * (f.p - 1) * (f.p - 1) < 256 &&
                      lane_div_plan(f.p, (uint32_t)L.S * (f.p - 1) * (f.p - 1), &ldv) && want_fuse;
    if (fuse) {
        prm.lane_m = ldv.m;
        prm.lane_sh = ldv.sh;
        prm.lane_qmask = ldv.qmask;
        prm.group_m = getenv("QADIC_FUSE_GROUP") ? atoi(getenv("QADIC_FUSE_GROUP")) : 8;
        if (prm.group_m < 1) prm.group_m = 1;
        for (int l = 0; l < k; ++l)
            for (int sidx = 0; sidx < KMAX_S; ++sidx) prm.W[l][sidx] = sidx < L.S ? ps.W[l][sidx] : 0;
        prm.c = c;
        prm.ldc = n * k;
        prm.c_plane = 0;
        prm.nibble_out = 0;
        return k == 2 ? launch_gemm<KIND_F4, true, 2>(ta, tb, prm, s, "fp4k gemm")
                      : launch_gemm<KIND_F4, true, 3>(ta, tb, prm, s, "fp4k gemm");
    }
    if (k == 1) {  // one plane: the GEMM writes C directly
        prm.c = c;
        prm.ldc = n;
        prm.c_plane = 0;
        prm.nibble_out = 0;
    } else {
        prm.c = dd;
        prm.ldc = L.ldd;
        prm.c_plane = m * L.ldd;
        prm.nibble_out = 1;
    }
    if (pair && mcast_mode() && prm.n_full >= 2) {
        // B tiles multicast across two CTA pairs (4-CTA clusters, 64-row boxes) on
        // the first column tiles; only C clusters of 4 fit (33 on B200), so the
        // last column tiles run concurrently as a CTA-pair launch on the SMs left
        // over, sized so both finish together (a multicast pair-tile costs
        // 1/QADIC_MCAST_GAIN of a plain one).
        CUtensorMap tbm;
        rc = make_tmap(&tbm, bs, (kdim + 1) / 2, L.S * n, L.ldk, Geo<KIND_F4, true, 0, true>::B_BOX);
        if (rc) return rc;
        const int C = gemm_max_clusters<KIND_F4, true, 0, true>();
        const int pairs_left = (num_sms() - 4 * C) / 2;
        const double gain = getenv("QADIC_MCAST_GAIN") ? atof(getenv("QADIC_MCAST_GAIN")) : 1.06;
        const double narrow = prm.n_tiles > prm.n_full ? (double)(n - (int64_t)prm.n_full * BN) / BN : 0.0;
        const double share = pairs_left / (pairs_left + 2.0 * C * gain);  // of the tile work
        int tail_full = (int)(share * (prm.n_full + narrow) - narrow + 0.5);
        if (tail_full < 0) tail_full = 0;
        if (tail_full > prm.n_full - 1) tail_full = prm.n_full - 1;
        const bool split = pairs_left >= 1 && (tail_full > 0 || prm.n_tiles > prm.n_full);
        Params pm = prm, pt = prm;
        pm.n_tile0 = 0;
        pm.n_full = pm.n_tiles = split ? prm.n_full - tail_full : prm.n_tiles;
        if (!split) pm.n_full = prm.n_full;
        pt.n_tile0 = pm.n_tiles;
        pt.n_tiles = prm.n_tiles - pm.n_tiles;
        pt.n_full = prm.n_full - pm.n_tiles;
        pt.pdl_tail = 1;
        const int pi = prof_begin(s, "fp4k gemm");
        cudaError_t e = launch_gemm_raw<KIND_F4, true, 0, true>(ta, tbm, pm, s);
        count_launch(1);
        if (e == cudaSuccess && split) {
            e = launch_gemm_raw<KIND_F4, true>(ta, tb, pt, s, pairs_left, true);
            count_launch(1);
        }
        prof_end(pi, s);
        if (e != cudaSuccess) {
            set_error(QADIC_ERR_CUDA, "fp4k gemm (multicast): %s", cudaGetErrorString(e));
            return QADIC_ERR_CUDA;
        }
        rc = check_launch("fp4k gemm", 0);
    } else {
        rc = pair ? launch_gemm<KIND_F4, true>(ta, tb, prm, s, "fp4k gemm")
                  : launch_gemm<KIND_F4, false>(ta, tb, prm, s, "fp4k gemm");
    }
    if (rc || k == 1) return rc;
    const uint32_t magic = small_magic(f.p);
    switch (k) {
        case 2: launch_combine<2>(dd, m, n, L, f.p, magic, ps, c, s); break;
        case 3: launch_combine<3>(dd, m, n, L, f.p, magic, ps, c, s); break;
        default: launch_combine<4>(dd, m, n, L, f.p, magic, ps, c, s); break;
    }
    return check_launch("fp4k combine");
}

// ---------------------------------------------------------------------------
// Exact uint64 GEMM (Layer K matmul_exact_u64, wraps mod 2^64) on INT8 tensor
// cores through byte planes.  With a = sum_i a_i 256^i, b = sum_j b_j 256^j:
//   C = sum_{s=0..7} 256^s D_s  (mod 2^64),   D_s = sum_{i+j=s} A_i B_j.
// The uint64 A matrix read as bytes IS the K-major operand A8 [M][8K] (byte i of
// element k at 8k+i); each D_s is ONE u8 x u8 GEMM of K'' = 8K against
// B^(s) [N][8K] with B^(s)[n][8k+i] = byte_{s-i}(B[k][n]) (0 when i > s), i.e.
// the 8 bytes bswap(B[k][n]) >> 8(7-s).  Only D_s mod 2^(64-8s) matters: exact
// in the u32 view of the s32 accumulator for s <= 3 while 4 * Kc * 255^2 < 2^32
// (K chunks of <= 16384), and the accumulator's wrap-around is exactly the
// needed mod 2^32 for s >= 4.  The epilogue adds D_s << 8s into C (uint64).
// ---------------------------------------------------------------------------
// 4 x 4 byte transpose: on return byte j of w[i] = old byte i of w[j]
__device__ __forceinline__ void transpose4_bytes(uint32_t (&w)[4]) {
    const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140), t1 = __byte_perm(w[0], w[1], 0x7362);
    const uint32_t t2 = __byte_perm(w[2], w[3], 0x5140), t3 = __byte_perm(w[2], w[3], 0x7362);
    w[0] = __byte_perm(t0, t2, 0x5410);
    w[1] = __byte_perm(t0, t2, 0x7632);
    w[2] = __byte_perm(t1, t3, 0x5410);
    w[3] = __byte_perm(t1, t3, 0x7632);
}

// 16 consecutive uint64 -> their byte planes: out[j] = 16 bytes (byte j of each word), j < 8
__device__ __forceinline__ void u64x16_byte_planes(const uint64_t (&v)[16], uint4 (&out)[8]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // words 4q .. 4q+3
        uint32_t lo[4] = {(uint32_t)v[4 * q], (uint32_t)v[4 * q + 1], (uint32_t)v[4 * q + 2], (uint32_t)v[4 * q + 3]};
        uint32_t hi[4] = {(uint32_t)(v[4 * q] >> 32), (uint32_t)(v[4 * q + 1] >> 32), (uint32_t)(v[4 * q + 2] >> 32),
                          (uint32_t)(v[4 * q + 3] >> 32)};
        transpose4_bytes(lo);
        transpose4_bytes(hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            reinterpret_cast<uint32_t*>(&out[j])[q] = lo[j];
            reinterpret_cast<uint32_t*>(&out[4 + j])[q] = hi[j];
        }
    }
}

// A [M][K] uint64, columns k0 .. k0+kc -> byte-plane-major rows:
//   out[m][i * kp + kk] = byte_i(A[m][k0 + kk]), i < nba, zero for kc <= kk < kp.
// Thread: 16 consecutive kk of one row (one 16-byte store per plane).
__global__ void __launch_bounds__(256) u64_aplanes_kernel(const uint64_t* __restrict__ a, int64_t M, int64_t K,
                                                          int64_t k0, int64_t kc, int nba, int64_t kp,
                                                          uint8_t* __restrict__ out, const int* __restrict__ plan) {
    // plan (device): planes past A's significant bytes are never read -- not written
    const int nw = plan ? plan[0] : nba;
    const int64_t per_row = kp / 16;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= M * per_row) return;
    const int64_t m = idx / per_row, kk0 = (idx % per_row) * 16;
    const uint64_t* src = a + m * K + k0 + kk0;
    uint64_t v[16];
    if (kk0 + 16 <= kc && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(src) + q);
            v[2 * q] = x.x;
            v[2 * q + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = kk0 + q < kc ? src[q] : 0ull;
    }
    uint4 pl[8];
    u64x16_byte_planes(v, pl);
    uint8_t* dst = out + m * (nba * kp) + kk0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < nba && i < nw) *reinterpret_cast<uint4*>(dst + i * kp) = pl[i];
}

// B [K][N] uint64, rows k0 .. k0+kc -> transposed byte planes:
//   out[j][n][kk] = byte_j(B[k0 + kk][n]), j < nbb, zero for kc <= kk < kp.
// Tile 128 kk x 32 n staged in shared memory (coalesced 256-byte row reads);
// thread (n, g) emits 16 kk per plane as one 16-byte store, 8 threads per
// 128-byte line of a plane row.
__global__ void __launch_bounds__(256) u64_btplanes_kernel(const uint64_t* __restrict__ b, int64_t K, int64_t N,
                                                           int64_t k0, int64_t kc, int nbb, int64_t kp,
                                                           uint8_t* __restrict__ out, const int* __restrict__ plan) {
    __shared__ uint64_t tile[128][33];
    const int nw = plan ? plan[1] : nbb;
    const int64_t n0 = (int64_t)blockIdx.x * 32, kk0 = (int64_t)blockIdx.y * 128;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll 4
    for (int r = ty; r < 128; r += 8) {
        const int64_t kk = kk0 + r, n = n0 + tx;
        tile[r][tx] = (kk < kc && n < N) ? __ldcs(b + (k0 + kk) * N + n) : 0ull;
    }
    __syncthreads();
    const int nl = threadIdx.x & 31, g = threadIdx.x >> 5;  // column n0 + nl, kk 16g .. 16g+15
    const int64_t n = n0 + nl;
    if (n >= N) return;
    uint64_t v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = tile[16 * g + q][nl];
    uint4 pl[8];
    u64x16_byte_planes(v, pl);
    uint8_t* dst = out + n * kp + kk0 + 16 * g;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < nbb && j < nw) *reinterpret_cast<uint4*>(dst + (int64_t)j * N * kp) = pl[j];
}

// OR of every word (significant byte count of the operand)
__global__ void u64_or_kernel(const uint64_t* __restrict__ x, int64_t n, unsigned long long* __restrict__ acc) {
    uint64_t v = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v |= x[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0 && v) atomicOr(acc, (unsigned long long)v);
}

// significant bytes of the two ORs (at least 1) -> plan[0], plan[1]
__global__ void u64_plan_kernel(const unsigned long long* __restrict__ ors, int* __restrict__ plan) {
    if (threadIdx.x < 2) {
        const unsigned long long v = ors[threadIdx.x];
        plan[threadIdx.x] = v ? (63 - __clzll((long long)v)) / 8 + 1 : 1;
    }
}


// ---------------------------------------------------------------------------
// I8K: the evaluation-plane decomposition of the FP4K engine on kind::i8 --
// residues 0..p-1 as int8 plane operands (exact in the int32 accumulator while
// K (p-1)^2 < 2^31), the same D planes, combine and workspace order.
// ---------------------------------------------------------------------------
// plane table, one byte per plane: T[code] byte s = sum_i E[s][i] digit_i mod p
__device__ __forceinline__ void build_plane_table8(uint2* tab, uint32_t p, int k, int S, const PlaneSpec& ps) {
    int ncodes = 1;
    for (int i = 0; i < k; ++i) ncodes *= (int)p;
    for (int c = threadIdx.x; c < ncodes; c += blockDim.x) {
        int r = c;
        uint32_t dig[kMaxK] = {};
        for (int i = 0; i < k; ++i) {
            dig[i] = (uint32_t)(r % (int)p);
            r /= (int)p;
        }
        uint32_t w[2] = {0, 0};
        for (int s = 0; s < S; ++s) {
            uint32_t v = 0;
            for (int i = 0; i < k; ++i) v += ps.E[s][i] * dig[i];
            w[s >> 2] |= (v % p) << (8 * (s & 3));
        }
        tab[c] = make_uint2(w[0], w[1]);
    }
}

// 16 table entries (8 plane bytes each) -> 16 bytes per plane: out[s]
__device__ __forceinline__ void entries16_to_planes(const uint2 (&e)[16], uint4 (&out)[8]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t lo[4] = {e[4 * q].x, e[4 * q + 1].x, e[4 * q + 2].x, e[4 * q + 3].x};
        uint32_t hi[4] = {e[4 * q].y, e[4 * q + 1].y, e[4 * q + 2].y, e[4 * q + 3].y};
        transpose4_bytes(lo);
        transpose4_bytes(hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            reinterpret_cast<uint32_t*>(&out[j])[q] = lo[j];
            reinterpret_cast<uint32_t*>(&out[4 + j])[q] = hi[j];
        }
    }
}

// Rows [R, Kd, K] of residues -> S byte planes [S][R][ld].  Thread: one row,
// 16 consecutive kk (16 K bytes in, one 16-byte store per plane).
template <int K>
__global__ void __launch_bounds__(256) planes8_a_kernel(const uint8_t* __restrict__ src, int64_t R, int64_t Kd,
                                                        uint32_t p, PlaneSpec ps, uint8_t* __restrict__ out,
                                                        int64_t ld, int64_t plane_stride) {
    __shared__ uint2 tab[PT_CODES];
    build_plane_table8(tab, p, K, ps.S, ps);
    __syncthreads();
    const CodeCoef<K> cc = make_code_coef<K>(p);
    const int64_t chunks = ld / 16;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < R * chunks;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / chunks, kk0 = (idx % chunks) * 16;
        const uint8_t* row = src + (r * Kd + kk0) * K;
        uint32_t in[4 * K];
        if (kk0 + 16 <= Kd && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
            for (int v = 0; v < K; ++v) {
                const uint4 x = __ldg(reinterpret_cast<const uint4*>(row) + v);
                in[4 * v] = x.x; in[4 * v + 1] = x.y; in[4 * v + 2] = x.z; in[4 * v + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int v = 0; v < 4 * K; ++v) in[v] = 0;
            for (int e = 0; e < 16 * K; ++e)
                if (kk0 + e / K < Kd) in[e >> 2] |= (uint32_t)row[e] << (8 * (e & 3));
        }
        uint32_t code[16];
        elem_codes<K, 4 * K>(in, cc, code);
        uint2 e[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) e[i] = kk0 + i < Kd ? tab[code[i]] : make_uint2(0, 0);
        uint4 pl[8];
        entries16_to_planes(e, pl);
        uint8_t* dst = out + r * ld + kk0;
#pragma unroll
        for (int sp = 0; sp < KMAX_S; ++sp)
            if (sp < ps.S) *reinterpret_cast<uint4*>(dst + sp * plane_stride) = pl[sp];
    }
}

// B [Kd, N, K] -> S transposed byte planes [S][N][ld].  Tile 128 kk x 32 j: the
// element codes are staged j-major in shared memory (a lane reads 4 consecutive
// elements = K words of a B row), then thread (j, g) looks up 16 kk of column j
// and writes 16 bytes per plane (8 threads per 128-byte plane-row segment).
template <int K>
__global__ void __launch_bounds__(256, 4) planes8_b_kernel(const uint8_t* __restrict__ b, int64_t Kd, int64_t N,
                                                        uint32_t p, PlaneSpec ps, uint8_t* __restrict__ out,
                                                        int64_t ld, int64_t plane_stride, int tiles_kk, int tiles_j) {
    __shared__ uint2 tab[PT_CODES];
    __shared__ __align__(16) uint16_t codes[32][128 + 8];  // [j][kk]: pass 2 reads 16 kk as two 16-byte loads
    build_plane_table8(tab, p, K, ps.S, ps);
    const CodeCoef<K> cc = make_code_coef<K>(p);
    const bool vec = ((N * K) % 4 == 0) && ((reinterpret_cast<uintptr_t>(b) & 3) == 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r4 = lane >> 3, c8 = lane & 7;  // pass 1: row of the warp's 4, 4-element chunk
    const int64_t ntiles = (int64_t)tiles_kk * tiles_j;
    // pass-1 words of one tile (rows 32 q + 4 warp + r4, elements 4 c8 .. 4 c8 + 3):
    // the next tile's are loaded into registers before this tile's pass 2, so the
    // loads overlap the lookups and stores
    uint32_t w[4][K];
    auto load = [&](int64_t t) {
        const int64_t kk0 = (t % tiles_kk) * 128, j0 = (t / tiles_kk) * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t gk = kk0 + 32 * q + 4 * warp + r4, gj = j0 + 4 * c8;
            if (vec && gk < Kd && gj + 4 <= N) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(b + (gk * N + gj) * K);
#pragma unroll
                for (int i = 0; i < K; ++i) w[q][i] = __ldg(src + i);
            } else {
#pragma unroll
                for (int i = 0; i < K; ++i) w[q][i] = 0;
                for (int e = 0; e < 4 * K; ++e)
                    if (gk < Kd && gj + e / K < N) w[q][e >> 2] |= (uint32_t)b[(gk * N + gj) * K + e] << (8 * (e & 3));
            }
        }
    };
    if ((int64_t)blockIdx.x < ntiles) load(blockIdx.x);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t kk0 = (t % tiles_kk) * 128, j0 = (t / tiles_kk) * 32;
        __syncthreads();  // table built / previous tile's codes consumed
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t cd[4];
            elem_codes<K, K>(w[q], cc, cd);
#pragma unroll
            for (int e = 0; e < 4; ++e) codes[4 * c8 + e][32 * q + 4 * warp + r4] = (uint16_t)cd[e];
        }
        __syncthreads();
        if (t + gridDim.x < ntiles) load(t + gridDim.x);
        // pass 2: column j0 + jl, kk 16 g .. 16 g + 15 of the tile; the 8 lanes of one
        // column write 128 contiguous bytes of each plane row (a warp: 4 whole lines)
        const int jl = 4 * warp + (lane >> 3), g = lane & 7;
        const int64_t gj = j0 + jl, col = kk0 + 16 * g;
        if (gj < N && col < ld) {
            const uint4 c0 = *reinterpret_cast<const uint4*>(&codes[jl][16 * g]);
            const uint4 c1 = *reinterpret_cast<const uint4*>(&codes[jl][16 * g + 8]);
            const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            uint2 e[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) e[i] = tab[(cw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu];
            uint4 pl[8];
            entries16_to_planes(e, pl);
            uint8_t* dst = out + gj * ld + col;
#pragma unroll
            for (int sp = 0; sp < KMAX_S; ++sp)
                if (sp < ps.S) *reinterpret_cast<uint4*>(dst + sp * plane_stride) = pl[sp];
        }
    }
}

// C[m, n, k] = A B over GF(p^k) (or F_p, k = 1) through S int8 plane GEMMs.
// Workspace: [B planes | A planes | D planes] (ldk = K bytes rounded to 16).
static size_t kara8_workspace(int S, int64_t m, int64_t kdim, int64_t n) {
    const int64_t ldk = round_up(kdim, 16), ldd = round_up((n + 1) / 2, 16);
    return (size_t)round_up(S * n * ldk, 1024) + (size_t)round_up(S * m * ldk, 1024) +
           (size_t)round_up(S * m * ldd, 1024);
}

static int run_kara8(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                     void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, bool b_ready) {
    const int k = (int)f.k;
    PlaneSpec ps;
    QADIC_REQUIRE(plan_planes(f, &ps), QADIC_ERR_UNSUPPORTED, "no plane decomposition with <= %d planes", KMAX_S);
    const int S = ps.S;
    const int64_t ldk = round_up(kdim, 16);
    KaraLayout L = {};
    L.S = S;
    L.ldk = ldk;
    L.ldd = round_up((n + 1) / 2, 16);
    L.b_bytes = (size_t)round_up(S * n * ldk, 1024);
    L.a_bytes = (size_t)round_up(S * m * ldk, 1024);
    L.d_bytes = (size_t)round_up(S * m * L.ldd, 1024);
    const size_t need = L.a_bytes + L.b_bytes + L.d_bytes;
    QADIC_REQUIRE(ws != nullptr && ws_bytes >= need, QADIC_ERR_VALUE, "workspace too small (%zu < %zu)", ws_bytes,
                  need);
    uint8_t* bs = static_cast<uint8_t*>(ws);
    uint8_t* as = bs + L.b_bytes;
    uint8_t* dd = as + L.a_bytes;
    auto planes = [&](auto kk) {
        constexpr int K = decltype(kk)::value;
        if (!b_ready) {
            const int tk = (int)((ldk + 127) / 128), tj = (int)((n + 31) / 32);
            const int64_t tiles = (int64_t)tk * tj;
            const int grid = (int)(tiles < 4LL * num_sms() ? tiles : 4LL * num_sms());
            QADIC_TIMED("i8k planes B", s,
                        planes8_b_kernel<K><<<grid, 256, 0, s>>>(b, kdim, n, f.p, ps, bs, ldk, n * ldk, tk, tj));
        }
        const int64_t items = m * (ldk / 16);
        const int grid = (int)((items + 255) / 256 < 8LL * num_sms() ? (items + 255) / 256 : 8LL * num_sms());
        QADIC_TIMED("i8k planes A", s,
                    planes8_a_kernel<K><<<grid, 256, 0, s>>>(a, m, kdim, f.p, ps, as, ldk, m * ldk));
    };
    switch (k) {
        case 1: planes(std::integral_constant<int, 1>{}); break;
        case 2: planes(std::integral_constant<int, 2>{}); break;
        case 3: planes(std::integral_constant<int, 3>{}); break;
        default: planes(std::integral_constant<int, 4>{}); break;
    }
    int rc = check_launch("i8k planes");
    if (rc) return rc;
    const bool pair = pair_mode();
    constexpr int BN = Cfg<KIND_I8>::BN;
    CUtensorMap ta, tb;
    rc = make_tmap(&ta, as, kdim, S * m, ldk, BM);
    if (rc) return rc;
    rc = make_tmap(&tb, bs, kdim, S * n, ldk, pair ? BN / 2 : BN);
    if (rc) return rc;
    Params prm = {};
    prm.group_m = GROUP_M;
    prm.M = m;
    prm.N = n;
    prm.p = f.p;
    prm.offset = 0;
    prm.magic64 = wide_magic(f.p);
    // plane sums <= kdim (p-1)^2: the epilogue's 32-bit reciprocal is exact while sum * p < 2^32
    if ((__int128)kdim * (f.p - 1) * (f.p - 1) * f.p < ((__int128)1 << 32)) prm.magic32 = small_magic(f.p);
    prm.epi_mod64 = getenv_flag("QADIC_EPI_MOD64");
    prm.m_tiles = (int)((m + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM));
    prm.n_tiles = (int)((n + BN - 1) / BN);
    prm.n_full = (int)(n / BN);
    prm.num_kb = (int)((kdim + BK - 1) / BK);
    prm.planes = S;
    if (k == 1) {  // one plane: the GEMM writes C directly
        prm.c = c;
        prm.ldc = n;
        prm.nibble_out = 0;
    } else {
        prm.c = dd;
        prm.ldc = L.ldd;
        prm.c_plane = m * L.ldd;
        prm.nibble_out = 1;
    }
    rc = pair ? launch_gemm<KIND_I8, true>(ta, tb, prm, s, "i8k gemm")
              : launch_gemm<KIND_I8, false>(ta, tb, prm, s, "i8k gemm");
    if (rc || k == 1) return rc;
    const uint32_t magic = small_magic(f.p);
    switch (k) {
        case 2: launch_combine<2>(dd, m, n, L, f.p, magic, ps, c, s); break;
        case 3: launch_combine<3>(dd, m, n, L, f.p, magic, ps, c, s); break;
        default: launch_combine<4>(dd, m, n, L, f.p, magic, ps, c, s); break;
    }
    return check_launch("i8k combine");
}

// ---------------------------------------------------------------------------
// Batched long-polynomial products on INT8 tensor cores (Toeplitz GEMM).
//   out_s[y] = sum_x a_s[x] b_s[y - x] mod p   (s = 0 .. batch-1, residues < p <= 127)
// Split b_s into V = ceil(nb / TL) blocks of TL coefficients: the product of a_s with
// block v is column v of D_s = T_s Bv_s^T, where T_s [M = na + TL - 1][TL] is the
// Toeplitz matrix T_s[x][l] = a_s[x - l] (K-major: row x is a reversed window of a_s)
// and Bv_s [V][TL] is b_s itself, zero padded.  One batched GEMM (the batch as the
// GEMM's planes, tcgen05 kind::i8, int32 TMEM sums of TL (p-1)^2 < 2^31, mod-p epilogue)
// stores D_s as its diagonal-shifted transpose E_s[v][x + v TL] = D_s[x][v] (uint8), so the
// overlap-add out_s[y] = sum_v E_s[v][y] mod p reads whole aligned vectors.  The arithmetic
// is the convolution itself (exact integers): the result equals polymul_fqt's for any
// packing.  Traffic per pair: T (M TL bytes) + E (V (M + (V-1) TL) bytes).
constexpr int TL_DEFAULT = 256;  // Toeplitz width (GEMM K): 0.103 ms vs 0.128 (128), 0.118 (512) at polylong

// apad[s][k] = a_s[na - 1 - (k - TL)] for TL <= k < TL + na, else 0 (a_s reversed, zero
// margins): the Toeplitz row x, chunk c is the 16 contiguous bytes at k = TL + na - 1 - x + 16c
__global__ void reverse_pad_kernel(const uint8_t* __restrict__ a, int64_t batch, int64_t na, int64_t len,
                                   uint8_t* __restrict__ apad, int TL) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < batch * len; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sidx = g / len, k = g - sidx * len, i = k - TL;
        apad[g] = (i >= 0 && i < na) ? a[sidx * na + (na - 1 - i)] : (uint8_t)0;
    }
}

__global__ void toeplitz_rows_kernel(const uint8_t* __restrict__ apad, int64_t batch, int64_t na, int64_t len,
                                     int64_t M, uint8_t* __restrict__ T, int TL) {
    // one thread per 16-byte chunk (s, x, c): T[s][x][16c + j] = a_s[x - 16c - j] = apad_s[o + j],
    // o = TL + na - 1 - x + 16c: five aligned words, funnel-shifted into place
    const int64_t chunks = TL / 16, total = batch * M * chunks;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sx = g / chunks;
        const int c = (int)(g - sx * chunks);
        const int64_t sidx = sx / M, x = sx - sidx * M;
        const int64_t o = TL + na - 1 - x + 16 * c;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(apad + sidx * len) + (o >> 2);
        const uint32_t sh = 8u * (uint32_t)(o & 3);
        uint32_t v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] = __ldg(w + k);
        uint32_t r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = __funnelshift_r(v[k], v[k + 1], sh);
        *reinterpret_cast<uint4*>(T + sx * TL + 16 * c) = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// The Toeplitz operand without materialising it: GEMM row x (Toeplitz row M-1-x) is
// apad[1 + x .. 1 + x + TL), so with 16 copies P_phi[j] = apad[1 + phi + j] (16-byte
// aligned) row 16 r + phi is P_phi[16 r ..] -- a tensor map with a 16-byte row stride
// over overlapping rows reads any tile (GEMM producer, a_phase).  16 x (na + 2 TL)
// bytes per pair instead of (na + TL) x TL.
__global__ void toeplitz_phase_kernel(const uint8_t* __restrict__ apad, int64_t batch, int64_t len, int64_t Lc,
                                      uint8_t* __restrict__ P) {
    const int64_t chunks = Lc / 16, total = batch * 16 * chunks;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sp = g / chunks, c = g - sp * chunks;
        const int64_t sidx = sp / 16;
        const int ph = (int)(sp - sidx * 16);
        const int64_t o = 1 + ph + 16 * c;
        const uint8_t* src = apad + sidx * len;
        uint32_t r[4];
        if (o + 20 <= len) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(src) + (o >> 2);
            const uint32_t sh = 8u * (uint32_t)(o & 3);
            uint32_t v[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) v[k] = __ldg(w + k);
#pragma unroll
            for (int k = 0; k < 4; ++k) r[k] = __funnelshift_r(v[k], v[k + 1], sh);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) r[k] = 0;
            for (int j = 0; j < 16; ++j)
                if (o + j < len) r[j >> 2] |= (uint32_t)src[o + j] << (8 * (j & 3));
        }
        *reinterpret_cast<uint4*>(P + sp * Lc + 16 * c) = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// Phase copies for the convolution mode: P[s][phi][j] = a_s[X0 - phi - j] (0 outside
// [0, na)), so GEMM row x~ = 16 r + phi of the phase map, P_phi[16 r + k] = a[X0 - x~ - k],
// is Toeplitz row X0 - x~ (T[x][k] = a[x - k]).
__global__ void conv_phase_kernel(const uint8_t* __restrict__ a, int64_t batch, int64_t na, int64_t X0, int64_t Lc,
                                  uint8_t* __restrict__ P) {
    const int64_t chunks = Lc / 16, total = batch * 16 * chunks;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sp = g / chunks, c = g - sp * chunks;
        const int64_t sidx = sp / 16;
        const int ph = (int)(sp - sidx * 16);
        const uint8_t* as = a + sidx * na;
        const int64_t top = X0 - ph - 16 * c;  // a index of byte 0 of this chunk (descending)
        const int64_t lo = top - 15;           // the chunk is a[lo .. top] reversed
        uint32_t r[4] = {0, 0, 0, 0};
        if (lo >= 0 && top < na && (reinterpret_cast<uintptr_t>(as) & 3) == 0) {
            // five aligned words cover a[lo .. top]; funnel-shift them into place, then reverse
            const int64_t w0 = lo >> 2;
            const uint32_t sh = 8u * (uint32_t)(lo & 3);
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(as) + w0;
            const int64_t nw = (na + 3) >> 2;  // words that hold a byte of a
            uint32_t v[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) v[k] = (w0 + k < nw) ? __ldg(aw + k) : 0u;
            uint32_t f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = __funnelshift_r(v[k], v[k + 1], sh);  // a[lo + 4k .. lo + 4k + 3]
#pragma unroll
            for (int k = 0; k < 4; ++k) r[k] = __byte_perm(f[3 - k], 0, 0x0123);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int64_t i = top - j;
                if (i >= 0 && i < na) r[j >> 2] |= (uint32_t)__ldg(as + i) << (8 * (j & 3));
            }
        }
        *reinterpret_cast<uint4*>(P + sp * Lc + 16 * c) = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// split-K partials of the convolution mode -> coefficients mod p (4 per thread)
__global__ void conv_reduce_kernel(const int32_t* __restrict__ part, int S, int64_t batch, int64_t ytot, int64_t ncoef,
                                   uint32_t p, uint64_t magic64, uint8_t* __restrict__ out, unsigned int* flag) {
    const int64_t q4 = (ytot + 3) / 4, total = batch * q4;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sidx = g / q4, y0 = (g - sidx * q4) * 4;
        uint32_t acc[4] = {0, 0, 0, 0};
        for (int j = 0; j < S; ++j) {
            const int32_t* src = part + ((int64_t)j * batch + sidx) * ytot + y0;
            if (y0 + 4 <= ytot && (ytot & 3) == 0) {
                const int4 v = __ldcs(reinterpret_cast<const int4*>(src));
                acc[0] += (uint32_t)v.x; acc[1] += (uint32_t)v.y; acc[2] += (uint32_t)v.z; acc[3] += (uint32_t)v.w;
            } else {
                for (int e = 0; e < 4; ++e)
                    if (y0 + e < ytot) acc[e] += (uint32_t)src[e];
            }
        }
        for (int e = 0; e < 4; ++e) {
            const int64_t y = y0 + e;
            if (y >= ytot) break;
            const uint32_t r = mod_u32(acc[e], p, magic64);
            if (y < ncoef) out[sidx * ncoef + y] = (uint8_t)r;
            else if (r) atomicOr(flag, 2u);
        }
    }
}

__global__ void blocks_kernel(const uint8_t* __restrict__ b, int64_t batch, int64_t nb, int64_t V,
                              uint8_t* __restrict__ Bv, int TL) {
    // Bv[s][v][l] = b_s[v TL + l] (0 past nb), 16 bytes per thread
    const int64_t chunks = V * TL / 16, total = batch * chunks;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sidx = g / chunks, e0 = (g - sidx * chunks) * 16;
        const uint8_t* bs = b + sidx * nb;
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int64_t i = e0 + j;
            const uint32_t v = i < nb ? (uint32_t)__ldg(bs + i) : 0u;
            w[j >> 2] |= v << (8 * (j & 3));
        }
        *reinterpret_cast<uint4*>(Bv + sidx * V * TL + e0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

constexpr int OV_SPLIT = 8;  // threads per 16-output group (each sums every 8th row v)

__global__ void toeplitz_overlap_diag_kernel(const uint8_t* __restrict__ E, int64_t batch, int64_t M, int64_t V,
                                             int64_t lde, uint32_t p, int64_t nfull, int64_t ncoef,
                                             uint8_t* __restrict__ out, unsigned int* flag, int TL) {
    const int64_t span = ((ncoef > nfull ? ncoef : nfull) + 15) / 16;
    const int part = threadIdx.x % OV_SPLIT;  // lanes of a group are consecutive: shuffle-combinable
    const int64_t total = batch * span, stride = (int64_t)gridDim.x * blockDim.x / OV_SPLIT;
    // warp-uniform trip count: every lane takes part in the group shuffles below
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / OV_SPLIT; __any_sync(0xffffffffu, g < total);
         g += stride) {
        const bool act = g < total;
        const int64_t gg = act ? g : 0;
        const int64_t sidx = gg / span, y0 = (gg - sidx * span) * 16;
        uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // byte j of the 16 in lane (j & 1) of acc[j >> 1]
        if (act && y0 < nfull) {
            const uint8_t* Es = E + sidx * V * lde;
            const int64_t vlo = y0 + 15 >= M ? (y0 + 15 - M) / TL : 0;
            const int64_t vhi = y0 / TL < V - 1 ? y0 / TL : V - 1;
            int terms = 0;
            for (int64_t v = vlo + part; v <= vhi; v += OV_SPLIT) {
                const int64_t lo = v * TL, hi = v * TL + M;  // written range of row v
                if (y0 + 15 < lo || y0 >= hi) continue;
                const uint4 w = __ldg(reinterpret_cast<const uint4*>(Es + v * lde + y0));
                uint32_t x[4] = {w.x, w.y, w.z, w.w};
                if (y0 < lo || y0 + 15 >= hi) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (y0 + j < lo || y0 + j >= hi) x[j >> 2] &= ~(0xFFu << (8 * (j & 3)));
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[2 * q] += x[q] & 0x00FF00FFu;
                    acc[2 * q + 1] += (x[q] >> 8) & 0x00FF00FFu;
                }
                if (++terms == 60) {  // 8 partial sums of <= 60 x 126 + p are combined below
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = ((acc[i] & 0xFFFFu) % p) | (((acc[i] >> 16) % p) << 16);
                    terms = 0;
                }
            }
        }
        // combine the group's partial sums (8 x < 7686 < 2^16 per lane)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int o = OV_SPLIT / 2; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
        if (part == 0 && act) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int64_t y = y0 + j;
                const int q = j >> 2, b = j & 3;
                const uint32_t sum = (acc[2 * q + (b & 1)] >> (16 * (b >> 1))) & 0xFFFFu;
                const uint32_t r = y < nfull ? sum % p : 0u;
                if (y < ncoef) out[sidx * ncoef + y] = (uint8_t)r;
                else if (r) atomicOr(flag, 2u);
            }
        }
    }
}

static int tz_width() {
    static const int w = getenv("QADIC_TZ_L") ? atoi(getenv("QADIC_TZ_L")) : TL_DEFAULT;
    return (w >= 128 && w % 128 == 0) ? w : TL_DEFAULT;
}
static int64_t tz_pad_len(int64_t na, int TL) { return round_up(na + 2 * TL + 32, 16); }
static int64_t tz_phase_len(int64_t na, int TL) { return round_up(na + 2 * TL + 16, 16); }
// the Toeplitz operand as 16 phase copies read through an overlapping-row tensor map
// (default) or materialised row by row (QADIC_TZ_MATERIALIZE=1, the earlier form)
static bool tz_materialize() {  // (the CTA-pair variant QADIC_TZ_PAIR=1 reads materialised rows)
    static const bool m = (getenv("QADIC_TZ_MATERIALIZE") && atoi(getenv("QADIC_TZ_MATERIALIZE")) != 0) ||
                          (getenv("QADIC_TZ_PAIR") && atoi(getenv("QADIC_TZ_PAIR")) != 0);
    return m;
}

static size_t toeplitz_workspace(int64_t batch, int64_t na, int64_t nb) {
    const int TL = tz_width();
    const int64_t M = na + TL - 1, V = (nb + TL - 1) / TL;
    const int64_t aop = tz_materialize() ? batch * M * TL : batch * 16 * tz_phase_len(na, TL);
    return (size_t)round_up(batch * tz_pad_len(na, TL), 1024) + (size_t)round_up(aop, 1024) +
           (size_t)round_up(batch * V * TL, 1024) +
           (size_t)round_up(batch * V * round_up(M + (V - 1) * TL + 16, 16), 1024) + 1024;
}

// 4-D map over the phase copies: {TL bytes, rows (16-byte stride, overlapping), 16 phases, batch}
static int make_tmap_phase(CUtensorMap* map, const void* base, int TL, int64_t rows, int64_t Lc, int64_t batch) {
    EncodeTiledFn fn = encode_fn();
    QADIC_REQUIRE(fn != nullptr, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[4] = {(cuuint64_t)TL, (cuuint64_t)rows, 16, (cuuint64_t)batch};
    cuuint64_t strides[3] = {16, (cuuint64_t)Lc, (cuuint64_t)(16 * Lc)};
    cuuint32_t box[4] = {(cuuint32_t)BK, 8, 16, 1};  // one box = a whole 128-row tile: [phase][8 rows][BK]
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QADIC_REQUIRE(r == CUDA_SUCCESS, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled (phase map) failed (%d)", (int)r);
    return QADIC_OK;
}

// ---- convolution mode (default for the long products): overlap-add in TMEM ----------
struct ConvPlan {
    int TL;
    int64_t X0, Lc, R, Vb, Vp, W;
};
static int conv_width() {  // K of one Toeplitz row block: 128 gives N = 256-column tiles at polylong
    static const int w = getenv("QADIC_CONV_L") ? atoi(getenv("QADIC_CONV_L")) : 128;
    return (w >= 128 && w % 128 == 0) ? w : 128;
}
static ConvPlan conv_plan(int64_t na, int64_t nb, int64_t ncoef) {
    ConvPlan c;
    c.TL = conv_width();
    c.X0 = na + c.TL - 1;
    c.X0 += (15 - c.X0 % 16 + 16) % 16;  // X0 = 15 (mod 16): every tile's first GEMM row on a phase row
    c.Lc = round_up(c.X0 + c.TL + 16, 16);
    c.R = (c.X0 + 16) / 16;
    c.Vb = (nb + c.TL - 1) / c.TL;
    const int64_t nfull = na + nb - 1, span = ncoef > nfull ? ncoef : nfull;
    c.Vp = (span + c.TL - 1) / c.TL;
    c.W = (na + c.TL - 2) / c.TL + 1;  // Toeplitz row blocks with a nonzero entry
    return c;
}
static bool conv_default() {
    static const bool old = (getenv("QADIC_TZ_OLD") && atoi(getenv("QADIC_TZ_OLD")) != 0) || tz_materialize();
    return !old;
}
constexpr int CONV_MAX_SPLIT = 16;
// split-K factor: enough units to fill the SMs, at least 4 Toeplitz row blocks per split
static int conv_splits(int64_t units, int64_t W) {
    int S = 1;
    while (S < CONV_MAX_SPLIT && units * S < num_sms_cached() && W / (2 * S) >= 4) S *= 2;
    return S;
}
static int64_t conv_cols(const ConvPlan& c) {  // N per column tile (256 = the full-rate int8 MMA)
    return std::min<int64_t>(256, round_up(c.Vp, 16));
}
static size_t conv_part_bytes(int64_t batch, const ConvPlan& c) {
    const int64_t tc = conv_cols(c), Np = round_up(c.Vp, tc);
    const int64_t units = batch * (c.TL / 128) * (Np / tc);  // upper bound (no pairs)
    const int S = conv_splits(units, c.W);
    return S > 1 ? (size_t)S * batch * Np * c.TL * sizeof(int32_t) : 0;
}
// workspace: [phase copies | b blocks | flag (1 KB) | split-K partials (optional: used
// when the room after the flag holds them, sized here for ncoef <= na + nb - 1)]
static size_t conv_fixed_bytes(int64_t batch, const ConvPlan& c) {
    return (size_t)round_up(batch * 16 * c.Lc, 1024) + (size_t)round_up(batch * c.Vb * c.TL, 1024) + 1024;
}
static size_t conv_workspace(int64_t batch, int64_t na, int64_t nb, int64_t ncoef) {
    const ConvPlan c = conv_plan(na, nb, ncoef);
    return conv_fixed_bytes(batch, c) + conv_part_bytes(batch, c);
}

static int run_conv(const uint8_t* a, int64_t na, const uint8_t* b, int64_t nb, int64_t batch, uint32_t p, uint8_t* out,
                    int64_t ncoef, void* ws, size_t ws_bytes, cudaStream_t s) {
    const ConvPlan c = conv_plan(na, nb, ncoef);
    const int TL = c.TL;
    QADIC_REQUIRE(ws && ws_bytes >= conv_fixed_bytes(batch, c), QADIC_ERR_VALUE, "workspace too small");
    QADIC_REQUIRE((__int128)std::min(na, nb) * (p - 1) * (p - 1) < ((__int128)1 << 31), QADIC_ERR_PARAMS,
                  "the int32 accumulator cannot hold min(len_a, len_b) * (p-1)^2");
    QADIC_REQUIRE(c.R < (1ll << 31) && c.Vp < (1ll << 31) && c.W * (TL / BK) < (1ll << 30) && batch < (1ll << 31),
                  QADIC_ERR_UNSUPPORTED, "long product beyond the tensor-map ranges");
    uint8_t* P = static_cast<uint8_t*>(ws);
    uint8_t* Bv = P + round_up(batch * 16 * c.Lc, 1024);
    unsigned int* flag = reinterpret_cast<unsigned int*>(Bv + round_up(batch * c.Vb * TL, 1024));
    int32_t* part = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(flag) + 1024);
    const size_t part_room = ws_bytes - conv_fixed_bytes(batch, c);
    const int sms = num_sms();
    auto grid_of = [&](int64_t n) {
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16));
    };
    QADIC_TIMED("polymul conv A", s, conv_phase_kernel<<<grid_of(batch * c.Lc), 256, 0, s>>>(a, batch, na, c.X0, c.Lc, P));
    QADIC_TIMED("polymul conv B", s, blocks_kernel<<<grid_of(batch * c.Vb * (TL / 16)), 256, 0, s>>>(b, batch, nb, c.Vb, Bv, TL));
    int rc = check_launch("conv operands");
    if (rc) return rc;
    cudaMemsetAsync(flag, 0, sizeof(unsigned int), s);
    constexpr int BN = Cfg<KIND_I8>::BN;
    CUtensorMap ta, tb;
    rc = make_tmap_phase(&ta, P, TL, c.R, c.Lc, batch);
    if (rc) return rc;
    // CTA pairs (cta_group::2): the two 128-row halves (y0 = 0, 128) of a 256-coefficient
    // block share the b blocks, each CTA loading half of the column tile; the B box holds
    // that half only (a single tile of Vp <= BN columns loads Vp / 2 rows, not BN / 2)
    const bool pair = TL % 256 == 0 && !(getenv("QADIC_CONV_PAIR") && atoi(getenv("QADIC_CONV_PAIR")) == 0);
    // every column tile has the same width (the box is fixed): one tile of Vp rounded to 16,
    // or full BN tiles over Vp rounded up to BN (the extra columns address coefficients past
    // the output and come out zero)
    // column tile: as wide as the MMA allows (N = 256: an N = 128 tile runs the int8 pipe at
    // about half rate), narrowed while the launch would leave SMs idle (small batches)
    const int tile_cols = (int)conv_cols(c);
    const int per_pair_rows = TL / (pair ? 2 * BM : BM);
    const int64_t Np = round_up(c.Vp, tile_cols);
    const int brows = pair ? tile_cols / 2 : tile_cols;
    // small batches: split the row blocks across CTAs (int32 partials + conv_reduce_kernel)
    int S = conv_splits(batch * per_pair_rows * (Np / tile_cols), c.W);
    const int64_t ytot = Np * TL;
    if (S > 1 && (size_t)S * batch * ytot * sizeof(int32_t) > part_room) S = 1;
    const int wc = (int)((c.W + S - 1) / S);
    S = (int)((c.W + wc - 1) / wc);  // every split non-empty
    {
        EncodeTiledFn fn = encode_fn();
        QADIC_REQUIRE(fn != nullptr, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        cuuint64_t dims[3] = {(cuuint64_t)TL, (cuuint64_t)c.Vb, (cuuint64_t)batch};
        cuuint64_t strides[2] = {(cuuint64_t)TL, (cuuint64_t)(c.Vb * TL)};
        cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)brows, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, Bv, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        QADIC_REQUIRE(r == CUDA_SUCCESS, QADIC_ERR_CUDA, "cuTensorMapEncodeTiled (conv B) failed (%d)", (int)r);
    }
    Params prm = {};
    prm.sf = e2m1_scale_word();
    prm.group_m = GROUP_M;
    prm.M = TL;
    prm.N = Np;
    prm.p = p;
    prm.magic64 = wide_magic(p);
    prm.m_tiles = per_pair_rows * S;
    prm.n_tiles = (int)(Np / tile_cols);
    prm.n_full = prm.n_tiles;
    prm.num_kb = (int)(c.W * (TL / BK));
    prm.planes = (int)batch;
    prm.c = out;
    prm.ldc = ncoef;
    prm.conv = 1;
    prm.conv_tl = TL;
    prm.conv_x0 = (int)c.X0;
    prm.conv_kpw = TL / BK;
    prm.conv_ncoef = ncoef;
    prm.conv_flag = flag;
    prm.conv_brows = brows;
    prm.conv_tn = tile_cols;
    prm.conv_rows = per_pair_rows;
    prm.conv_wc = wc;
    prm.conv_w = (int)c.W;
    prm.conv_part = S > 1 ? part : nullptr;
    prm.conv_ytot = ytot;
    rc = pair ? launch_gemm<KIND_I8, true>(ta, tb, prm, s, "polymul conv gemm")
              : launch_gemm<KIND_I8, false>(ta, tb, prm, s, "polymul conv gemm");
    if (rc || S == 1) return rc;
    QADIC_TIMED("polymul conv reduce", s,
                conv_reduce_kernel<<<grid_of(batch * ((ytot + 3) / 4)), 256, 0, s>>>(part, S, batch, ytot, ncoef, p,
                                                                                   wide_magic(p), out, flag));
    return check_launch("conv reduce");
}

static int run_toeplitz(const uint8_t* a, int64_t na, const uint8_t* b, int64_t nb, int64_t batch, uint32_t p,
                        uint8_t* out, int64_t ncoef, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (conv_default()) return run_conv(a, na, b, nb, batch, p, out, ncoef, ws, ws_bytes, s);
    const int TL = tz_width();
    const int64_t M = na + TL - 1, V = (nb + TL - 1) / TL, len = tz_pad_len(na, TL);
    QADIC_REQUIRE(ws && ws_bytes >= toeplitz_workspace(batch, na, nb), QADIC_ERR_VALUE, "workspace too small");
    QADIC_REQUIRE(batch * M < (1ll << 31) && batch * V < (1ll << 31), QADIC_ERR_UNSUPPORTED,
                  "batch x length beyond the TMA row range");
    const bool mat = tz_materialize();
    const int64_t Lc = tz_phase_len(na, TL);
    uint8_t* apad = static_cast<uint8_t*>(ws);
    uint8_t* T = apad + round_up(batch * len, 1024);  // materialised rows or the 16 phase copies
    uint8_t* Bv = T + round_up(mat ? batch * M * TL : batch * 16 * Lc, 1024);
    uint8_t* Dt = Bv + round_up(batch * V * TL, 1024);
    unsigned int* flag =
        reinterpret_cast<unsigned int*>(Dt + round_up(batch * V * round_up(M + (V - 1) * TL + 16, 16), 1024));
    const int sms = num_sms();
    auto grid_of = [&](int64_t n) {
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16));
    };
    QADIC_TIMED("polymul toeplitz pad", s, reverse_pad_kernel<<<grid_of(batch * len), 256, 0, s>>>(a, batch, na, len, apad, TL));
    if (mat)
        QADIC_TIMED("polymul toeplitz A", s,
                    toeplitz_rows_kernel<<<grid_of(batch * M * (TL / 16)), 256, 0, s>>>(apad, batch, na, len, M, T, TL));
    else
        QADIC_TIMED("polymul toeplitz A", s,
                    toeplitz_phase_kernel<<<grid_of(batch * Lc), 256, 0, s>>>(apad, batch, len, Lc, T));
    QADIC_TIMED("polymul toeplitz B", s, blocks_kernel<<<grid_of(batch * V * (TL / 16)), 256, 0, s>>>(b, batch, nb, V, Bv, TL));
    int rc = check_launch("toeplitz operands");
    if (rc) return rc;
    // single-CTA tiles: the short-K, narrow-N tiles of this GEMM are latency-bound per tile, and
    // 148 independent CTAs beat 74 pairs (measured 0.094 vs 0.103 ms per polylong batch)
    static const bool pair = getenv("QADIC_TZ_PAIR") && atoi(getenv("QADIC_TZ_PAIR")) != 0;
    constexpr int BN = Cfg<KIND_I8>::BN;
    // GEMM rows = the M Toeplitz rows, columns = the V blocks of b, stored as the
    // diagonal-shifted transpose E[v][x + v TL] (rows of lde >= M + (V - 1) TL + 16 bytes)
    const int64_t lde = round_up(M + (V - 1) * TL + 16, 16);
    CUtensorMap ta, tb;
    const bool phase = !mat && !pair;
    rc = phase ? make_tmap_phase(&ta, T, TL, (M + 15) / 16, Lc, batch) : make_tmap(&ta, T, TL, batch * M, TL, BM);
    if (rc) return rc;
    rc = make_tmap(&tb, Bv, TL, batch * V, TL, pair ? BN / 2 : BN);
    if (rc) return rc;
    Params prm = {};
    prm.sf = e2m1_scale_word();
    prm.group_m = GROUP_M;
    prm.M = M;
    prm.N = V;
    prm.ldc = lde;
    prm.p = p;
    prm.offset = p * ((1u << 25) / p + 1);
    prm.magic64 = wide_magic(p);
    prm.m_tiles = (int)((M + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM));
    prm.n_tiles = (int)((V + BN - 1) / BN);
    prm.n_full = (int)(V / BN);
    prm.num_kb = (int)((TL + BK - 1) / BK);
    prm.c = Dt;
    prm.c_plane = V * lde;
    prm.diag_shift = TL;
    prm.planes = (int)batch;
    prm.nibble_out = 0;
    prm.a_phase = phase ? 1 : 0;
    rc = pair ? launch_gemm<KIND_I8, true>(ta, tb, prm, s, "polymul toeplitz gemm")
              : launch_gemm<KIND_I8, false>(ta, tb, prm, s, "polymul toeplitz gemm");
    if (rc) return rc;
    cudaMemsetAsync(flag, 0, sizeof(unsigned int), s);
    const int64_t nfull = na + nb - 1;
    QADIC_TIMED("polymul overlap", s,
                toeplitz_overlap_diag_kernel<<<grid_of(batch * ((std::max(nfull, ncoef) + 15) / 16) * OV_SPLIT), 256, 0, s>>>(
                    Dt, batch, M, V, lde, p, nfull, ncoef, out, flag, TL));
    return check_launch("toeplitz overlap");
}

}  // namespace tc

size_t tc_toeplitz_workspace(int64_t batch, int64_t na, int64_t nb) {
    // (split-K partials sized for the batched API's output length, 2 max(na, nb) - 1)
    return tc::conv_default() ? tc::conv_workspace(batch, na, nb, 2 * std::max(na, nb) - 1)
                              : tc::toeplitz_workspace(batch, na, nb);
}

int tc_polymul_toeplitz(const uint8_t* a, int64_t na, const uint8_t* b, int64_t nb, int64_t batch, uint32_t p,
                        uint8_t* out, int64_t ncoef, void* ws, size_t ws_bytes, cudaStream_t s) {
    QADIC_REQUIRE(p >= 2 && p <= 127, QADIC_ERR_UNSUPPORTED, "the tensor-core product needs p <= 127");
    QADIC_REQUIRE((int64_t)tc::tz_width() * (p - 1) * (p - 1) < (1ll << 31), QADIC_ERR_PARAMS, "int32 sum bound");
    return tc::run_toeplitz(a, na, b, nb, batch, p, out, ncoef, ws, ws_bytes, s);
}

bool tc_u64_ok(int64_t m, int64_t k, int64_t n, const void* a) {
    return m >= 128 && n >= 128 && k >= 16 && (k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
}

int tc_matmul_u64(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t m, int64_t k, int64_t n,
                  cudaStream_t s) {
    using namespace tc;
    constexpr int64_t KC = 16384;  // 4 * KC * 255^2 < 2^32
    keep_mempool();
    // D_s = sum_{i+j=s} A_i B_j^T over the byte planes that can be nonzero (i < nba,
    // j < nbb): plane s runs one GEMM whose K'' is the concatenation of its valid
    // segments (A plane i against B plane s-i), so only the nonzero byte products
    // are issued -- sum_s #{i} = 24 per word MAC at 5 + 5 bytes, not 36.  nba / nbb
    // (the operands' significant bytes: 5 for the reference drivers' packed words)
    // are found on the device -- an OR reduction and a plan the GEMM launches read --
    // so the call stays asynchronous on the caller's stream and capturable; the byte
    // planes are laid out for all 8 bytes (the insignificant ones are zeros nobody reads).
    // The opt-in single-launch form (QADIC_U64_INNER) keeps host-side segment tables
    // and multiplies all 8 x 8 byte pairs.
    const bool inner = getenv_flag("QADIC_U64_INNER");
    const int nba = 8, nbb = 8;  // plane layout (and the inner form's segment tables)
    const int nplanes = 8;       // shifts 8s >= 64 vanish mod 2^64
    const int64_t kc_max = k < KC ? k : KC;
    const int64_t kp = (kc_max + BK - 1) / BK * BK;  // segment length (bytes), BK-aligned
    const size_t abytes = (size_t)m * nba * kp, bbytes = (size_t)nbb * n * kp;
    uint8_t* ws = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), abytes + bbytes + 64, s) != cudaSuccess) {
        cudaGetLastError();
        set_error(QADIC_ERR_CUDA, "matmul_exact_u64: cannot allocate %zu bytes of byte planes", abytes + bbytes);
        return QADIC_ERR_CUDA;
    }
    uint8_t* a8 = ws;
    uint8_t* bt = ws + abytes;
    unsigned long long* dor = reinterpret_cast<unsigned long long*>(ws + abytes + bbytes);
    int* plan = reinterpret_cast<int*>(dor + 2);
    if (!inner) {
        cudaMemsetAsync(dor, 0, 2 * sizeof(unsigned long long), s);
        QADIC_TIMED("u64 or", s, u64_or_kernel<<<1024, 256, 0, s>>>(a, m * k, dor));
        QADIC_TIMED("u64 or", s, u64_or_kernel<<<1024, 256, 0, s>>>(b, k * n, dor + 1));
        QADIC_TIMED("u64 or", s, u64_plan_kernel<<<1, 32, 0, s>>>(dor, plan));
    }
    const bool pair = pair_mode();
    constexpr int BN = Cfg<KIND_I8>::BN;
    int rc = check_launch("u64 prepare");
    for (int64_t k0 = 0; k0 < k && rc == QADIC_OK; k0 += KC) {
        const int64_t kc = (k - k0 < KC) ? k - k0 : KC;
        const int64_t ta = m * (kp / 16);
        QADIC_TIMED("u64 byte planes A", s,
                    u64_aplanes_kernel<<<(unsigned)((ta + 255) / 256), 256, 0, s>>>(a, m, k, k0, kc, nba, kp, a8,
                                                                                    inner ? nullptr : plan));
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)(kp / 128));
        QADIC_TIMED("u64 byte planes B", s, u64_btplanes_kernel<<<grid, 256, 0, s>>>(b, k, n, k0, kc, nbb, kp, bt, inner ? nullptr : plan));
        rc = check_launch("u64 byte planes");
        if (rc) break;
        CUtensorMap ta_map, tb_map;
        rc = make_tmap(&ta_map, a8, nba * kp, m, nba * kp, BM);
        if (rc) break;
        rc = make_tmap(&tb_map, bt, kp, (int64_t)nbb * n, kp, pair ? BN / 2 : BN);
        if (rc) break;
        Params base = {};
        base.M = m;
        base.N = n;
        base.ldc = n;
        base.p = 2;
        base.m_tiles = (int)((m + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM));
        base.n_tiles = (int)((n + BN - 1) / BN);
        base.n_full = (int)(n / BN);
        base.seg_kpb = (int)(kp / BK);
        base.seg_kp = (int)kp;
        // raster group of 8 m tiles (a squarer wave: fewer operand re-reads of the long
        // segmented K from DRAM; 9.62-9.70 vs 9.74-9.76 ms at 8192^3 for 16)
        base.group_m = getenv("QADIC_U64_GROUP_M") ? std::max(1, atoi(getenv("QADIC_U64_GROUP_M"))) : 8;
        base.c64 = c;
        if (inner) {
            // one launch: every shift s of an output tile back to back on one CTA pair
            // (no per-launch tails; C accumulated in program order by the same threads).
            // Measured slower (8192^3: 11.0 vs 10.6 ms): a tile's segments of all shifts
            // spread the operand working set, the shift-major launches reuse one B plane
            // across every m tile in L2.  Opt-in.
            Params prm = base;
            prm.plane_inner = 1;
            prm.planes = nplanes;
            for (int sp = 0; sp < nplanes; ++sp) {
                const int i_lo = sp - (nbb - 1) > 0 ? sp - (nbb - 1) : 0;
                const int i_hi = sp < nba - 1 ? sp : nba - 1;
                prm.seg_lo[sp] = i_lo;
                prm.seg_cnt[sp] = i_hi - i_lo + 1;
            }
            prm.num_kb = prm.seg_cnt[0] * prm.seg_kpb;
            prm.acc64 = k0 > 0 ? 1 : 0;
            rc = pair ? launch_gemm<KIND_I8, true>(ta_map, tb_map, prm, s, "u64 byte-plane gemm")
                      : launch_gemm<KIND_I8, false>(ta_map, tb_map, prm, s, "u64 byte-plane gemm");
            continue;
        }
        for (int sp = 0; sp < nplanes && rc == QADIC_OK; ++sp) {  // one launch per shift (default)
            Params prm = base;
            prm.seg_dev = plan;  // segments of shift sp from the device plan (shift 0 always has one)
            prm.seg_s = sp;
            prm.seg_kpb = base.seg_kpb;
            prm.num_kb = base.seg_kpb;  // placeholder; the kernel derives it
            prm.planes = 1;
            prm.shift = 8 * sp;
            prm.acc64 = (sp > 0 || k0 > 0) ? 1 : 0;
            rc = pair ? launch_gemm<KIND_I8, true>(ta_map, tb_map, prm, s, "u64 byte-plane gemm")
                      : launch_gemm<KIND_I8, false>(ta_map, tb_map, prm, s, "u64 byte-plane gemm");
        }
    }
    cudaFreeAsync(ws, s);
    return rc;
}

// Largest |integer value| of the centred representative e2m1_lut() builds when the
// non-negative set is out of range: v = r for 2r <= p-1, else r - p.  That is p/2
// (not (p-1)/2): for p = 2 residue 1 is stored as -1.  The non-negative set is
// bounded inside e2m1_lut itself (it falls back to this one when K*max^2 >= 2^24).
static int64_t e2m1_max_abs(uint32_t p) {
    int64_t h = 0;
    for (uint32_t r = 0; r < p; ++r) {
        const int64_t v = (2 * r <= p - 1) ? (int64_t)r : (int64_t)r - (int64_t)p;
        h = std::max<int64_t>(h, v < 0 ? -v : v);
    }
    return h;
}

// planes of the decomposition plan_planes() picks (Toom-Cook when 2k-1 <= p+1)
static int kara_planes(uint32_t p, int k) { return (2 * k - 1 <= (int)p + 1) ? 2 * k - 1 : k * (k + 1) / 2; }

bool tc_kara_ok(uint32_t p, int64_t kdim, int k) {
    int ncodes = 1;
    for (int i = 0; i < k; ++i) ncodes *= (int)p;
    const int64_t h = e2m1_max_abs(p);
    return p <= 7 && kara_planes(p, k) <= tc::KMAX_S && ncodes <= tc::PT_CODES &&
           (__int128)kdim * h * h < ((__int128)1 << 24);
}

size_t tc_kara_workspace(uint32_t p, int64_t m, int64_t kdim, int64_t n, int k) {
    tc::KaraLayout L = tc::kara_plan(kara_planes(p, k), m, kdim, n, k);
    return L.tab_bytes + L.a_bytes + L.b_bytes + L.d_bytes;
}

int tc_kara_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                      void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, int reuse) {
    QADIC_REQUIRE(tc_kara_ok(f.p, kdim, (int)f.k), QADIC_ERR_PARAMS,
                  "fp4k engine needs p <= 7, K*h^2 < 2^24 (h = max |centred residue|) and at most %d planes", tc::KMAX_S);
    return tc::run_kara(f, a, b, m, kdim, n, ws, ws_bytes, c, s, reuse);
}

int tc_kara_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                      size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    FieldConst f = {};
    f.p = p;
    f.k = 1;
    f.t = 8;
    f.magic = small_magic(p);
    f.xpow[0][0] = 1;
    return tc_kara_gf_matmul(f, a, b, m, kdim, n, ws, ws_bytes, c, s, 0);
}

// I8K engine: evaluation planes on int8 (p <= 7 for the nibble D planes and the
// SWAR combine; K (p-1)^2 < 2^31 for the int32 accumulator)
bool tc_kara8_ok(uint32_t p, int64_t kdim, int k) {
    int ncodes = 1;
    for (int i = 0; i < k; ++i) ncodes *= (int)p;
    return p <= 7 && kara_planes(p, k) <= tc::KMAX_S && ncodes <= tc::PT_CODES &&
           (__int128)kdim * (p - 1) * (p - 1) < ((__int128)1 << 31);
}

size_t tc_kara8_workspace(uint32_t p, int64_t m, int64_t kdim, int64_t n, int k) {
    return tc::kara8_workspace(kara_planes(p, k), m, kdim, n);
}

int tc_kara8_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                       void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, bool b_ready) {
    QADIC_REQUIRE(tc_kara8_ok(f.p, kdim, (int)f.k), QADIC_ERR_PARAMS,
                  "i8k engine needs p <= 7, K*(p-1)^2 < 2^31 and at most %d planes", tc::KMAX_S);
    return tc::run_kara8(f, a, b, m, kdim, n, ws, ws_bytes, c, s, b_ready);
}

int tc_kara8_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                       size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    FieldConst f = {};
    f.p = p;
    f.k = 1;
    f.t = 8;
    f.magic = small_magic(p);
    f.xpow[0][0] = 1;
    return tc_kara8_gf_matmul(f, a, b, m, kdim, n, ws, ws_bytes, c, s, false);
}

// ---- entry points used by matmul_api.cu ---------------------------------------
size_t tc_workspace(int kind, int64_t m, int64_t kdim, int64_t n, int k) {
    const int64_t Kb = kdim * k;
    const int64_t inner = kind == tc::KIND_I8 ? Kb : (Kb + 1) / 2;
    const int64_t ld = tc::round_up(inner, 16);
    return (size_t)tc::round_up(n * k * ld, 1024) + (size_t)tc::round_up(m * ld, 1024);
}

// F4 needs p <= 7 and an fp32-exact sum of K*k products of the centred representatives
bool tc_f4_ok(uint32_t p, int64_t kdim, int k) {
    if (p > 7) return false;
    const int64_t h = e2m1_max_abs(p);
    return (__int128)kdim * k * h * h < ((__int128)1 << 24);
}

int tc_gf_matmul(int kind, const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                 void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    if (kind == tc::KIND_I8) {
        QADIC_REQUIRE((__int128)kdim * f.k * (f.p - 1) * (f.p - 1) < ((__int128)1 << 31), QADIC_ERR_PARAMS,
                      "inner dimension %lld overflows the int32 plane accumulator", (long long)kdim);
    } else {
        QADIC_REQUIRE(tc_f4_ok(f.p, kdim, (int)f.k), QADIC_ERR_PARAMS,
                      "fp4 engine needs p <= 7 and K*k*h^2 < 2^24 (h = max |centred residue|)");
    }
    return tc::run(kind, f, a, b, m, kdim, n, ws, ws_bytes, c, s);
}

int tc_right_cmm(int kind, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p,
                 void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s) {
    FieldConst f = {};
    f.p = p;
    f.k = 1;
    f.t = 8;
    f.magic = small_magic(p);
    f.xpow[0][0] = 1;
    return tc_gf_matmul(kind, f, a, b, m, kdim, n, ws, ws_bytes, c, s);
}

}  // namespace qadic
