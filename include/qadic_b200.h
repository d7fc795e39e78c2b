/* qadic_b200.h -- C ABI of the B200-native qadic hot path (libqadic_b200.so).
 *
 * Drop-in boundary for the reference package `qadic` (arXiv 0809.0063).
 * Every pointer argument is a DEVICE pointer (cudaMalloc / torch CUDA
 * storage) unless stated otherwise; `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream).  Calls are asynchronous on `stream`
 * and return a qadic_status; a non-zero status leaves a message retrievable
 * with qadic_last_error().  No torch types cross this boundary.
 *
 * Citations are into /root/reference/pkg/src/qadic/ (file:line of the
 * reference interface each entry point replaces).
 */
#ifndef QADIC_B200_H
#define QADIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QADIC_ABI_VERSION 1

#if defined(__GNUC__)
#define QADIC_API __attribute__((visibility("default")))
#else
#define QADIC_API
#endif

typedef enum qadic_status {
    QADIC_OK = 0,
    QADIC_ERR_SHAPE = 1,       /* ValueError("incompatible shapes") _speed.pyx:61-62 / DimensionMismatch errors.py */
    QADIC_ERR_PARAMS = 2,      /* ParamsViolation: a digit or word bound would overflow (params.py:99-141) */
    QADIC_ERR_VALUE = 3,       /* ValueError: argument outside its domain (e.g. d*t >= 64, _speed.pyx:135-136) */
    QADIC_ERR_CUDA = 4,        /* CUDA runtime / launch failure */
    QADIC_ERR_UNSUPPORTED = 5  /* shape or field outside what this build supports */
} qadic_status;

typedef enum qadic_engine {
    QADIC_ENGINE_AUTO = 0,     /* the measured-fastest exact engine: F4K_TC when valid, else I8_TC */
    QADIC_ENGINE_I8_TC = 1,    /* tcgen05.mma kind::i8 on coefficient planes, int32 TMEM accumulators */
    QADIC_ENGINE_F64_DMMA = 2, /* the paper's formulation: DQT-packed FP64 words on DMMA tensor cores */
    QADIC_ENGINE_F4_TC = 3,    /* tcgen05.mma kind::mxf4 (E2M1, unit block scales) on centred residues, p <= 7 */
    QADIC_ENGINE_F4K_TC = 4,   /* F4 on evaluation planes (Toom-Cook over F_p: 2k-1 when 2k-1 <= p+1, else
                                  k(k+1)/2 Karatsuba) + mod-p combine: the fewest MACs */
    QADIC_ENGINE_I8K_TC = 5    /* the same evaluation planes on tcgen05 kind::i8 (residues as int8, int32
                                  TMEM accumulators), p <= 7 */
} qadic_engine;

/* Flags OR-ed into the engine argument of qadic_gf_matmul_u8 for a caller that sweeps
 * column panels of B against one A on one stream and workspace (the multi-GPU
 * row-block step): COL_PANEL on the first panel, A_READY on the later ones -- the
 * FP4K engine then keeps A's evaluation planes in the workspace instead of
 * re-converting A per panel.  Other engines ignore them. */
#define QADIC_ENGINE_FLAG_COL_PANEL 0x100
#define QADIC_ENGINE_FLAG_A_READY 0x200
/* F64_DMMA engine: force the two-sided DQT form with in-register REDQ folds every
 * fold_period terms (the paper's schedule; AUTO takes the one-sided form when the
 * fold period is below 64, where the folds make the two-sided form ALU-bound). */
#define QADIC_ENGINE_FLAG_F64_TWO_SIDED 0x400

QADIC_API int qadic_abi_version(void);
QADIC_API const char *qadic_last_error(void);
/* number of kernels this library launched since load (instrumentation) */
QADIC_API int64_t qadic_launch_count(void);
/* per-kernel CUDA-event timing on the launching stream (instrumentation):
 * enable, run, then collect "name,count,total_ms" lines (synchronises). */
QADIC_API void qadic_profile_enable(int on);
QADIC_API int qadic_profile_collect(char *buf, size_t len);

/* ---------------------------------------------------------------------------
 * Layer K: the operator/plugin kernels (_kernels/__init__.py:52-69).
 * Semantics identical to _kernels/_speed.pyx (uint64 wraps mod 2^64).
 * ------------------------------------------------------------------------- */

/* C[m,n] = A[m,k] @ B[k,n] over uint64 mod 2^64.  _speed.pyx:15-30, 58-66.
 * Large shapes run on INT8 tensor cores through byte planes; the operands'
 * significant byte counts are found on the device (no host synchronisation), so the
 * call is asynchronous on `stream` and may be captured in a CUDA graph. */
QADIC_API int qadic_matmul_exact_u64(const uint64_t *a, const uint64_t *b, uint64_t *c,
                           int64_t m, int64_t k, int64_t n, void *stream);

/* C = A @ B mod p, reducing every `chunk` inner steps (floor-mod, int64).
 * _speed.pyx:33-55, 69-82 ; pure.py:20-28 */
QADIC_API int qadic_matmul_mod_i64(const int64_t *a, const int64_t *b, int64_t *c,
                         int64_t m, int64_t k, int64_t n, int64_t p, int64_t chunk,
                         void *stream);

/* out[na+nb-1] = full convolution.  _speed.pyx:85-92,105-110 / 95-102,113-118 */
QADIC_API int qadic_conv_exact_u64(const uint64_t *a, int64_t na, const uint64_t *b, int64_t nb,
                         uint64_t *out, void *stream);
QADIC_API int qadic_conv_exact_i64(const int64_t *a, int64_t na, const int64_t *b, int64_t nb,
                         int64_t *out, void *stream);

/* out[n, d+1]: u_i = (r >> it) - p*((r//p) >> it).  _speed.pyx:121-140.
 * The division is an FP64 reciprocal multiply (fdiv.py:338-363) for r < 2^53,
 * integer division above. */
QADIC_API int qadic_redq_compress_u64(const uint64_t *r, int64_t n, int64_t p, int32_t t, int32_t d,
                            uint64_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * REDQ bulk reduction (redq.py:318-343): compress + correct, then either
 * repack (packed_out[n]) or emit digits (digits_out[n, d+1], uint64).
 * Either output may be NULL.
 * ------------------------------------------------------------------------- */
QADIC_API int qadic_reduce_words(const uint64_t *words, int64_t n, int64_t p, int32_t t, int32_t d,
                       uint64_t *packed_out, uint64_t *digits_out, void *stream);

/* ---------------------------------------------------------------------------
 * DQT pack / unpack (dqt.py:39-92, cmm.py:72-85,130-145, polymul.py:126-151).
 * ------------------------------------------------------------------------- */

/* words[rows, ceil(cols/k)] = row-packed (FORWARD, reverse=0) or digit-reversed
 * (REVERSED, reverse=1) groups of k consecutive uint8 entries, zero-padded. */
QADIC_API int qadic_pack_rows_u8(const uint8_t *m, int64_t rows, int64_t cols, int32_t k, int32_t t,
                       int32_t reverse, uint64_t *words, void *stream);
/* inverse of qadic_pack_rows_u8 for reduced digits: out[rows, cols] uint8 */
QADIC_API int qadic_unpack_rows_u8(const uint64_t *words, int64_t rows, int64_t cols, int32_t k,
                         int32_t t, int32_t reverse, uint8_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * GF(p^k) field description shared by the GF entry points.
 * Built on the host from GFqField (gfext.py:103-213): L/H correction tables
 * (gfext.py:176-213) are re-expressed with coefficient bytes instead of
 * discrete-log handles (entry = sum coeff_l << 8l), and the fold rows
 * xpow[i] = X^i mod f (gfext.py:200-205) drive the INT8 plane expansion.
 * ------------------------------------------------------------------------- */
typedef struct qadic_field_desc {
    int32_t p;                /* prime, 2 <= p <= 127 on the GPU path */
    int32_t k;                /* extension degree, 1 <= k <= 4 */
    int32_t t;                /* radix exponent, q = 2^t */
    int32_t u_bits;           /* ceil(log2 p): L/H index bits per digit (gfext.py:178) */
    uint8_t xpow[7][4];       /* X^i mod f coefficients, i = 0..2k-2 */
    const uint32_t *l_table;  /* device, 2^(u_bits*k) entries */
    const uint32_t *h_table;  /* device, 2^(u_bits*k) entries */
} qadic_field_desc;

/* cfg2 -- out[batch, k] = sum_j v1[b,j]*v2[b,j] over GF(p^k), coefficient I/O
 * (uint8 [batch, len, k]).  GFqField.fgdp, gfext.py:268-297, batched. */
QADIC_API int qadic_gf_dot_batch_u8(const qadic_field_desc *f, const uint8_t *v1, const uint8_t *v2,
                          int64_t batch, int64_t len, uint8_t *out, void *stream);

/* The same dot products in the paper's accumulation form: every element packed
 * into a DQT word held in a double, the packed products summed by DFMA (exact: every
 * sum < 2^53), then REDQ + L/H.  Bit-identical to qadic_gf_dot_batch_u8 (which sums
 * the packed product's digits on the coefficient bytes instead); k = 3 rows use the
 * digit-sum form. */
QADIC_API int qadic_gf_dot_batch_f64_u8(const qadic_field_desc *f, const uint8_t *v1, const uint8_t *v2,
                                        int64_t batch, int64_t len, uint8_t *out, void *stream);

/* cfg3 / cfg5 -- C[m,n,k] = A[m,kdim,k] @ B[kdim,n,k] over GF(p^k), coefficient
 * I/O.  GFqField.matmul, gfext.py:311-345.  fold_period (F64 engine only) is the
 * number of inner terms accumulated between in-register REDQ folds (0 = none,
 * requires kdim <= the field's dot bound); the INT8 engine needs no folds while
 * kdim*k*(p-1)^2 < 2^31.  `workspace` must hold qadic_gf_matmul_workspace()
 * bytes (device). */
QADIC_API size_t qadic_gf_matmul_workspace(const qadic_field_desc *f, int64_t m, int64_t kdim, int64_t n,
                                 int32_t engine);
QADIC_API int qadic_gf_matmul_u8(const qadic_field_desc *f, const uint8_t *a, const uint8_t *b,
                       int64_t m, int64_t kdim, int64_t n, int32_t engine, int32_t fold_period,
                       void *workspace, size_t workspace_bytes, uint8_t *c, void *stream);

/* cfg3 / cfg5 end to end -- the same product with HOST operands (pinned or
 * pageable; any of a, b, c may also be a device pointer).  B is copied once,
 * A and C move in row panels of `panel_rows` (0 = about sixteen panels) on two
 * internal copy streams, so the H2D of panel i+1, the compute of panel i and the
 * D2H of panel i-1 overlap.  Work is ordered on `stream`: when it completes, c
 * holds the result.  `workspace` (device) must hold
 * qadic_gf_matmul_host_workspace() bytes.  Replaces the host round trip around
 * GFqField.matmul (gfext.py:311-345) that a caller with numpy arrays makes. */
QADIC_API size_t qadic_gf_matmul_host_workspace(const qadic_field_desc *f, int64_t m, int64_t kdim, int64_t n,
                                                int32_t engine, int64_t panel_rows);
QADIC_API int qadic_gf_matmul_host_u8(const qadic_field_desc *f, const uint8_t *a, const uint8_t *b,
                                      int64_t m, int64_t kdim, int64_t n, int32_t engine, int32_t fold_period,
                                      int64_t panel_rows, void *workspace, size_t workspace_bytes, uint8_t *c,
                                      void *stream);

/* cfg4 -- C[m,n] = A[m,kdim] @ B[kdim,n] mod p with B row-compressed d+1
 * entries per word at radix 2^t (cmm.right_cmm(a, compress_rows(b)),
 * cmm.py:244-276, 97-110).  uint8 I/O. */
QADIC_API size_t qadic_right_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int64_t p, int32_t d,
                                           int32_t engine);
QADIC_API int qadic_right_cmm_u8(const uint8_t *a, const uint8_t *b, int64_t m, int64_t kdim, int64_t n,
                       int64_t p, int32_t t, int32_t d, int32_t engine, void *workspace,
                       size_t workspace_bytes, uint8_t *c, void *stream);

/* cfg1 -- out[n, 2k-1] = a[n,k] * b[n,k] over F_p for n independent pairs:
 * one packed product + simultaneous reduction per pair.  polymul.polymul_fqt,
 * polymul.py:274-313 (one word per operand), batched.  For k = 4 and
 * 4 (p-1)^2 <= 255 (p = 2, 3, 5) the transform runs at q = 2^8 whatever t says: the
 * DQT word of an operand is its four coefficient bytes, the packed product one
 * 32 x 32 -> 64-bit multiply, and all digits are reduced at once by a byte-lane
 * reciprocal multiply (no correction step: byte-aligned digits do not borrow).  The
 * result is the same for every admissible q. */
QADIC_API int qadic_polymul_batch_u8(const uint8_t *a, const uint8_t *b, int64_t n, int32_t k, int64_t p,
                           int32_t t, uint8_t *out, void *stream);

/* The same products always in the paper's form: DQT words at q = 2^t, one packed
 * product per pair, REDQ with the FP64 reciprocal (fdiv.py:66-93) and the correction
 * pass (redq.py:118-143).  Bit-identical to qadic_polymul_batch_u8. */
QADIC_API int qadic_polymul_batch_redq_u8(const uint8_t *a, const uint8_t *b, int64_t n, int32_t k, int64_t p,
                                int32_t t, uint8_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * Handle conversion for the discrete-log API (gfext.py:43-46, 136-146):
 *   out[i*width + j] = table[idx[i]*width + j]        (index -> coefficients)
 *   out[i] = index_of_code[sum_l c[i,l] p^l]           (coefficients -> index)
 * ------------------------------------------------------------------------- */
QADIC_API int qadic_gather_u8(const int64_t *idx, int64_t n, const uint8_t *table, int64_t table_rows,
                    int32_t width, uint8_t *out, void *stream);
QADIC_API int qadic_index_of_coeffs(const uint8_t *c, int64_t n, int32_t k, int32_t p,
                          const int64_t *index_of_code, int64_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * Long-polynomial products on packed words (csrc/polymul_long.cu):
 * polymul.polymul_fqt / _wordconv_reduce / _kara_words (polymul.py:159-313) for a
 * batch of pairs.  aw [batch][na], bw [batch][nb]: packed words (k = d+1 digits at
 * radix 2^t, digits <= ma / mb); a REDQ fold every (2^t - 1 - (p-1)) / (k ma mb)
 * inner terms, final REDQ, overlap-add mod p into out [batch][ncoef] (uint8 when
 * out_u8, else int64).  algo 0 = classical, 1 = Karatsuba (breadth-first levels
 * while n > threshold words).  stats (optional, host): the schedule's word
 * products and reductions; flags bit 0 = a value beyond the top digit (validate),
 * bit 1 = a nonzero coefficient at or beyond ncoef.  Asynchronous on `stream`
 * unless stats is given (the flags are read back: synchronous).
 * ------------------------------------------------------------------------- */
typedef struct qadic_polymul_stats {
    int64_t word_muls;
    int64_t reductions;
    int64_t leaves;
    int32_t levels;
    uint32_t flags;
} qadic_polymul_stats;
QADIC_API int qadic_polymul_words_batch(const uint64_t *aw, int64_t na, const uint64_t *bw, int64_t nb,
                                        int64_t batch, int64_t p, int32_t t, int32_t d, int64_t ma, int64_t mb,
                                        int32_t algo, int64_t threshold, int32_t validate, int32_t out_u8,
                                        void *out, int64_t ncoef, qadic_polymul_stats *stats, void *stream);

/* The same batched products on INT8 tensor cores (p <= 127, uint8 residues):
 * out[s][y] = sum_x a[s][x] b[s][y-x] mod p as one batched Toeplitz GEMM (T_s[x][l] =
 * a_s[x-l], 128 columns; b_s as 128-coefficient blocks; mod-p epilogue) plus an
 * overlap-add.  out [batch][ncoef] uint8 (positions past na+nb-2 are zero);
 * `workspace` (device) must hold qadic_polymul_tc_workspace() bytes.  Asynchronous. */
QADIC_API size_t qadic_polymul_tc_workspace(int64_t batch, int64_t na, int64_t nb);
QADIC_API int qadic_polymul_tc_u8(const uint8_t *a, int64_t na, const uint8_t *b, int64_t nb, int64_t batch,
                                  int64_t p, uint8_t *out, int64_t ncoef, void *workspace, size_t ws_bytes,
                                  void *stream);

/* ---------------------------------------------------------------------------
 * Any-field DQT word path (csrc/generic.cu): the reference's composition for the
 * fields / primes outside the uint8 coefficient engines (p > 127, k > 4, wide
 * L/H tables).  Handles are int64 (gfext.py:43-46), words uint64; the word
 * product itself is qadic_matmul_exact_u64 (INT8 byte-plane tensor cores).
 * ------------------------------------------------------------------------- */
typedef struct qadic_gf_generic_desc {
    int64_t p;                    /* prime < 2^26 */
    int32_t k;                    /* extension degree, p^k <= 2^22 */
    int32_t t;                    /* radix exponent: (2k-1) t <= 64 */
    int32_t u_bits;               /* ceil(log2 p) bits per digit of the L/H index (gfext.py:178) */
    int32_t reserved;
    const int32_t *l_code;        /* device: code_of_index[l_table], 2^(u_bits k) entries */
    const int32_t *h_code;        /* device: code_of_index[h_table] */
    const int64_t *index_of_code; /* device: p^k entries */
} qadic_gf_generic_desc;

/* out[i] = table[idx[i]]  (pack_table gather, gfext.py:329-330) */
QADIC_API int qadic_gather_u64(const int64_t *idx, int64_t n, const uint64_t *table, uint64_t *out, void *stream);
/* acc[b] = sum_j pack[v1[b,j]] * pack[v2[b,j]] (uint64; GFqField.fgdp's word dot,
 * gfext.py:287-290, batched over rows) */
QADIC_API int qadic_gf_words_dot(const int64_t *v1, const int64_t *v2, int64_t rows, int64_t len,
                                 const uint64_t *pack, uint64_t *acc, void *stream);
/* handles[i] = L[u_0..u_{k-1}] + H[u_{k-1}..u_{2k-2}] with u = REDQ digits of acc[i]
 * (gfext.py:291-296, 331-358: compress, L/H lookups, addition on codes) */
QADIC_API int qadic_gf_words_finish(const uint64_t *acc, int64_t n, const qadic_gf_generic_desc *f,
                                    int64_t *out, void *stream);
/* int64 entries (any value < 2^t) <-> packed words; cmm.py:72-85 / 130-145 */
QADIC_API int qadic_pack_rows_i64(const int64_t *m, int64_t rows, int64_t cols, int32_t k, int32_t t,
                                  int32_t reverse, uint64_t *words, void *stream);
QADIC_API int qadic_unpack_rows_i64(const uint64_t *words, int64_t rows, int64_t cols, int32_t k, int32_t t,
                                    int32_t reverse, int64_t *out, void *stream);
/* out[i] = ((acc[i] >> d t) & (2^t - 1)) mod p  (cmm_multiply's middle digit, cmm.py:200-204) */
QADIC_API int qadic_extract_middle(const uint64_t *acc, int64_t n, int64_t p, int32_t t, int32_t d, int64_t *out,
                                   void *stream);
/* full_cmm's one REDQ per word over the (dq+1)(dth+1)-digit grid, corrected digits
 * scattered to out[m, n] (cmm.py:349-359) */
QADIC_API int qadic_full_cmm_reduce(const uint64_t *acc, int64_t mw, int64_t nw, int64_t p, int32_t t, int32_t dq,
                                    int32_t dth, int64_t m, int64_t n, int64_t *out, void *stream);
/* Tabulated correction over a batch (build_correction_table / correct_tabulated,
 * redq.py:194-300): digits of words[i] (REDQ-compressed at radix 2^t) -- or the
 * given compressed digits[i, 0..d] -- corrected by overlapping width-j block
 * lookups in `table` (entries packed ceil(log2 p) bits per residue; base_p != 0:
 * index sum u_i p^i, else the bit-block index); out[n, d+1].  Give exactly one of
 * words / digits. */
QADIC_API int qadic_redq_tabulated(const uint64_t *words, const uint64_t *digits, int64_t n, int64_t p, int32_t t,
                                   int32_t d, const uint64_t *table, int64_t table_entries, int32_t j,
                                   int32_t base_p, uint64_t *out, void *stream);
/* correct_digits_array (redq.py:308-315): mu_i = (u_i + c u_{i+1}) mod p (uint64 wrap),
 * c = (p - q mod p) mod p, top digit kept; identity when q mod p == 0 */
QADIC_API int qadic_correct_digits(const uint64_t *u, int64_t n, int32_t width, int64_t p, int64_t q_mod_p,
                                   uint64_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * FDIV certification scans (fdiv.exhaustive_check / applied_fdiv_exhaustive,
 * fdiv.py:405-461; Table 1, Alg. 4).
 * Every (r, p) in [0, 2^beta) x [1, 2^beta) in beta-bit binary arithmetic:
 * x = round2(r * round1(1/p)), diff = floor(x) - r // p.  Modes: 0 = up,
 * 1 = nearest (ties to even), 2 = down (the reference's _MODE_ORDER).
 * `out` / `mismatches` are HOST pointers; the call returns when they are
 * filled (synchronous on `stream`).  beta in 4..22 (the reference: 4..16).
 * ------------------------------------------------------------------------- */
typedef struct qadic_fdiv_scan_report {
    uint64_t pairs_checked;
    uint64_t range_violations;     /* diff outside [range_lo, range_hi] */
    uint64_t bound_violations;     /* diff > 0 with r <= bound_threshold */
    int64_t k_minus_1_r, k_minus_1_p; /* first (p-major) pair with diff = -1 when range_lo = -1; else -1 */
    int64_t k_plus_1_r, k_plus_1_p;   /* first (p-major) pair with diff = +1 when range_hi = 1; else -1 */
    int64_t smallest_overflow_r;      /* least r with diff > 0 over all p, -1 if none */
} qadic_fdiv_scan_report;

/* one case (mode1, mode2): bound_threshold < 0 means the case has no bound */
QADIC_API int qadic_fdiv_scan(int32_t beta, int32_t mode1, int32_t mode2, int32_t range_lo, int32_t range_hi,
                              int64_t bound_threshold, qadic_fdiv_scan_report *out, void *stream);
/* Alg. 4 for the three paired cases (mode2 = up / nearest / down with the
 * reciprocal mode fdiv._PAIRED_MODE1 gives): y -= (r >= bound[mode2] && p*y > r),
 * counts y != r // p over all (r, p, mode2). */
QADIC_API int qadic_fdiv_applied_scan(int32_t beta, const int64_t bound[3], uint64_t *mismatches, void *stream);
/* Native binary64 applied division on sampled pairs (fdiv.native_applied_random,
 * reference src/fdiv.py:464-488): r[j*per_p + i] against divisor p[j] with
 * invp[j] = RU(1/p[j]); y = floor(RN(r*invp)) - (r > threshold && p*y > r);
 * counts y != r // p.  Device pointers; synchronous (returns the count). */
QADIC_API int qadic_fdiv_native_check(const int64_t *r, int64_t per_p, const int64_t *p, const double *invp,
                                      int64_t n_p, int64_t threshold, uint64_t *mismatches, void *stream);

/* ---------------------------------------------------------------------------
 * Diagnostics: measured pipe peaks (no reference
 * counterpart).  Runs one on-chip probe (operands in shared memory / registers,
 * no memory traffic) and returns the operations executed (*ops: 2 per MAC) and
 * the event-timed duration (*ms); synchronous on `stream`.
 *   kind 0: tcgen05.mma cta_group::2 kind::mxf4.block_scale (M256 N256 K64)
 *   kind 1: tcgen05.mma cta_group::2 kind::i8 (M256 N256 K32)
 *   kind 2: mma.sync m8n8k4 f64 (DMMA)
 *   data 0: zero operands, 1: residue-like operands (what the engines feed), 2: random bits
 * ------------------------------------------------------------------------- */
QADIC_API int qadic_diag_pipe_peak(int32_t kind, int32_t data, int64_t iters, double *ops, float *ms, void *stream);
/* Host-only: the byte-lane quotient constants qadic_polymul_batch_u8 uses for prime p
 * and digits <= dmax (s = ((v * m) >> sh) on every byte lane): returns 1 when
 * d - p * ((d * m) >> sh) lies in [0, p) for every d <= dmax, 2 when in [0, 2p), 0 when no
 * pair with dmax * m <= 255 exists.  No device work (CPU-testable). */
QADIC_API int qadic_diag_lane_quotient(uint32_t p, uint32_t dmax, uint32_t *m, uint32_t *sh);
/* Same-size copy ceiling of the single-wave batched kernels: out = a ^ b over
 * 16-byte vectors (two input streams of in_bytes, one output stream of out_bytes
 * <= 2 in_bytes), per_thread vectors of each input per thread (1, 2, 4, 8), one
 * launch with programmatic dependent launch like the cfg1 / cfg2 kernels. */
QADIC_API int qadic_diag_copy(const void *a, const void *b, int64_t in_bytes, void *out, int64_t out_bytes,
                              int32_t per_thread, int32_t threads, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QADIC_B200_H */
