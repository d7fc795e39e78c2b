// Operation-level matmul entry points: bound checks (the reference's
// a-priori conditions, src/params.py:99-141, src/gfext.py:320-325,
// src/cmm.py:170-175) and engine selection.
#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {
int make_field_const(const qadic_field_desc* d, FieldConst* f);
size_t tc_workspace(int kind, int64_t m, int64_t kdim, int64_t n, int k);
bool tc_f4_ok(uint32_t p, int64_t kdim, int k);
int tc_gf_matmul(int kind, const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                 void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s);
int tc_right_cmm(int kind, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p,
                 void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s);
size_t tc_kara_workspace(uint32_t p, int64_t m, int64_t kdim, int64_t n, int k);
bool tc_kara_ok(uint32_t p, int64_t kdim, int k);
int tc_kara_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                      void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s);
int tc_kara_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                      size_t ws_bytes, uint8_t* c, cudaStream_t s);
size_t f64_gf_workspace(int64_t m, int64_t kdim, int64_t n);
size_t f64_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int d);
int f64_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                  int fold, void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s);
int f64_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, int t, int d,
                  void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s);
}  // namespace qadic

using namespace qadic;

// AUTO: the FP4 tensor-core engine when the centred residues are exact E2M1
// values and the fp32 sum is exact (p <= 7), else INT8 (measured: both are
// 10-25x faster than the FP64 engine; FP4 runs the MMA at twice the int8 rate)
static int resolve_engine(int32_t engine, uint32_t p, int64_t kdim, int k) {
    if (engine != QADIC_ENGINE_AUTO) return engine;
    // Karatsuba planes: inner dimension K per plane (the sums never exceed it)
    if (tc_kara_ok(p, kdim, k)) return QADIC_ENGINE_F4K_TC;
    return tc_f4_ok(p, kdim, k) ? QADIC_ENGINE_F4_TC : QADIC_ENGINE_I8_TC;
}
static int tc_kind(int eng) { return eng == QADIC_ENGINE_F4_TC ? 1 : 0; }

extern "C" {

size_t qadic_gf_matmul_workspace(const qadic_field_desc* f, int64_t m, int64_t kdim, int64_t n, int32_t engine) {
    if (!f || m < 0 || kdim < 0 || n < 0) return 0;
    const int eng = resolve_engine(engine, (uint32_t)f->p, kdim, f->k);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_workspace((uint32_t)f->p, m, kdim, n, f->k);
    return eng == QADIC_ENGINE_F64_DMMA ? f64_gf_workspace(m, kdim, n) : tc_workspace(tc_kind(eng), m, kdim, n, f->k);
}

int qadic_gf_matmul_u8(const qadic_field_desc* fd, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim,
                       int64_t n, int32_t engine, int32_t fold_period, void* ws, size_t ws_bytes, uint8_t* c,
                       void* stream) {
    FieldConst f;
    int rc = make_field_const(fd, &f);
    if (rc) return rc;
    QADIC_REQUIRE(m >= 0 && kdim >= 0 && n >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    if (m == 0 || n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (kdim == 0) {
        cudaMemsetAsync(c, 0, (size_t)(m * n * f.k), s);
        return check_launch("gf_matmul (empty K)");
    }
    const int eng = resolve_engine(engine, f.p, kdim, (int)f.k);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_gf_matmul(f, a, b, m, kdim, n, ws, ws_bytes, c, s);
    if (eng == QADIC_ENGINE_I8_TC || eng == QADIC_ENGINE_F4_TC)
        return tc_gf_matmul(tc_kind(eng), f, a, b, m, kdim, n, ws, ws_bytes, c, s);
    QADIC_REQUIRE(eng == QADIC_ENGINE_F64_DMMA, QADIC_ERR_VALUE, "unknown engine %d", engine);
    // accumulation bound of the packed words between folds:
    // carry digit (< p) + span * k * (p-1)^2 must stay below q (polymul.py:159-167)
    const int64_t q = 1ll << f.t;
    const int64_t per = (int64_t)f.k * (f.p - 1) * (f.p - 1);
    if (fold_period <= 0) {
        QADIC_REQUIRE(kdim * per < q, QADIC_ERR_PARAMS,
                      "inner dimension %lld exceeds the digit capacity of q=2**%u; give a fold period",
                      (long long)kdim, f.t);
        fold_period = 0;
    } else {
        QADIC_REQUIRE(fold_period % 4 == 0, QADIC_ERR_VALUE, "F64 fold period must be a multiple of 4 (DMMA k4)");
        QADIC_REQUIRE((int64_t)fold_period * per <= q - 1 - (f.p - 1), QADIC_ERR_PARAMS,
                      "fold period %d exceeds the accumulation budget", fold_period);
        if (kdim <= fold_period) fold_period = 0;
    }
    return f64_gf_matmul(f, a, b, m, kdim, n, fold_period, ws, ws_bytes, c, s);
}

size_t qadic_right_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int64_t p, int32_t d, int32_t engine) {
    if (m < 0 || kdim < 0 || n < 0 || d < 0) return 0;
    const int eng = resolve_engine(engine, (uint32_t)p, kdim, 1);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_workspace((uint32_t)p, m, kdim, n, 1);
    return eng == QADIC_ENGINE_F64_DMMA ? f64_cmm_workspace(m, kdim, n, d) : tc_workspace(tc_kind(eng), m, kdim, n, 1);
}

int qadic_right_cmm_u8(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, int64_t p,
                       int32_t t, int32_t d, int32_t engine, void* ws, size_t ws_bytes, uint8_t* c, void* stream) {
    QADIC_REQUIRE(m >= 0 && kdim >= 0 && n >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    QADIC_REQUIRE(p >= 2 && p <= 127, QADIC_ERR_UNSUPPORTED, "GPU path supports 2 <= p <= 127");
    QADIC_REQUIRE(d >= 0 && t >= 1 && (int64_t)(d + 1) * t <= 53, QADIC_ERR_PARAMS,
                  "q**%d exceeds the 2**53 word budget", d + 1);
    // strict middle-product digit capacity (params.py:112-128) + delayed_sum (params.py:130-141)
    QADIC_REQUIRE((__int128)kdim * (p - 1) * (p - 1) < ((__int128)1 << t), QADIC_ERR_PARAMS,
                  "k_dim=%lld fills or exceeds the digit capacity of q=2**%d", (long long)kdim, t);
    if (m == 0 || n == 0) return QADIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (kdim == 0) {
        cudaMemsetAsync(c, 0, (size_t)(m * n), s);
        return check_launch("right_cmm (empty K)");
    }
    const int eng = resolve_engine(engine, (uint32_t)p, kdim, 1);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_right_cmm(a, b, m, kdim, n, (uint32_t)p, ws, ws_bytes, c, s);
    if (eng == QADIC_ENGINE_I8_TC || eng == QADIC_ENGINE_F4_TC)
        return tc_right_cmm(tc_kind(eng), a, b, m, kdim, n, (uint32_t)p, ws, ws_bytes, c, s);
    QADIC_REQUIRE(eng == QADIC_ENGINE_F64_DMMA, QADIC_ERR_VALUE, "unknown engine %d", engine);
    return f64_right_cmm(a, b, m, kdim, n, (uint32_t)p, t, d, ws, ws_bytes, c, s);
}

}  // extern "C"
