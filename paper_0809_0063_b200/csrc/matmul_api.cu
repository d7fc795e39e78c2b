// Operation-level matmul entry points: bound checks (the reference's
// a-priori conditions, src/params.py:99-141, src/gfext.py:320-325,
// src/cmm.py:170-175) and engine selection.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "qadic_common.cuh"
#include "qadic_internal.h"
#include "host_stage.h"

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
                      void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, int reuse);
int tc_kara_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                      size_t ws_bytes, uint8_t* c, cudaStream_t s);
bool tc_kara8_ok(uint32_t p, int64_t kdim, int k);
size_t tc_kara8_workspace(uint32_t p, int64_t m, int64_t kdim, int64_t n, int k);
int tc_kara8_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                       void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, bool b_ready);
int tc_kara8_right_cmm(const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n, uint32_t p, void* ws,
                       size_t ws_bytes, uint8_t* c, cudaStream_t s);
size_t f64_gf_workspace(int64_t m, int64_t kdim, int64_t n, int k);
size_t f64_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int d);
int f64_gf_matmul(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                  int fold, void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s, bool two_sided);
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

// device-pointer GF(p^k) matmul on the resolved engine; reuse (REUSE_* bits, fp4k
// engine): B planes already in `ws` (row panels of one host call), or the
// column-panel layout with A planes already in `ws`
static int gf_matmul_dev(const FieldConst& f, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim, int64_t n,
                         int32_t engine, int32_t fold_period, void* ws, size_t ws_bytes, uint8_t* c, cudaStream_t s,
                         int reuse) {
    const bool b_ready = reuse & REUSE_B_READY;
    const int eng = resolve_engine(engine, f.p, kdim, (int)f.k);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_gf_matmul(f, a, b, m, kdim, n, ws, ws_bytes, c, s, reuse);
    if (eng == QADIC_ENGINE_I8K_TC) return tc_kara8_gf_matmul(f, a, b, m, kdim, n, ws, ws_bytes, c, s, b_ready);
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
    return f64_gf_matmul(f, a, b, m, kdim, n, fold_period, ws, ws_bytes, c, s, (reuse & F64_TWO_SIDED) != 0);
}

extern "C" {

size_t qadic_gf_matmul_workspace(const qadic_field_desc* f, int64_t m, int64_t kdim, int64_t n, int32_t engine) {
    if (!f || m < 0 || kdim < 0 || n < 0) return 0;
    engine &= 0xff;
    const int eng = resolve_engine(engine, (uint32_t)f->p, kdim, f->k);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_workspace((uint32_t)f->p, m, kdim, n, f->k);
    if (eng == QADIC_ENGINE_I8K_TC) return tc_kara8_workspace((uint32_t)f->p, m, kdim, n, f->k);
    return eng == QADIC_ENGINE_F64_DMMA ? f64_gf_workspace(m, kdim, n, f->k)
                                        : tc_workspace(tc_kind(eng), m, kdim, n, f->k);
}

int qadic_gf_matmul_u8(const qadic_field_desc* fd, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim,
                       int64_t n, int32_t engine, int32_t fold_period, void* ws, size_t ws_bytes, uint8_t* c,
                       void* stream) {
    // column-panel sweep flags (QADIC_ENGINE_FLAG_*) ride on the engine argument
    int reuse = 0;
    if (engine & QADIC_ENGINE_FLAG_COL_PANEL) reuse |= REUSE_COL_PANEL;
    if (engine & QADIC_ENGINE_FLAG_A_READY) reuse |= REUSE_COL_PANEL | REUSE_A_READY;
    if (engine & QADIC_ENGINE_FLAG_F64_TWO_SIDED) reuse |= F64_TWO_SIDED;
    engine &= 0xff;
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
    return gf_matmul_dev(f, a, b, m, kdim, n, engine, fold_period, ws, ws_bytes, c, s, reuse);
}

size_t qadic_right_cmm_workspace(int64_t m, int64_t kdim, int64_t n, int64_t p, int32_t d, int32_t engine) {
    if (m < 0 || kdim < 0 || n < 0 || d < 0) return 0;
    const int eng = resolve_engine(engine, (uint32_t)p, kdim, 1);
    if (eng == QADIC_ENGINE_F4K_TC) return tc_kara_workspace((uint32_t)p, m, kdim, n, 1);
    if (eng == QADIC_ENGINE_I8K_TC) return tc_kara8_workspace((uint32_t)p, m, kdim, n, 1);
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
    if (eng == QADIC_ENGINE_I8K_TC) return tc_kara8_right_cmm(a, b, m, kdim, n, (uint32_t)p, ws, ws_bytes, c, s);
    if (eng == QADIC_ENGINE_I8_TC || eng == QADIC_ENGINE_F4_TC)
        return tc_right_cmm(tc_kind(eng), a, b, m, kdim, n, (uint32_t)p, ws, ws_bytes, c, s);
    QADIC_REQUIRE(eng == QADIC_ENGINE_F64_DMMA, QADIC_ERR_VALUE, "unknown engine %d", engine);
    return f64_right_cmm(a, b, m, kdim, n, (uint32_t)p, t, d, ws, ws_bytes, c, s);
}

// ---- host-buffer pipeline ---------------------------------------------------------
// C = A B with host (or mixed host/device) operands: B is copied once, A and C
// travel in row panels on two copy streams so that H2D of panel i+1, the
// compute of panel i and the D2H of panel i-1 overlap (PCIe is full duplex).
// Device scratch: [engine workspace for one panel | B | 2 A panels | 2 C panels].
// Pageable (unregistered) host operands go through pinned slots (host_stage.cu):
// the host thread copies panel i in and panel i-3 out while the device works,
// so such a call returns with the result in place (a pageable DMA would be
// synchronous anyway).

static int64_t host_panel_rows(int64_t m, int64_t panel_rows) {
    // default ~12 panels of >= 256 rows (measured at cfg5: 768-row panels 8.6 ms
    // pinned / ~13-15 ms pageable, against 8.8 / ~15-19 ms with 512 rows)
    int64_t pr = panel_rows > 0 ? panel_rows : ((m + 11) / 12 + 127) / 128 * 128;
    if (panel_rows <= 0 && pr < 256) pr = 256;
    if (pr < 1) pr = 1;
    return pr < m ? pr : m;
}
static size_t align_up(size_t x) { return (x + 1023) / 1024 * 1024; }

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct CopyStreams {
    cudaStream_t h2d = nullptr, d2h = nullptr;
};
static CopyStreams& copy_streams() {
    static CopyStreams cs[64];
    int dev = 0;
    cudaGetDevice(&dev);
    CopyStreams& c = cs[dev & 63];
    if (!c.h2d) {
        cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking);
    }
    return c;
}

size_t qadic_gf_matmul_host_workspace(const qadic_field_desc* f, int64_t m, int64_t kdim, int64_t n, int32_t engine,
                                      int64_t panel_rows) {
    if (!f || m < 0 || kdim < 0 || n < 0) return 0;
    engine &= 0xff;
    const int64_t pr = host_panel_rows(m, panel_rows);
    const int64_t k = f->k;
    return align_up(qadic_gf_matmul_workspace(f, pr, kdim, n, engine)) + align_up((size_t)(kdim * n * k)) +
           2 * align_up((size_t)(pr * kdim * k)) + 2 * align_up((size_t)(pr * n * k));
}

int qadic_gf_matmul_host_u8(const qadic_field_desc* fd, const uint8_t* a, const uint8_t* b, int64_t m, int64_t kdim,
                            int64_t n, int32_t engine, int32_t fold_period, int64_t panel_rows, void* ws,
                            size_t ws_bytes, uint8_t* c, void* stream) {
    const int eflags = (engine & QADIC_ENGINE_FLAG_F64_TWO_SIDED) ? F64_TWO_SIDED : 0;
    engine &= 0xff;
    FieldConst f;
    int rc = make_field_const(fd, &f);
    if (rc) return rc;
    QADIC_REQUIRE(m >= 0 && kdim >= 0 && n >= 0, QADIC_ERR_SHAPE, "incompatible shapes");
    if (m == 0 || n == 0) return QADIC_OK;
    QADIC_REQUIRE(a && b && c, QADIC_ERR_VALUE, "null operand");
    const int64_t k = f.k;
    const int64_t pr = host_panel_rows(m, panel_rows);
    const size_t need = qadic_gf_matmul_host_workspace(fd, m, kdim, n, engine, panel_rows);
    QADIC_REQUIRE(ws != nullptr && ws_bytes >= need, QADIC_ERR_VALUE, "workspace too small (%zu < %zu)", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    const bool a_dev = is_device_ptr(a), b_dev = is_device_ptr(b), c_dev = is_device_ptr(c);
    const size_t eng_ws = align_up(qadic_gf_matmul_workspace(fd, pr, kdim, n, engine));
    uint8_t* base = static_cast<uint8_t*>(ws);
    uint8_t* bbuf = base + eng_ws;
    uint8_t* abuf[2] = {bbuf + align_up((size_t)(kdim * n * k)), nullptr};
    abuf[1] = abuf[0] + align_up((size_t)(pr * kdim * k));
    uint8_t* cbuf[2] = {abuf[1] + align_up((size_t)(pr * kdim * k)), nullptr};
    cbuf[1] = cbuf[0] + align_up((size_t)(pr * n * k));
    CopyStreams& cs = copy_streams();
    const int64_t panels = (m + pr - 1) / pr;
    static const bool no_stage = std::getenv("QADIC_NO_STAGE") != nullptr;
    const bool a_st = !no_stage && !a_dev && kdim > 0 && is_pageable(a);
    const bool b_st = !no_stage && !b_dev && kdim > 0 && is_pageable(b);
    const bool c_st = !no_stage && !c_dev && is_pageable(c);
    std::unique_ptr<StageLease> st;
    if (a_st || b_st || c_st) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        QADIC_REQUIRE(cap == cudaStreamCaptureStatusNone, QADIC_ERR_VALUE,
                      "pageable host operands cannot be captured in a CUDA graph (use pinned or device buffers)");
        st.reset(new StageLease(std::max((size_t)(pr * kdim * k), (size_t)(pr * n * k))));
        QADIC_REQUIRE(st->ok(), QADIC_ERR_CUDA, "pinned staging buffer allocation failed");
    }
    std::vector<cudaEvent_t> evs;
    auto event = [&]() {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        evs.push_back(e);
        return e;
    };
    auto after = [&](cudaStream_t waiter, cudaStream_t producer) {
        cudaEvent_t e = event();
        cudaEventRecord(e, producer);
        cudaStreamWaitEvent(waiter, e, 0);
        return e;
    };
    // the scratch buffers may still be in use by earlier work on s
    after(cs.h2d, s);
    after(cs.d2h, s);
    const uint8_t* bsrc = b;
    if (b_st) {  // B in slot-sized chunks through the input slots
        const size_t tot = (size_t)(kdim * n * k), ch = (size_t)std::max(pr * kdim * k, pr * n * k);
        for (size_t off = 0, j = 0; off < tot; off += ch, ++j)
            st->h2d((int)(j % kStageIn), bbuf + off, b + off, std::min(ch, tot - off), cs.h2d);
        bsrc = bbuf;
        after(s, cs.h2d);
    } else if (!b_dev && kdim > 0) {
        cudaMemcpyAsync(bbuf, b, (size_t)(kdim * n * k), cudaMemcpyHostToDevice, cs.h2d);
        bsrc = bbuf;
        after(s, cs.h2d);
    }
    std::vector<cudaEvent_t> done_c(panels), done_d(panels);
    auto d2h = [&](int64_t i) {
        const int64_t r0 = i * pr, rows = (r0 + pr <= m ? pr : m - r0);
        cudaStreamWaitEvent(cs.d2h, done_c[i], 0);
        uint8_t* dst = c_st ? st->slot(kStageIn + (int)(i % kStageIn)) : c + r0 * n * k;
        cudaMemcpyAsync(dst, cbuf[i & 1], (size_t)(rows * n * k), cudaMemcpyDeviceToHost, cs.d2h);
        done_d[i] = event();
        cudaEventRecord(done_d[i], cs.d2h);
    };
    auto unstage = [&](int64_t i) {  // pinned slot -> caller's pageable C (host waits for the D2H)
        const int64_t r0 = i * pr, rows = (r0 + pr <= m ? pr : m - r0);
        cudaEventSynchronize(done_d[i]);
        parallel_copy(c + r0 * n * k, st->slot(kStageIn + (int)(i % kStageIn)), (size_t)(rows * n * k));
    };
    for (int64_t i = 0; i < panels && rc == QADIC_OK; ++i) {
        const int64_t r0 = i * pr, rows = (r0 + pr <= m ? pr : m - r0);
        const uint8_t* ap = a + r0 * kdim * k;
        if (!a_dev && kdim > 0) {
            if (i >= 2) cudaStreamWaitEvent(cs.h2d, done_c[i - 2], 0);  // panel i-2 no longer reads this buffer
            if (a_st)
                st->h2d((int)(i % kStageIn), abuf[i & 1], ap, (size_t)(rows * kdim * k), cs.h2d);
            else
                cudaMemcpyAsync(abuf[i & 1], ap, (size_t)(rows * kdim * k), cudaMemcpyHostToDevice, cs.h2d);
            ap = abuf[i & 1];
            after(s, cs.h2d);
        }
        uint8_t* cp = c_dev ? c + r0 * n * k : cbuf[i & 1];
        if (!c_dev && i >= 2) cudaStreamWaitEvent(s, done_d[i - 2], 0);  // its D2H has drained this buffer
        if (kdim == 0) {
            cudaMemsetAsync(cp, 0, (size_t)(rows * n * k), s);
            rc = check_launch("gf_matmul_host (empty K)");
        } else {
            rc = gf_matmul_dev(f, ap, bsrc, rows, kdim, n, engine, fold_period, base, eng_ws, cp, s,
                               (i > 0 ? REUSE_B_READY : 0) | eflags);
        }
        done_c[i] = event();
        cudaEventRecord(done_c[i], s);
        // D2H lags one panel so a pageable destination does not serialise the loop
        if (!c_dev && i >= 1) d2h(i - 1);
        if (c_st && i >= kStageIn) unstage(i - kStageIn);  // frees the slot d2h(i) will use
    }
    if (rc == QADIC_OK && !c_dev) {
        d2h(panels - 1);
        after(s, cs.d2h);  // stream-ordered completion: s sees every copy
        if (c_st)
            for (int64_t j = std::max<int64_t>(0, panels - kStageIn); j < panels; ++j) unstage(j);
    }
    st.reset();  // waits for the DMAs that read the input slots
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (rc) return rc;
    return check_launch("gf_matmul_host_u8");
}

}  // extern "C"
