// ABI bookkeeping for libqadic_b200.so: version, error strings, launch count,
// and the exact host constants of the FP64 reciprocal division.
#include <math.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>

#include <atomic>

#include "qadic_common.cuh"
#include "qadic_internal.h"

#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace qadic {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

// ---- optional per-kernel timing with CUDA events on the launching stream ----
struct ProfRec {
    const char* name;
    cudaEvent_t start, stop;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof_open;   // recorded, not yet collected
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t pool_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

int prof_begin(cudaStream_t s, const char* name) {
    if (!g_prof_on) return -1;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r{name, pool_event(), pool_event()};
    cudaEventRecord(r.start, s);
    g_prof_open.push_back(r);
    return (int)g_prof_open.size() - 1;
}

void prof_end(int idx, cudaStream_t s) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_prof_open[idx].stop, s);
}

void set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    int n = snprintf(g_err, sizeof g_err, "[qadic status %d] ", code);
    vsnprintf(g_err + n, sizeof g_err - n, fmt, ap);
    va_end(ap);
}

bool pdl_enabled() {
    static const bool on = !(getenv("QADIC_NO_PDL") && atoi(getenv("QADIC_NO_PDL")) != 0);
    return on;
}

int pdl_prefetch_enabled() {
    // QADIC_PDL_PREFETCH=0 switches the pre-wait L2 prefetch of the batched kernels off (A/B)
    static const int on = pdl_enabled() && !(getenv("QADIC_PDL_PREFETCH") && atoi(getenv("QADIC_PDL_PREFETCH")) == 0);
    return on;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char* what, int launched) {
    count_launch(launched);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(QADIC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
        return QADIC_ERR_CUDA;
    }
    return QADIC_OK;
}

void keep_mempool() {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<bool> kept[64];
    if (kept[dev & 63].exchange(true)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
}

int num_sms_cached() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

double host_reciprocal_up(int64_t p) {
    double base = 1.0 / (double)p;
    // residual base*p - 1 is exact under FMA (base has 53 bits, p < 2^26)
    if (fma(base, (double)p, -1.0) < 0.0) base = nextafter(base, INFINITY);
    return base;
}

double host_case2_bound() {
    // ceil(2^106 / (3*2^53 + 2)) for beta = 53
    return 3002399751580331.0;
}

}  // namespace qadic

extern "C" {

void qadic_profile_enable(int on) { qadic::g_prof_on = on != 0; }

/* Synchronise every recorded event pair and write "name,count,total_ms\n"
 * lines (one per kernel name, insertion order) into buf; resets the log. */
int qadic_profile_collect(char* buf, size_t len) {
    using namespace qadic;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<std::string> order;
    std::map<std::string, std::pair<int, double>> acc;
    for (auto& r : g_prof_open) {
        cudaEventSynchronize(r.stop);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.start, r.stop);
        auto it = acc.find(r.name);
        if (it == acc.end()) {
            order.push_back(r.name);
            acc[r.name] = {1, ms};
        } else {
            it->second.first += 1;
            it->second.second += ms;
        }
        g_event_pool.push_back(r.start);
        g_event_pool.push_back(r.stop);
    }
    g_prof_open.clear();
    size_t used = 0;
    if (len) buf[0] = 0;
    for (auto& n : order) {
        int w = snprintf(buf + used, len > used ? len - used : 0, "%s,%d,%.6f\n", n.c_str(), acc[n].first,
                         acc[n].second);
        if (w < 0 || used + w >= len) return QADIC_ERR_VALUE;
        used += w;
    }
    return QADIC_OK;
}

int qadic_abi_version(void) { return QADIC_ABI_VERSION; }
const char* qadic_last_error(void) { return qadic::g_err; }
int64_t qadic_launch_count(void) { return qadic::g_launches.load(); }

}  // extern "C"
