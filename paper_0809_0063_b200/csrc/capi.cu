// ABI bookkeeping for libqadic_b200.so: version, error strings, launch count,
// and the exact host constants of the FP64 reciprocal division.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "qadic_common.cuh"
#include "qadic_internal.h"

namespace qadic {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    int n = snprintf(g_err, sizeof g_err, "[qadic status %d] ", code);
    vsnprintf(g_err + n, sizeof g_err - n, fmt, ap);
    va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char* what) {
    count_launch(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(QADIC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
        return QADIC_ERR_CUDA;
    }
    return QADIC_OK;
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

int qadic_abi_version(void) { return QADIC_ABI_VERSION; }
const char* qadic_last_error(void) { return qadic::g_err; }
int64_t qadic_launch_count(void) { return qadic::g_launches.load(); }

}  // extern "C"
