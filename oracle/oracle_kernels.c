/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's native
 * kernels (/root/reference/pkg/src/qadic/_kernels/_speed.pyx), used by
 * oracle/qadic_oracle.py as a faster checker and as the CPU baseline.
 * Never linked into the product library.
 *
 *   oracle_matmul_exact_u64   _speed.pyx:15-30, 58-66  (uint64, wraps mod 2^64)
 *   oracle_redq_compress_u64  _speed.pyx:121-140       (u_i=(r>>it)-p*(s>>it))
 *   oracle_matmul_fold_u64    the fold-every-chunk composition of
 *                             polymul.py:198-208 (acc += chunk product;
 *                             redq.reduce_words_array between chunks,
 *                             redq.py:318-332) applied to a matrix product
 *
 * Rows are split across OpenMP threads; per-row arithmetic follows the
 * reference loops exactly, so results are bit-identical.
 */
#include <stdint.h>
#include <string.h>
#include <omp.h>

int oracle_num_threads(void) { return omp_get_max_threads(); }

void oracle_matmul_exact_u64(const uint64_t *a, const uint64_t *b, uint64_t *c,
                             int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t *ci = c + i * n;
        memset(ci, 0, (size_t)n * sizeof(uint64_t));
        for (int64_t kk = 0; kk < k; ++kk) {
            uint64_t av = a[i * k + kk];
            const uint64_t *bk = b + kk * n;
            for (int64_t j = 0; j < n; ++j) ci[j] += av * bk[j];
        }
    }
}

void oracle_redq_compress_u64(const uint64_t *r, int64_t n, int64_t p, int t, int d,
                              uint64_t *out) {
    const uint64_t pp = (uint64_t)p;
#pragma omp parallel for schedule(static)
    for (int64_t idx = 0; idx < n; ++idx) {
        uint64_t ri = r[idx], s = ri / pp;
        for (int i = 0; i <= d; ++i)
            out[idx * (d + 1) + i] = (ri >> (i * t)) - pp * (s >> (i * t));
    }
}

/* digit-reduce one word: compress (one division) + correct + repack */
static inline uint64_t fold_word(uint64_t r, uint64_t p, int t, int d, uint64_t c) {
    uint64_t s = r / p, u[64], out = 0;
    for (int i = 0; i <= d; ++i) u[i] = (r >> (i * t)) - p * (s >> (i * t));
    for (int i = 0; i <= d; ++i) {
        uint64_t mu = (i < d) ? (u[i] + c * u[i + 1]) % p : u[i];
        out += mu << (i * t);
    }
    return out;
}

void oracle_matmul_fold_u64(const uint64_t *a, const uint64_t *b, uint64_t *acc,
                            int64_t m, int64_t k, int64_t n, int64_t p, int t, int d,
                            int64_t chunk) {
    const uint64_t pp = (uint64_t)p;
    const uint64_t q = (uint64_t)1 << t;
    const uint64_t c = (q % pp == 0) ? 0 : (pp - q % pp) % pp;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t *ci = acc + i * n;
        memset(ci, 0, (size_t)n * sizeof(uint64_t));
        for (int64_t k0 = 0; k0 < k; k0 += chunk) {
            int64_t k1 = k0 + chunk < k ? k0 + chunk : k;
            for (int64_t kk = k0; kk < k1; ++kk) {
                uint64_t av = a[i * k + kk];
                const uint64_t *bk = b + kk * n;
                for (int64_t j = 0; j < n; ++j) ci[j] += av * bk[j];
            }
            if (k1 < k)
                for (int64_t j = 0; j < n; ++j) ci[j] = fold_word(ci[j], pp, t, d, c);
        }
    }
}
