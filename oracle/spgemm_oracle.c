/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the kkSpGEMM hot path.
 * See spgemm_oracle.h for the contract and the pinning evidence.  Never
 * linked into the product library.
 */
#include "spgemm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

int orc_flops_stats(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols,
                    const int64_t* b_rowptr, int64_t* per_row, int64_t* total,
                    int64_t* max_row)
{
    /* csr_matrix.cpp:143-150 */
    int64_t t = 0, mx = 0;
    for (int32_t i = 0; i < m; ++i) {
        int64_t f = 0;
        for (int64_t p = a_rowptr[i]; p < a_rowptr[i + 1]; ++p) {
            const int32_t j = a_cols[p];
            f += b_rowptr[j + 1] - b_rowptr[j];
        }
        if (per_row)
            per_row[i] = f;
        t += f;
        if (f > mx)
            mx = f;
    }
    *total = t;
    *max_row = mx;
    return 0;
}

int orc_compressed_row_sizes(int32_t n, int32_t k, const int64_t* b_rowptr,
                             const int32_t* b_cols, int32_t* sizes)
{
    /* compression.cpp:34-45: LL keyed on col/32; used() = distinct words */
    const int32_t words = (k + 31) / 32;
    int32_t* stamp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(words > 0 ? words : 1));
    if (!stamp)
        return 1;
    for (int32_t w = 0; w < words; ++w)
        stamp[w] = -1;
    for (int32_t j = 0; j < n; ++j) {
        int32_t cnt = 0;
        for (int64_t q = b_rowptr[j]; q < b_rowptr[j + 1]; ++q) {
            const int32_t w = b_cols[q] / 32;
            if (stamp[w] != j) {
                stamp[w] = j;
                ++cnt;
            }
        }
        sizes[j] = cnt;
    }
    free(stamp);
    return 0;
}

int orc_decide_compression(int32_t m, int32_t n, int32_t k, const int64_t* a_rowptr,
                           const int32_t* a_cols, const int64_t* b_rowptr,
                           const int32_t* b_cols, int64_t total_flops, double gate,
                           int mode, int64_t* cflops, int64_t* cmax, int* applied)
{
    int32_t* sizes = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!sizes)
        return 1;
    orc_compressed_row_sizes(n, k, b_rowptr, b_cols, sizes);
    /* compression.cpp:111-117 */
    int64_t tot = 0, mx = 0;
    for (int32_t i = 0; i < m; ++i) {
        int64_t f = 0;
        for (int64_t p = a_rowptr[i]; p < a_rowptr[i + 1]; ++p)
            f += sizes[a_cols[p]];
        tot += f;
        if (f > mx)
            mx = f;
    }
    free(sizes);
    *cflops = tot;
    *cmax = mx;
    /* compression.cpp:131-147: strict ppm gate */
    int apply = 0;
    if (mode == 1)
        apply = 1;
    else if (mode == 2)
        apply = 0;
    else {
        double g = gate < 0.0 ? 0.0 : (gate > 1.0 ? 1.0 : gate);
        const int64_t threshold_ppm = llround((1.0 - g) * 1000000.0);
        apply = total_flops > 0 && tot * 1000000 < total_flops * threshold_ppm;
    }
    *applied = apply;
    return 0;
}

int orc_symbolic_row_sizes(int32_t m, int32_t k, const int64_t* a_rowptr,
                           const int32_t* a_cols, const int64_t* b_rowptr,
                           const int32_t* b_cols, int64_t* row_sizes)
{
    int32_t* stamp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
    if (!stamp)
        return 1;
    for (int32_t c = 0; c < k; ++c)
        stamp[c] = -1;
    for (int32_t i = 0; i < m; ++i) {
        int64_t cnt = 0;
        for (int64_t p = a_rowptr[i]; p < a_rowptr[i + 1]; ++p) {
            const int32_t j = a_cols[p];
            for (int64_t q = b_rowptr[j]; q < b_rowptr[j + 1]; ++q) {
                const int32_t c = b_cols[q];
                if (stamp[c] != i) {
                    stamp[c] = i;
                    ++cnt;
                }
            }
        }
        row_sizes[i] = cnt;
    }
    free(stamp);
    return 0;
}

int orc_numeric(int32_t m, int32_t k, const int64_t* a_rowptr, const int32_t* a_cols,
                const double* a_vals, const int64_t* b_rowptr, const int32_t* b_cols,
                const double* b_vals, const int64_t* c_rowptr, int32_t* c_cols,
                double* c_vals)
{
    /* Dense accumulator with the output span as touched list
     * (accumulators.hpp:299-320); visiting order = process_row :259-267. */
    int64_t* where = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
    if (!where)
        return 1;
    for (int32_t c = 0; c < k; ++c)
        where[c] = -1;
    int rc = 0;
    for (int32_t i = 0; i < m; ++i) {
        const int64_t lo = c_rowptr[i], hi = c_rowptr[i + 1];
        int64_t used = lo;
        for (int64_t p = a_rowptr[i]; p < a_rowptr[i + 1]; ++p) {
            const int32_t j = a_cols[p];
            const double av = a_vals[p];
            for (int64_t q = b_rowptr[j]; q < b_rowptr[j + 1]; ++q) {
                const int32_t c = b_cols[q];
                const double prod = av * b_vals[q];
                if (where[c] < lo) { /* first touch in this row */
                    if (used >= hi) {
                        rc = 3;
                        goto done;
                    }
                    where[c] = used;
                    c_cols[used] = c;
                    c_vals[used] = prod;
                    ++used;
                } else {
                    c_vals[where[c]] += prod;
                }
            }
        }
        if (used != hi) {
            rc = 3;
            goto done;
        }
    }
done:
    free(where);
    return rc;
}

typedef struct {
    int32_t c;
    double v;
} orc_pair;

static int orc_pair_cmp(const void* x, const void* y)
{
    const int32_t a = ((const orc_pair*)x)->c, b = ((const orc_pair*)y)->c;
    return (a > b) - (a < b);
}

int orc_sort_rows(int32_t m, const int64_t* rowptr, int32_t* cols, double* vals)
{
    int64_t cap = 0;
    for (int32_t i = 0; i < m; ++i)
        if (rowptr[i + 1] - rowptr[i] > cap)
            cap = rowptr[i + 1] - rowptr[i];
    orc_pair* tmp = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(cap > 0 ? cap : 1));
    if (!tmp)
        return 1;
    for (int32_t i = 0; i < m; ++i) {
        const int64_t lo = rowptr[i], len = rowptr[i + 1] - rowptr[i];
        for (int64_t q = 0; q < len; ++q) {
            tmp[q].c = cols[lo + q];
            tmp[q].v = vals ? vals[lo + q] : 0.0;
        }
        qsort(tmp, (size_t)len, sizeof(orc_pair), orc_pair_cmp);
        for (int64_t q = 0; q < len; ++q) {
            cols[lo + q] = tmp[q].c;
            if (vals)
                vals[lo + q] = tmp[q].v;
        }
    }
    free(tmp);
    return 0;
}

double orc_max_rel_error(int64_t nnz, const double* expected, const double* actual)
{
    /* oracle.cpp:146-150 */
    double mx = 0.0;
    for (int64_t q = 0; q < nnz; ++q) {
        const double e = expected[q], v = actual[q];
        const double denom = fmax(fabs(e), fabs(v));
        const double err = denom == 0.0 ? 0.0 : fabs(e - v) / denom;
        if (err > mx || err != err)
            mx = err;
    }
    return mx;
}

int orc_resolve_config(int phase, int32_t k, double avg_row_flops, int applied,
                       int cfg_accumulator, int cfg_scheme, int32_t cfg_l1_capacity,
                       int32_t dense_cutoff_k, double avg_flops_cutoff,
                       int64_t row_upper_bound, orc_resolved* out)
{
    /* engine.cpp:367-395; phase 0 Symbolic, 1 Numeric */
    const int compressed = phase == 0 && applied;
    out->effective_k = compressed ? (int32_t)(((int64_t)k + 31) / 32) : k;
    if (cfg_accumulator != 0) {
        out->accumulator = cfg_accumulator;
        out->scheme = cfg_scheme;
    } else if (out->effective_k < dense_cutoff_k) {
        out->accumulator = 3;
        out->scheme = cfg_scheme;
    } else if (avg_row_flops < avg_flops_cutoff) {
        out->accumulator = 1;
        out->scheme = cfg_scheme;
    } else {
        out->accumulator = 2;
        out->scheme = 1;
    }
    int64_t bound = row_upper_bound < out->effective_k ? row_upper_bound : out->effective_k;
    if (bound < 1)
        bound = 1;
    out->l2_capacity = (int32_t)bound;
    out->l1_capacity = cfg_l1_capacity > 0 ? cfg_l1_capacity : out->l2_capacity;
    return 0;
}

/* ---- per-row canonical digests (test infrastructure) ---------------------
 * The canonical form of a row (src/oracle.cpp:105-120 sorts each row by
 * column) summarised as an ORDER-INDEPENDENT 64-bit digest: the sum of a
 * mixed hash of every (column, value bits) pair plus a hash of the row
 * length, so any column order gives the digest of the sorted row.  Equal
 * digests <=> equal sorted columns and bitwise-equal values (up to 2^-64).
 * libkkspgemm.so computes the same function on the device (spg_row_digests).
 * The product C is formed row by row with the numeric restatement above (dense
 * accumulator, left-to-right sums) and never stored, in nthreads threads. */
#include <pthread.h>

static uint64_t orc_mix64(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

static uint64_t orc_entry_hash(int32_t col, double v)
{
    uint64_t bits;
    memcpy(&bits, &v, sizeof(bits));
    return orc_mix64(((uint64_t)(uint32_t)col * 0x9E3779B97F4A7C15ull) ^ orc_mix64(bits));
}

int orc_row_digests(int32_t m, const int64_t* rowptr, const int32_t* cols, const double* vals, uint64_t* out)
{
    for (int32_t i = 0; i < m; ++i) {
        uint64_t d = orc_mix64((uint64_t)(rowptr[i + 1] - rowptr[i]) + 0x2545F4914F6CDD1Dull);
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q)
            d += orc_entry_hash(cols[q], vals[q]);
        out[i] = d;
    }
    return 0;
}

typedef struct {
    int32_t m, k;
    const int64_t *a_rowptr, *b_rowptr;
    const int32_t *a_cols, *b_cols;
    const double *a_vals, *b_vals;
    uint64_t* out;
    int64_t* sizes;
    int32_t next;
    pthread_mutex_t mu;
} digest_job;

static void* digest_worker(void* arg)
{
    digest_job* J = (digest_job*)arg;
    double* acc = (double*)malloc(sizeof(double) * (size_t)(J->k > 0 ? J->k : 1));
    int32_t* seen = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J->k > 0 ? J->k : 1));
    int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J->k > 0 ? J->k : 1));
    if (!acc || !seen || !touched) {
        free(acc);
        free(seen);
        free(touched);
        return (void*)1;
    }
    for (int32_t c = 0; c < J->k; ++c)
        seen[c] = -1;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int32_t i0 = J->next;
        J->next = i0 + 256 < J->m ? i0 + 256 : J->m;
        pthread_mutex_unlock(&J->mu);
        if (i0 >= J->m)
            break;
        const int32_t i1 = i0 + 256 < J->m ? i0 + 256 : J->m;
        for (int32_t i = i0; i < i1; ++i) {
            int64_t used = 0;
            for (int64_t p = J->a_rowptr[i]; p < J->a_rowptr[i + 1]; ++p) {
                const int32_t j = J->a_cols[p];
                const double av = J->a_vals[p];
                for (int64_t q = J->b_rowptr[j]; q < J->b_rowptr[j + 1]; ++q) {
                    const int32_t c = J->b_cols[q];
                    const double prod = av * J->b_vals[q];
                    if (seen[c] != i) { /* first touch: the sum starts at the first product */
                        seen[c] = i;
                        acc[c] = prod;
                        touched[used++] = c;
                    } else {
                        acc[c] += prod;
                    }
                }
            }
            uint64_t d = orc_mix64((uint64_t)used + 0x2545F4914F6CDD1Dull);
            for (int64_t t = 0; t < used; ++t)
                d += orc_entry_hash(touched[t], acc[touched[t]]);
            J->out[i] = d;
            if (J->sizes)
                J->sizes[i] = used;
        }
    }
    free(acc);
    free(seen);
    free(touched);
    return NULL;
}

int orc_product_row_digests(int32_t m, int32_t k, const int64_t* a_rowptr, const int32_t* a_cols,
                            const double* a_vals, const int64_t* b_rowptr, const int32_t* b_cols,
                            const double* b_vals, int nthreads, uint64_t* out, int64_t* sizes)
{
    digest_job J = {m, k, a_rowptr, b_rowptr, a_cols, b_cols, a_vals, b_vals, out, sizes, 0};
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1)
        nthreads = 1;
    if (nthreads > 256)
        nthreads = 256;
    pthread_t th[256];
    int rc = 0;
    for (int t = 0; t < nthreads; ++t)
        pthread_create(&th[t], NULL, digest_worker, &J);
    for (int t = 0; t < nthreads; ++t) {
        void* r = NULL;
        pthread_join(th[t], &r);
        if (r)
            rc = 1;
    }
    pthread_mutex_destroy(&J.mu);
    return rc;
}
