/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the kkSpGEMM hot path.
 *
 * This is the parity oracle.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it, and only as
 * the checker.  The product path (libkkspgemm.so) never links or calls it.
 *
 * Every function restates the reference algorithm at the cited file:line of
 * /root/reference/proj (read-only upstream).  Pinned by:
 *   - the reference's own golden vectors (tests/golden/reference_kats.json),
 *   - bitwise comparison with the reference library compiled from its own
 *     sources into oracle/_ref/ (tests/test_oracle.py).
 * Build flags: -O2 -ffp-contract=off, no -march (SURVEY.md §8a FMA caveat).
 */
#ifndef KK_SPGEMM_ORACLE_H
#define KK_SPGEMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* flops_stats, src/csr_matrix.cpp:136-154.  per_row may be NULL. */
int orc_flops_stats(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols,
                    const int64_t* b_rowptr, int64_t* per_row, int64_t* total,
                    int64_t* max_row);

/* compressed_row_sizes, src/compression.cpp:25-48: distinct col/32 per row. */
int orc_compressed_row_sizes(int32_t n, int32_t k, const int64_t* b_rowptr,
                             const int32_t* b_cols, int32_t* sizes);

/* decide_compression, src/compression.cpp:99-148.  mode 0=Auto 1=Always
 * 2=Never.  Fills compressed flops/max and the applied bit (ppm gate). */
int orc_decide_compression(int32_t m, int32_t n, int32_t k, const int64_t* a_rowptr,
                           const int32_t* a_cols, const int64_t* b_rowptr,
                           const int32_t* b_cols, int64_t total_flops, double gate,
                           int mode, int64_t* cflops, int64_t* cmax, int* applied);

/* symbolic row sizes, src/engine.cpp:397-446 (SymbolicSink :210-221): the
 * number of distinct columns of C(i,:).  Independent of compression. */
int orc_symbolic_row_sizes(int32_t m, int32_t k, const int64_t* a_rowptr,
                           const int32_t* a_cols, const int64_t* b_rowptr,
                           const int32_t* b_cols, int64_t* row_sizes);

/* numeric, src/engine.cpp:448-491 with process_row :251-290 and the
 * accumulators' first-touch for_each order (accumulators.hpp:110-114,
 * 217-221, 322-326).  c_rowptr is the symbolic result; cols are written in
 * first-touch order and each value is the left-to-right sum starting from
 * the first product (a*b unfused, then +).  Returns 0, or 3 when a row does
 * not match the structure (engine.cpp:238-245). */
int orc_numeric(int32_t m, int32_t k, const int64_t* a_rowptr, const int32_t* a_cols,
                const double* a_vals, const int64_t* b_rowptr, const int32_t* b_cols,
                const double* b_vals, const int64_t* c_rowptr, int32_t* c_cols,
                double* c_vals);

/* sort_rows / canonicalize, src/csr_matrix.cpp:110-127, src/oracle.cpp:105-120.
 * In place, stable by column (columns are unique within a row). */
int orc_sort_rows(int32_t m, const int64_t* rowptr, int32_t* cols, double* vals);

/* compare_canonical relative error, src/oracle.cpp:122-159, over equal
 * structures.  Returns max |e-v|/max(|e|,|v|) (0 when both are 0). */
double orc_max_rel_error(int64_t nnz, const double* expected, const double* actual);

/* resolve_config, src/engine.cpp:367-395.  accumulator/scheme codes follow
 * engine.hpp:14-16 (Scheme 0 Seq 1 Flat; Accumulator 0 Auto 1 LL 2 LP 3 Dense). */
typedef struct orc_resolved {
    int32_t accumulator, scheme, l1_capacity, effective_k, l2_capacity;
} orc_resolved;
int orc_resolve_config(int phase, int32_t k, double avg_row_flops, int applied,
                       int cfg_accumulator, int cfg_scheme, int32_t cfg_l1_capacity,
                       int32_t dense_cutoff_k, double avg_flops_cutoff,
                       int64_t row_upper_bound, orc_resolved* out);

/* Per-row canonical digests: an order-independent 64-bit hash of each row's
 * (column, value bits) set and its length, the digest of the row sorted as
 * canonicalize does (src/oracle.cpp:105-120).  orc_row_digests digests a
 * given CSR; orc_product_row_digests forms each row of C = A*B with the
 * numeric restatement (left-to-right sums from the first product) in
 * nthreads threads and digests it without storing C (sizes[i] = row size,
 * may be NULL).  libkkspgemm.so's spg_row_digests is the device twin. */
int orc_row_digests(int32_t m, const int64_t* rowptr, const int32_t* cols, const double* vals, uint64_t* out);
int orc_product_row_digests(int32_t m, int32_t k, const int64_t* a_rowptr, const int32_t* a_cols,
                            const double* a_vals, const int64_t* b_rowptr, const int32_t* b_cols,
                            const double* b_vals, int nthreads, uint64_t* out, int64_t* sizes);

#ifdef __cplusplus
}
#endif
#endif
