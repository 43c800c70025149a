/*
 * kkspgemm — B200-native two-phase SpGEMM (kkSpGEMM, arXiv 1801.03065).
 *
 * C ABI of libkkspgemm.so: plain pointers and sizes, no C++ or torch types.
 * It replaces the reference's handle API in
 *   /root/reference/proj/include/spgemm/engine.hpp:79-103
 * (symbolic / numeric / multiply / resolve_config / flat_position), with the
 * structures of engine.hpp:12-72, csr_matrix.hpp:19-56 and compression.hpp:45-58
 * flattened into the structs below.  All compute runs in hand-written sm_100a
 * kernels; there is no CPU fallback — every entry point that needs the GPU
 * fails with SPG_ERR_CUDA when no device is present.
 *
 * Conventions (reference common.hpp:12-14): index_t = int32 (rows, columns),
 * offset_t = flops_t = int64 (row offsets, nnz, flop counts).  Matrices are
 * CSR with int64 row_offsets[num_rows+1], int32 col_indices, fp64 values, all
 * in device memory.  row_offsets[0] need not be 0: a row-block view of a
 * larger matrix (row_offsets + lo, same col/val arrays) is accepted as is,
 * which is how multi-GPU shards are passed.
 *
 * Calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy default
 * stream).  spg_symbolic synchronises the stream (small host reads for the
 * reference's host-side decisions: flop/compression totals, nnz(C));
 * spg_numeric is asynchronous unless `stats` is non-NULL, except for the one
 * pass per handle that records the structure-reuse slot replay.  One handle
 * must not run concurrent spg_numeric calls.
 */
#ifndef KKSPGEMM_H
#define KKSPGEMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: the reference's exception taxonomy (common.hpp:16-52) --- */
enum {
    SPG_OK = 0,
    SPG_ERR_CONTRACT = 1,    /* ContractError: dimension mismatch, bad argument  */
    SPG_ERR_REUSE = 2,       /* ReuseError: operands do not match the handle     */
    SPG_ERR_POOL_SIZING = 4, /* PoolSizingError: one L2 chunk exceeds the budget */
    SPG_ERR_INTERNAL = 5,    /* std::logic_error: structure/bound violation      */
    SPG_ERR_CUDA = 6,        /* CUDA runtime failure or no device                */
    SPG_ERR_NOMEM = 7        /* device allocation failed                          */
};

/* engine.hpp:14-16 */
enum { SPG_SCHEME_SEQUENTIAL = 0, SPG_SCHEME_FLAT_PARALLEL = 1 };
enum { SPG_ACC_AUTO = 0, SPG_ACC_LL = 1, SPG_ACC_LP = 2, SPG_ACC_DENSE = 3 };
/* compression.hpp:60 */
enum { SPG_COMPRESSION_AUTO = 0, SPG_COMPRESSION_ALWAYS = 1, SPG_COMPRESSION_NEVER = 2 };
/* memory_pool.hpp:16-19 */
enum { SPG_POOL_ONE2ONE = 0, SPG_POOL_MANY2MANY = 1 };
/* engine.hpp:33 */
enum { SPG_PHASE_SYMBOLIC = 0, SPG_PHASE_NUMERIC = 1 };

/* CsrMatrix (csr_matrix.hpp:19-36), device-resident view. */
typedef struct spg_csr {
    int32_t num_rows;
    int32_t num_cols;
    int64_t nnz;                /* row_offsets[num_rows] - row_offsets[0]; the
                                   numeric reuse fingerprint (engine.cpp:451-453) */
    const int64_t* row_offsets; /* [num_rows+1], device */
    const int32_t* col_indices; /* device */
    const double* values;       /* device; may be NULL for spg_symbolic */
} spg_csr;

/* SpgemmConfig (engine.hpp:18-31).  worker_count and row_block are accepted
 * for source compatibility; on the GPU the row grain is the warp. */
typedef struct spg_config {
    int32_t scheme;
    int32_t accumulator;
    int32_t l1_capacity;
    int32_t dense_cutoff_k;
    double avg_flops_cutoff;
    double lp_max_occupancy;
    double compression_gate;
    int32_t compression;
    int32_t collapse_divisor;
    int32_t worker_count;
    int32_t sort_output;
    int32_t row_block;
    int32_t pool_mode;
    int64_t pool_budget_bytes;
} spg_config;

/* ResolvedConfig (engine.hpp:36-42) */
typedef struct spg_resolved {
    int32_t accumulator;
    int32_t scheme;
    int32_t l1_capacity;
    int32_t effective_k;
    int32_t l2_capacity;
} spg_resolved;

/* PhaseStats (engine.hpp:44-48) */
typedef struct spg_phase_stats {
    double ms;
    int64_t pool_allocations;
    int64_t l2_inserts;
} spg_phase_stats;

/* FlopsStats scalars (csr_matrix.hpp:50-56); per_row_flops stays on device. */
typedef struct spg_flops_stats {
    int64_t total_flops;
    int64_t max_row_flops;
    double avg_degree_a;
    double avg_row_flops;
} spg_flops_stats;

/* CompressionReport (compression.hpp:45-51) */
typedef struct spg_compression_report {
    double cf;
    double cmrf;
    int64_t compressed_flops;
    int64_t compressed_max_row_flops;
    int32_t applied;
} spg_compression_report;

/* Every host field of SpgemmHandle (engine.hpp:53-72) plus the device
 * pointers the handle owns. */
typedef struct spg_handle_info {
    int32_t m, n, k;
    int64_t nnz_a, nnz_b, nnz_c;
    spg_flops_stats flops;
    spg_compression_report compression;
    int64_t max_row_size;
    double avg_row_size;
    double avg_row_size_estimate;
    spg_resolved symbolic_choice;
    spg_resolved numeric_choice;
    spg_config config;
    spg_phase_stats symbolic_stats;
    double compress_ms;
    const int64_t* d_c_row_offsets; /* [m+1], device, owned by the handle */
    const int64_t* d_per_row_flops; /* [m], device, owned by the handle   */
    int64_t compressed_nnz_b;       /* (word index, bits) pairs of the compressed B
                                       rows A references (compress_rows output size) */
    int32_t heavy_path;             /* rows beyond the warp tables: 0 none, 1 hashed
                                       buckets, 2 column slabs (diagnostic) */
    int32_t b_sorted;               /* symbolic saw every referenced B row sorted */
} spg_handle_info;

typedef struct spg_handle* spg_handle_t;

/* Host-side description used to rebuild a device handle from the fields of a
 * reference SpgemmHandle (the engine.hpp shim path).  c_row_offsets is HOST
 * memory [m+1].  A handle whose config.accumulator is Auto and whose
 * numeric_choice is what resolve_config yields keeps the GPU's own numeric
 * plan (fast kernels, slot replay); an edited choice is honoured as forced. */
typedef struct spg_handle_desc {
    int32_t m, n, k;
    int64_t nnz_a, nnz_b;
    const int64_t* c_row_offsets;
    spg_flops_stats flops;
    spg_compression_report compression;
    int64_t max_row_size;
    double avg_row_size;
    double avg_row_size_estimate;
    spg_resolved symbolic_choice;
    spg_resolved numeric_choice;
    spg_config config;
    spg_phase_stats symbolic_stats;
    double compress_ms;
    const int64_t* per_row_flops;   /* HOST [m] (FlopsStats::per_row_flops) or NULL:
                                       enables the heavy-row order and the slot replay */
} spg_handle_desc;

/* Last error message of the calling thread ("" after success). */
const char* spg_last_error(void);

/* Defaults of SpgemmConfig (engine.hpp:18-31). */
int spg_config_init(spg_config* cfg);

/* resolve_config (engine.hpp:86-88, engine.cpp:367-395); pure host. */
int spg_resolve_config(int32_t phase, int32_t k, const spg_flops_stats* stats,
                       const spg_compression_report* report, const spg_config* cfg,
                       int64_t row_upper_bound, spg_resolved* out);

/* flat_position (engine.hpp:103, engine.cpp:360-365); pure host.
 * prefix[0..len) non-decreasing, prefix[0] = 0. */
int spg_flat_position(const int64_t* prefix, int64_t len, int64_t t, int32_t* seg,
                      int64_t* off);

/* symbolic (engine.hpp:92, engine.cpp:397-446): flop statistics, graph
 * compression with the ppm gate, the compressed (or raw) structure union, and
 * the device exclusive scan into C's row offsets.  Synchronises `stream`. */
int spg_symbolic(const spg_csr* a, const spg_csr* b, const spg_config* cfg, spg_handle_t* out,
                 void* stream);

/* numeric (engine.hpp:97-98, engine.cpp:448-491): fills C = A*B into the
 * structure of `h`.  c_cols/c_vals are device buffers of nnz_c entries,
 * row-major in the order of the handle's row offsets.  Column order within a
 * row is the reference's first-touch order unless config.sort_output.
 * Throws (returns) SPG_ERR_REUSE when dimensions or nnz fingerprints differ
 * from the handle.  Asynchronous unless stats != NULL. */
int spg_numeric(spg_handle_t h, const spg_csr* a, const spg_csr* b, int32_t* c_cols,
                double* c_vals, spg_phase_stats* stats, void* stream);

/* numeric restricted to C rows [row_begin, row_end) (extension, no reference
 * counterpart): same buffers and contract as spg_numeric, entries of other
 * rows untouched.  Lets a host caller copy finished row blocks of C out while
 * later blocks compute (paper_1801_03065_b200/host.py).  Only full-range
 * passes count toward recording the slot replay. */
int spg_numeric_rows(spg_handle_t h, const spg_csr* a, const spg_csr* b, int32_t row_begin,
                     int32_t row_end, int32_t* c_cols, double* c_vals, spg_phase_stats* stats,
                     void* stream);

/* Query / mutate / rebuild handles. */
int spg_handle_info_get(spg_handle_t h, spg_handle_info* out);
int spg_handle_copy_row_offsets(spg_handle_t h, int64_t* host_dst);
int spg_handle_copy_per_row_flops(spg_handle_t h, int64_t* host_dst);
/* Stream-ordered device-to-device copy of C's row offsets ([m+1] int64). */
int spg_handle_copy_row_offsets_device(spg_handle_t h, int64_t* device_dst, void* stream);
/* Replace the handle's config and numeric choice (acceptance_main.cpp:417-425
 * edits handle.config; SURVEY Appendix A forces handle.numeric_choice). */
int spg_handle_set_numeric(spg_handle_t h, const spg_config* cfg, const spg_resolved* numeric_choice);
int spg_handle_import(const spg_handle_desc* desc, spg_handle_t* out, void* stream);
/* Device error word raised by an asynchronous spg_numeric (0 = none);
 * synchronises the handle's stream. */
int spg_handle_check(spg_handle_t h);
void spg_handle_destroy(spg_handle_t h);

/* Per-row column sort of a device CSR in place (csr_matrix.cpp:110-127,
 * the sort_output pass engine.cpp:466-485). */
int spg_sort_rows(int32_t m, const int64_t* d_row_offsets, int32_t* d_cols, double* d_vals,
                  void* stream);

/* Transpose of a device CSR (csr_matrix.cpp:82-108: entries of each result
 * row in increasing original-row order) into caller buffers: d_t_row_offsets
 * [a->num_cols + 1], d_t_cols/d_t_vals [a->nnz].  Used for R = P^T of the
 * multigrid triple product.  Synchronises once (the longest result row). */
int spg_transpose(const spg_csr* a, int64_t* d_t_row_offsets, int32_t* d_t_cols, double* d_t_vals,
                  void* stream);

/* Per-row canonical digests of a device CSR (extension; the device side of
 * the reference's canonicalize + compare_canonical, oracle.cpp:105-159):
 * d_out[i] = sum over the row's entries of mix(column, value bits) plus
 * mix(row length), mix the splitmix64 finalizer — independent of the column
 * order, so it is the digest of the sorted row.  The oracle computes the same
 * function on the CPU; equal digests mean equal sorted columns and bitwise
 * equal values.  Stream-ordered. */
int spg_row_digests(int32_t m, const int64_t* d_row_offsets, const int32_t* d_cols, const double* d_vals,
                    uint64_t* d_out, void* stream);

/* Per-row multiplication counts (flops_stats per_row_flops, csr_matrix.cpp:136-154)
 * into device memory d_out[a->num_rows]; stream-ordered.  Used for the
 * flop-balanced row partition of the multi-GPU path. */
int spg_row_flops(const spg_csr* a, const spg_csr* b, int64_t* d_out, void* stream);

/* Structure-reuse replay state of a handle (extension, no reference
 * counterpart): 0 = the handle runs the hashing kernels only, 1 = eligible
 * (the slot map is recorded on the second numeric pass), 2 = recorded (later
 * passes replay it while A's and B's structure fingerprints match). */
int spg_handle_replay_state(spg_handle_t h);

/* Number of kernels this library launched since load (evidence counter). */
int64_t spg_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
