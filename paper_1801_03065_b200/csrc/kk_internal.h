// Host-side declarations shared by the C ABI (kk_api.cu) and the kernel
// launchers (kk_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace kk {

struct DevCounters;

enum AccKind : int { kAccLL = 1, kAccLP = 2, kAccDense = 3 };
enum RowVariant : int { kVarNumeric = 0, kVarSymRaw = 1, kVarSymCompressed = 2 };

// Per-warp accumulator layout (bytes are relative to the warp's region).
struct TabLayout {
    int acc = kAccLP;
    int32_t T = 0;     // LP slots / LL buckets / dense domain
    int32_t S = 0;     // key capacity (first-touch positions)
    int shift = 0;     // 32 - log2(T) for hashed maps
    uint32_t off_map = 0, off_aux = 0, off_ids = 0, off_pay = 0;
    uint64_t bytes = 0;
    bool has_ids = true, has_pay = true;
};

TabLayout make_layout(int acc, int variant, int32_t S, int32_t domain, double occupancy,
                      bool external_rows);

struct Totals {
    unsigned long long total_f, max_f, total_cf, max_cf;
    unsigned long long nnz_bc; // compressed pairs written (the compress pass)
    unsigned long long unsorted; // > 0: some compressed B row is not strictly column-sorted
    unsigned long long max_alen; // longest A row (cursor arrays of the column-slab kernel)
    unsigned long long hist_f[64];
    unsigned long long hist_cf[64];
};

struct ScanTotals {
    unsigned long long max_size;
    unsigned long long hist[64];
};

struct PoolDesc {
    char* base = nullptr;
    uint64_t chunk_bytes = 0;
    int32_t num_chunks = 0;
    int32_t mode = 0; // 0 one2one, 1 many2many
    int* states = nullptr;
};

struct RowLaunch {
    // operands
    const int64_t* a_rowptr;
    const int32_t* a_cols;
    const double* a_vals;
    const int64_t* b_rowptr;
    const int32_t* b_cols;
    const double* b_vals;
    const int32_t* csize;
    const int2* cpair;   // compressed B: {word index, bits} in B's own slots, allocation
                         // base; index with cpair_of(L) (rebased by b_rowptr[0])
    // rows
    const int32_t* list; // nullptr: rows [0, nrows)
    int64_t nrows;
    int32_t row_lo, row_hi; // numeric: only rows in [row_lo, row_hi) when row_hi > 0
    const unsigned long long* d_nrows; // symbolic heavy kernel: row count on the device (else nrows)
    const unsigned long long* gate; // numeric fast kernel: exit when gate[0..1] == gate[2..3] (replayed)
    int32_t no_segments;            // symbolic fast kernel: always use 32-product windows (A/B switch)
    int32_t l1_keys;                // the reference's level-1 key capacity (statistics only)
    // outputs
    int64_t* sym_sizes;          // symbolic: sizes[i] (== rowptr + 1)
    const int64_t* c_rowptr;     // numeric
    int32_t* c_cols;
    double* c_vals;
    DevCounters* ctr;
    // shape
    TabLayout lay;
    int wpb;
    int grid;
    bool l2;
    PoolDesc pool;
};

// kernel launchers (kk_kernels.cu); each returns cudaGetLastError()
cudaError_t launch_compress(int32_t n, const int64_t* b_rowptr, const int32_t* b_cols,
                            int32_t* csize, int2* cp_alloc, unsigned long long* nnz_bc, unsigned long long* unsorted,
                            const int* band, cudaStream_t st);
cudaError_t launch_flops(int32_t m, double avg_len, const int64_t* a_rowptr,
                         const int32_t* a_cols, const int64_t* b_rowptr, const int32_t* csize,
                         int64_t* out_f, int64_t* out_cf, Totals* tot, cudaStream_t st);
struct BinParams {
    int8_t bucket_class[64];
    int64_t class_off[32];
};
cudaError_t launch_bin_scatter(int32_t m, const int64_t* bound, const int64_t* rowptr_c,
                               int64_t clamp, const BinParams& bp,
                               unsigned long long* class_fill, int32_t* list, cudaStream_t st);
cudaError_t launch_row_kernel(const RowLaunch& L, int acc, bool flat, int variant,
                              cudaStream_t st);
int row_kernel_max_blocks_per_sm(int acc, bool flat, int variant, bool l2, int wpb,
                                 size_t smem);
cudaError_t scan_sizes_inplace(int64_t* rowptr, int64_t m, ScanTotals* tot, cudaStream_t st);
cudaError_t launch_sort_rows(int32_t m, const int64_t* rowptr, int32_t* cols, double* vals,
                             int64_t max_row, cudaStream_t st);
cudaError_t launch_row_flops(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols,
                             const int64_t* b_rowptr, int64_t* out, cudaStream_t st);
cudaError_t launch_transpose_count(int32_t m, int32_t n, const int64_t* rowptr, const int32_t* cols,
                                   int64_t* t_rowptr, ScanTotals* tot, cudaStream_t st);
cudaError_t launch_transpose_fill(int32_t m, int32_t n, const int64_t* rowptr, const int32_t* cols,
                                  const double* vals, const int64_t* t_rowptr, int32_t* t_cols, double* t_vals,
                                  int64_t max_row, cudaStream_t st);
cudaError_t launch_col_range(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols, int* out2, cudaStream_t st);
cudaError_t launch_row_bucket_hist(int32_t m, const int64_t* rowptr, ScanTotals* tot,
                                   cudaStream_t st);
cudaError_t launch_row_digests(int32_t m, const int64_t* rowptr, const int32_t* cols, const double* vals,
                               unsigned long long* out, cudaStream_t st);
cudaError_t launch_collect_empty_rows(int32_t m, const int64_t* c_rowptr, int32_t* list, unsigned long long* count,
                                      cudaStream_t st);
cudaError_t launch_check_empty_rows(const int32_t* list, int64_t n, const int64_t* a_rowptr, const int32_t* a_cols,
                                    const int64_t* b_rowptr, int32_t row_lo, int32_t row_hi, DevCounters* ctr,
                                    cudaStream_t st);

// fast paths (kk_fast.cu)
cudaError_t launch_numeric_fast(const RowLaunch& L, cudaStream_t st);
int numeric_fast_blocks_per_sm(int wpb, size_t smem);
cudaError_t launch_numeric_flat_fast(const RowLaunch& L, cudaStream_t st);
int numeric_flat_fast_blocks_per_sm(int wpb, size_t smem);
// rows of at most kTinyKeys (numeric) / kTinySymKeys (symbolic) keys, a
// thread per row (kk_tiny.cu)
constexpr int kTinyKeys = 16;
constexpr int kTinySymKeys = 32;
cudaError_t launch_numeric_tiny(const RowLaunch& L, cudaStream_t st);
cudaError_t launch_symbolic_tiny(const RowLaunch& L, bool compressed, unsigned long long* retry_count,
                                 int32_t* retry_list, cudaStream_t st);
cudaError_t launch_symbolic_fast(const RowLaunch& L, bool compressed, bool pipe, unsigned long long* retry_count,
                                 int32_t* retry_list, cudaStream_t st);
int symbolic_fast_blocks_per_sm(bool compressed, bool pipe, int wpb, size_t smem);

// heavy rows (kk_heavy.cu)
cudaError_t launch_symbolic_heavy(const RowLaunch& L, bool compressed, int32_t words, int32_t dom_words, int grid,
                                  cudaStream_t st);
cudaError_t launch_numeric_heavy(const RowLaunch& L, void* stage, int64_t stage_cap,
                                 int32_t bucket_keys, int32_t nb, int64_t min_products, int64_t max_products,
                                 int queue, int grid, cudaStream_t st);
cudaError_t sort_rows_by_flops_desc(int32_t* list, int64_t n, const int64_t* prf, cudaStream_t st);
int numeric_heavy_blocks_per_sm(int32_t nb);

// heavy rows by column slabs (kk_slab.cu); needs column-sorted B rows
struct SlabPlan {
    int4* items = nullptr;          // {row, part, parts, split slot}
    int64_t n_items = 0;
    void* scratch = nullptr;        // per warp cursor state
    int64_t max_a_row = 0;
    int64_t warps = 0;              // resident warps (multiple of the CTA's)
    unsigned long long* split_out = nullptr;
    unsigned int* split_done = nullptr;
    int64_t n_split = 0;
};
cudaError_t build_slab_items(const int32_t* list, int64_t n, const int64_t* a_rowptr, const int64_t* c_rowptr,
                             int64_t k, int64_t* item_off, int4* items, unsigned long long* split_count,
                             cudaStream_t st);
cudaError_t launch_numeric_slab(const RowLaunch& L, const SlabPlan& P, int64_t k, const int64_t* prf,
                                cudaStream_t st);
int numeric_slab_warps();
int slab_warps_per_cta();
size_t slab_scratch_per_entry();

// structure-reuse replay (kk_replay.cu)
struct ReplayLaunch {
    const int64_t* a_rowptr;
    const int32_t* a_cols;
    const double* a_vals;
    const int64_t* b_rowptr;
    const int32_t* b_cols;
    const double* b_vals;
    const int64_t* c_rowptr;
    int32_t* c_cols;
    double* c_vals;
    int32_t* ccache;          // C columns in first-touch order
    void* map;                // uint8_t / uint16_t slot per product
    const int64_t* prod_off;  // [m+1] first product of each row
    int64_t m;
    int32_t row_lo, row_hi;   // rows [row_lo, row_hi) (replay numeric)
    const unsigned long long* gate; // run only when gate[0..1] == gate[2..3]
    DevCounters* ctr;
    int32_t T;                // build: per-warp hash size (pow2 >= 2 * max row)
    int shift;                // build: 32 - log2(T)
    int wpb;
    uint64_t warp_bytes;
};
cudaError_t launch_fingerprint(int64_t rows, const int64_t* rowptr, const int32_t* cols, unsigned long long* out0,
                               unsigned long long* out1, cudaStream_t st);
cudaError_t launch_replay_build(ReplayLaunch R, int width, cudaStream_t st);
cudaError_t launch_replay_numeric(ReplayLaunch R, int width, int32_t max_row, cudaStream_t st);

void count_launch(int n = 1);
int sm_count();

#ifdef __CUDACC__
// compressed pairs indexed by absolute B positions of the (possibly offset) B view
__device__ __forceinline__ const int2* cpair_of(const RowLaunch& L)
{
    return L.cpair ? L.cpair - __ldg(L.b_rowptr) : nullptr;
}
#endif

} // namespace kk
