// TEST INFRASTRUCTURE ONLY — a C wrapper over the UNMODIFIED reference
// library, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libspgemm_ref.so.  Used as (1) the pin for the C restatement
// (oracle/spgemm_oracle.c), (2) the golden-fixture generator
// (tests/golden/make_golden.py) and (3) the CPU baseline / `bench.py --impl
// reference` arm.  Nothing in the product path links it.
//
// The wrapped API is the reference's own: spgemm::symbolic / numeric /
// multiply (include/spgemm/engine.hpp:79-103), flops_stats
// (csr_matrix.hpp:58), compressed_row_sizes / decide_compression
// (compression.hpp:36-69), build_csr / transpose (csr_matrix.hpp:40-42),
// generate_synthetic (synthetic.hpp:17) and the test fixtures
// tests/test_util.hpp:14-58.

#include <chrono>
#include <cstring>
#include <exception>
#include <random>
#include <string>

#include "spgemm/bench.hpp"
#include "spgemm/compression.hpp"
#include "spgemm/csr_matrix.hpp"
#include "spgemm/engine.hpp"
#include "spgemm/matrix_market.hpp"
#include "spgemm/oracle.hpp"
#include "spgemm/synthetic.hpp"
#include "test_util.hpp"

using namespace spgemm;

namespace {
thread_local std::string g_err;

template <class F> int guard(F&& f)
{
    try {
        f();
        return 0;
    } catch (const ReuseError& e) {
        g_err = e.what();
        return 2;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 1;
    } catch (const PoolSizingError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}
} // namespace

extern "C" {

struct ref_cfg {
    int scheme;
    int accumulator;
    int32_t l1_capacity;
    int32_t dense_cutoff_k;
    double avg_flops_cutoff;
    double lp_max_occupancy;
    double compression_gate;
    int compression;
    int collapse_divisor;
    int worker_count;
    int sort_output;
    int32_t row_block;
    int pool_mode;
    int64_t pool_budget_bytes;
};

struct ref_info {
    int32_t m, n, k;
    int64_t nnz_a, nnz_b, nnz_c;
    int64_t total_flops, max_row_flops;
    double avg_degree_a, avg_row_flops;
    double cf, cmrf;
    int64_t compressed_flops, compressed_max_row_flops;
    int32_t applied;
    int64_t max_row_size;
    double avg_row_size, avg_row_size_estimate;
    int32_t sym_acc, sym_scheme, sym_l1, sym_effk, sym_l2;
    int32_t num_acc, num_scheme, num_l1, num_effk, num_l2;
    double sym_ms;
    int64_t sym_pool_allocations, sym_l2_inserts;
    double compress_ms;
};

struct ref_stats {
    double ms;
    int64_t pool_allocations, l2_inserts;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_cfg_default(ref_cfg* c)
{
    SpgemmConfig d;
    c->scheme = static_cast<int>(d.scheme);
    c->accumulator = static_cast<int>(d.accumulator);
    c->l1_capacity = d.l1_capacity;
    c->dense_cutoff_k = d.dense_cutoff_k;
    c->avg_flops_cutoff = d.avg_flops_cutoff;
    c->lp_max_occupancy = d.lp_max_occupancy;
    c->compression_gate = d.compression_gate;
    c->compression = static_cast<int>(d.compression);
    c->collapse_divisor = d.collapse_divisor;
    c->worker_count = d.worker_count;
    c->sort_output = d.sort_output ? 1 : 0;
    c->row_block = d.row_block;
    c->pool_mode = static_cast<int>(d.pool_mode);
    c->pool_budget_bytes = d.pool_budget_bytes;
}

static SpgemmConfig to_cfg(const ref_cfg* c)
{
    SpgemmConfig d;
    if (!c)
        return d;
    d.scheme = static_cast<Scheme>(c->scheme);
    d.accumulator = static_cast<AccumulatorKind>(c->accumulator);
    d.l1_capacity = c->l1_capacity;
    d.dense_cutoff_k = c->dense_cutoff_k;
    d.avg_flops_cutoff = c->avg_flops_cutoff;
    d.lp_max_occupancy = c->lp_max_occupancy;
    d.compression_gate = c->compression_gate;
    d.compression = static_cast<CompressionMode>(c->compression);
    d.collapse_divisor = c->collapse_divisor;
    d.worker_count = c->worker_count;
    d.sort_output = c->sort_output != 0;
    d.row_block = c->row_block;
    d.pool_mode = static_cast<PoolMode>(c->pool_mode);
    d.pool_budget_bytes = c->pool_budget_bytes;
    return d;
}

// ---- matrices ----------------------------------------------------------
void* ref_mat_new(int32_t rows, int32_t cols, const int64_t* rowptr, const int32_t* ci,
                  const double* vals, int sorted)
{
    auto* m = new CsrMatrix;
    m->num_rows = rows;
    m->num_cols = cols;
    m->row_offsets.assign(rowptr, rowptr + rows + 1);
    const int64_t base = rowptr[0];
    const int64_t nnz = rowptr[rows] - base;
    for (auto& r : m->row_offsets)
        r -= base;
    m->col_indices.assign(ci + base, ci + base + nnz);
    if (vals)
        m->values.assign(vals + base, vals + base + nnz);
    else
        m->values.assign(static_cast<std::size_t>(nnz), 1.0);
    m->sorted_rows = sorted != 0;
    return m;
}

void ref_mat_free(void* m) { delete static_cast<CsrMatrix*>(m); }

// the reference's MatrixMarket reader (matrix_market.cpp); NULL on error
void* ref_read_mm(const char* path)
{
    CsrMatrix* out = nullptr;
    const int rc = guard([&] { out = new CsrMatrix(read_matrix_market(path, nullptr)); });
    return rc == 0 ? out : nullptr;
}

void ref_mat_shape(void* mp, int32_t* rows, int32_t* cols, int64_t* nnz)
{
    const auto* m = static_cast<CsrMatrix*>(mp);
    *rows = m->num_rows;
    *cols = m->num_cols;
    *nnz = m->nnz();
}

void ref_mat_export(void* mp, int64_t* rowptr, int32_t* ci, double* vals)
{
    const auto* m = static_cast<CsrMatrix*>(mp);
    std::memcpy(rowptr, m->row_offsets.data(), sizeof(int64_t) * m->row_offsets.size());
    std::memcpy(ci, m->col_indices.data(), sizeof(int32_t) * m->col_indices.size());
    std::memcpy(vals, m->values.data(), sizeof(double) * m->values.size());
}

void* ref_build_csr(int32_t rows, int32_t cols, int64_t ntrip, const int32_t* r,
                    const int32_t* c, const double* v)
{
    void* out = nullptr;
    const int rc = guard([&] {
        std::vector<Triplet> t(static_cast<std::size_t>(ntrip));
        for (int64_t q = 0; q < ntrip; ++q)
            t[q] = {r[q], c[q], v[q]};
        out = new CsrMatrix(build_csr(rows, cols, t));
    });
    return rc == 0 ? out : nullptr;
}

void* ref_transpose(void* m) { return new CsrMatrix(transpose(*static_cast<CsrMatrix*>(m))); }

void* ref_generate_synthetic(int kind, int32_t rows, int32_t cols, int32_t target,
                             uint64_t seed)
{
    void* out = nullptr;
    guard([&] {
        out = new CsrMatrix(
            generate_synthetic(static_cast<SyntheticKind>(kind), rows, cols, target, seed));
    });
    return out;
}

// tests/test_util.hpp fixtures, driven by a caller-owned mt19937_64
void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }
void* ref_random_csr(void* rng, int32_t rows, int32_t cols, double density)
{
    return new CsrMatrix(test::random_csr(*static_cast<std::mt19937_64*>(rng), rows, cols, density));
}
void* ref_shuffle_rows(void* m, uint64_t seed)
{
    return new CsrMatrix(test::shuffle_rows(*static_cast<CsrMatrix*>(m), seed));
}
void* ref_synthetic_by_index(int idx, int32_t rows, int32_t cols, int32_t target, uint64_t seed)
{
    return new CsrMatrix(test::synthetic_by_index(idx, rows, cols, target, seed));
}

// ---- hot path ------------------------------------------------------------
int ref_flops_stats(void* a, void* b, int64_t* per_row, int64_t* total, int64_t* mx)
{
    return guard([&] {
        const FlopsStats s = flops_stats(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b));
        if (per_row)
            std::memcpy(per_row, s.per_row_flops.data(), sizeof(int64_t) * s.per_row_flops.size());
        *total = s.total_flops;
        *mx = s.max_row_flops;
    });
}

int ref_compressed_row_sizes(void* b, int32_t* out)
{
    return guard([&] {
        const auto s = compressed_row_sizes(*static_cast<CsrMatrix*>(b), 1);
        std::memcpy(out, s.data(), sizeof(int32_t) * s.size());
    });
}

int ref_decide_compression(void* a, void* b, double gate, int mode, int64_t* cflops,
                           int64_t* cmax, double* cf, double* cmrf, int* applied)
{
    return guard([&] {
        const CsrMatrix& A = *static_cast<CsrMatrix*>(a);
        const CsrMatrix& B = *static_cast<CsrMatrix*>(b);
        const auto d = decide_compression(A, B, flops_stats(A, B), gate,
                                          static_cast<CompressionMode>(mode), 1);
        *cflops = d.report.compressed_flops;
        *cmax = d.report.compressed_max_row_flops;
        *cf = d.report.cf;
        *cmrf = d.report.cmrf;
        *applied = d.report.applied ? 1 : 0;
    });
}

void* ref_symbolic(void* a, void* b, const ref_cfg* cfg)
{
    void* out = nullptr;
    guard([&] {
        out = new SpgemmHandle(
            symbolic(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b), to_cfg(cfg)));
    });
    return out;
}

void ref_handle_free(void* h) { delete static_cast<SpgemmHandle*>(h); }

static void fill_rc(const ResolvedConfig& r, int32_t* acc, int32_t* sch, int32_t* l1,
                    int32_t* effk, int32_t* l2)
{
    *acc = static_cast<int32_t>(r.accumulator);
    *sch = static_cast<int32_t>(r.scheme);
    *l1 = r.l1_capacity;
    *effk = r.effective_k;
    *l2 = r.l2_capacity;
}

int ref_handle_info(void* hp, ref_info* o)
{
    const auto& h = *static_cast<SpgemmHandle*>(hp);
    o->m = h.m;
    o->n = h.n;
    o->k = h.k;
    o->nnz_a = h.nnz_a;
    o->nnz_b = h.nnz_b;
    o->nnz_c = h.nnz_c();
    o->total_flops = h.flops.total_flops;
    o->max_row_flops = h.flops.max_row_flops;
    o->avg_degree_a = h.flops.avg_degree_a;
    o->avg_row_flops = h.flops.avg_row_flops;
    o->cf = h.compression.cf;
    o->cmrf = h.compression.cmrf;
    o->compressed_flops = h.compression.compressed_flops;
    o->compressed_max_row_flops = h.compression.compressed_max_row_flops;
    o->applied = h.compression.applied ? 1 : 0;
    o->max_row_size = h.max_row_size;
    o->avg_row_size = h.avg_row_size;
    o->avg_row_size_estimate = h.avg_row_size_estimate;
    fill_rc(h.symbolic_choice, &o->sym_acc, &o->sym_scheme, &o->sym_l1, &o->sym_effk, &o->sym_l2);
    fill_rc(h.numeric_choice, &o->num_acc, &o->num_scheme, &o->num_l1, &o->num_effk, &o->num_l2);
    o->sym_ms = h.symbolic_stats.ms;
    o->sym_pool_allocations = h.symbolic_stats.pool_allocations;
    o->sym_l2_inserts = h.symbolic_stats.l2_inserts;
    o->compress_ms = h.compress_ms;
    return 0;
}

int ref_handle_rowptr(void* hp, int64_t* out)
{
    const auto& h = *static_cast<SpgemmHandle*>(hp);
    std::memcpy(out, h.c_row_offsets.data(), sizeof(int64_t) * h.c_row_offsets.size());
    return 0;
}

int ref_handle_per_row_flops(void* hp, int64_t* out)
{
    const auto& h = *static_cast<SpgemmHandle*>(hp);
    std::memcpy(out, h.flops.per_row_flops.data(), sizeof(int64_t) * h.flops.per_row_flops.size());
    return 0;
}

// Overrides on a handle, as SURVEY Appendix A's forced-variant probes and
// acceptance_main.cpp:417-425 do.
void ref_handle_set_workers(void* hp, int workers)
{
    static_cast<SpgemmHandle*>(hp)->config.worker_count = workers;
}

int ref_numeric(void* a, void* b, void* hp, int32_t* c_cols, double* c_vals, ref_stats* st)
{
    return guard([&] {
        PhaseStats ps;
        const CsrMatrix c = numeric(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b),
                                    *static_cast<SpgemmHandle*>(hp), &ps);
        if (c_cols)
            std::memcpy(c_cols, c.col_indices.data(), sizeof(int32_t) * c.col_indices.size());
        if (c_vals)
            std::memcpy(c_vals, c.values.data(), sizeof(double) * c.values.size());
        if (st) {
            st->ms = ps.ms;
            st->pool_allocations = ps.pool_allocations;
            st->l2_inserts = ps.l2_inserts;
        }
    });
}

// One full NoReuse multiply (cli.cpp:137-151 semantics); returns wall ms.
double ref_multiply_ms(void* a, void* b, const ref_cfg* cfg, int64_t* nnz_c)
{
    double ms = -1.0;
    guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const MultiplyResult r =
            multiply(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b), to_cfg(cfg));
        ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                 .count();
        if (nnz_c)
            *nnz_c = r.c.nnz();
    });
    return ms;
}

// the reference's results reader + Dolan-Moré profile (bench.cpp:55-175), as
// cli.cpp:291-298 chains them; returns 0 or the guard code
int ref_profile_csv(const char* in, const char* out, int points)
{
    return guard([&] { write_profile_csv(out, compute_profile(read_bench_csv(in), points)); });
}

// gustavson_serial multiplication count (oracle.cpp:9-48)
int64_t ref_gustavson_mults(void* a, void* b)
{
    int64_t n = -1;
    guard([&] {
        n = gustavson_serial(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b))
                .multiplications;
    });
    return n;
}

} // extern "C"
