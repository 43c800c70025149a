// engine.hpp drop-in: the reference's C++ handle API
// (/root/reference/proj/include/spgemm/engine.hpp:79-103) implemented over the
// C ABI of libkkspgemm.so (include/kkspgemm.h).  A maintainer replaces
// proj/src/engine.cpp with this file and links libkkspgemm.so + libcudart;
// every other reference TU and every caller (cli.cpp bench/verify, the unit
// and acceptance tests) builds unchanged against the same header.
//
// The host SpgemmHandle stays the source of truth (handle copies and edits of
// handle.config / numeric_choice behave exactly as in the reference,
// acceptance_main.cpp:417-425).  Behind it, a small cache keeps the DEVICE
// handle and device operand buffers of recently used handles, keyed by the
// identity of the handle's c_row_offsets buffer and checked against a digest
// of every field the device plan depends on (row offsets included), so
//   * multiply() = symbolic() + numeric() uploads the operands once and runs
//     the numeric on the device handle symbolic() built;
//   * repeated numeric() on one handle (structure reuse) reaches the GPU's
//     slot replay from the third pass on;
//   * an Auto handle imported from host fields keeps the GPU's own plan.
// Operands and C travel through one pinned staging pair with the copies split
// into chunks that overlap (async H2D/D2H on one stream while the host copies
// the next chunk).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include <cuda_runtime.h>

#include "kkspgemm.h"
#include "spgemm/engine.hpp"

namespace spgemm {

namespace {

[[noreturn]] void raise(int rc)
{
    const std::string msg = spg_last_error();
    switch (rc) {
    case SPG_ERR_CONTRACT: throw ContractError(msg);
    case SPG_ERR_REUSE: throw ReuseError(msg);
    case SPG_ERR_POOL_SIZING: throw PoolSizingError(msg);
    case SPG_ERR_INTERNAL: throw std::logic_error(msg);
    default: throw SpgemmError(msg);
    }
}

void check(int rc)
{
    if (rc != SPG_OK)
        raise(rc);
}

void cuda(cudaError_t e)
{
    if (e != cudaSuccess)
        throw SpgemmError(std::string("CUDA: ") + cudaGetErrorString(e));
}

// host memcpy split over the host's cores (a single thread moves ~5-10 GB/s,
// well below the host link)
void par_copy(void* dst, const void* src, size_t n)
{
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (size_t{4} << 20) || hw == 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (n + hw - 1) / hw;
    for (unsigned t = 1; t < hw; ++t) {
        const size_t off = per * t;
        if (off >= n)
            break;
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(per, n - off));
        });
    }
    std::memcpy(dst, src, std::min(per, n));
    for (auto& x : th)
        x.join();
}

// A vector about to be value-initialised to n elements: its storage is
// reserved, marked for huge pages and its pages populated from several
// threads (the kernel's page faults then run in parallel instead of inside
// the single-threaded fill), so resize's zero-fill runs at memset speed.
// Without MADV_POPULATE_WRITE (Linux < 5.14) this is just resize.
template <class T> void fill_fresh(std::vector<T>& v, size_t n)
{
    const size_t bytes = n * sizeof(T);
    if (bytes >= (size_t{64} << 20) && v.capacity() < n) {
        v.reserve(n);
        const uintptr_t pg = 4096;
        char* a0 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(v.data()) + pg - 1) & ~(pg - 1));
        char* a1 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(v.data()) + bytes) & ~(pg - 1));
        if (a1 > a0) {
            madvise(a0, static_cast<size_t>(a1 - a0), MADV_HUGEPAGE);
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
            const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
            const size_t len = static_cast<size_t>(a1 - a0);
            const size_t per = ((len + hw - 1) / hw + pg - 1) & ~(pg - 1);
            std::vector<std::thread> th;
            for (unsigned t = 0; t < hw; ++t) {
                const size_t off = per * t;
                if (off >= len)
                    break;
                th.emplace_back([=] { madvise(a0 + off, std::min(per, len - off), MADV_POPULATE_WRITE); });
            }
            for (auto& x : th)
                x.join();
        }
    }
    v.resize(n);
}

// pinned staging: host vectors are pageable, so copies go through a pinned
// bounce buffer in chunks, the (multi-threaded) host copy of chunk i+1
// overlapping the DMA of chunk i
struct Staging {
    static constexpr size_t kChunk = size_t{64} << 20;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    Staging()
    {
        for (int q = 0; q < 2; ++q) {
            cuda(cudaHostAlloc(&buf[q], kChunk, cudaHostAllocPortable));
            cuda(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
        }
    }
    ~Staging()
    {
        for (int q = 0; q < 2; ++q) {
            if (done[q])
                cudaEventDestroy(done[q]);
            if (buf[q])
                cudaFreeHost(buf[q]);
        }
    }
    Staging(const Staging&) = delete;
    Staging& operator=(const Staging&) = delete;

    void up(void* dst, const void* src, size_t bytes, cudaStream_t st)
    {
        const char* s = static_cast<const char*>(src);
        char* d = static_cast<char*>(dst);
        for (size_t off = 0, q = 0; off < bytes; off += kChunk, q ^= 1) {
            const size_t n = bytes - off < kChunk ? bytes - off : kChunk;
            cuda(cudaEventSynchronize(done[q])); // the buffer's previous DMA has drained
            par_copy(buf[q], s + off, n);
            cuda(cudaMemcpyAsync(d + off, buf[q], n, cudaMemcpyHostToDevice, st));
            cuda(cudaEventRecord(done[q], st));
        }
    }

    void down(void* dst, const void* src, size_t bytes, cudaStream_t st)
    {
        const char* s = static_cast<const char*>(src);
        char* d = static_cast<char*>(dst);
        size_t pend_off[2] = {0, 0}, pend_n[2] = {0, 0};
        auto drain = [&](int q) {
            if (pend_n[q]) {
                cuda(cudaEventSynchronize(done[q]));
                par_copy(d + pend_off[q], buf[q], pend_n[q]);
                pend_n[q] = 0;
            }
        };
        int q = 0;
        for (size_t off = 0; off < bytes; off += kChunk, q ^= 1) {
            const size_t n = bytes - off < kChunk ? bytes - off : kChunk;
            drain(q);
            cuda(cudaMemcpyAsync(buf[q], s + off, n, cudaMemcpyDeviceToHost, st));
            cuda(cudaEventRecord(done[q], st));
            pend_off[q] = off;
            pend_n[q] = n;
        }
        drain(q);
        drain(q ^ 1);
    }
};

// device copy of one host CSR (buffers grow, never shrink)
struct DevCsr {
    int64_t* ro = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
    size_t cap_rows = 0, cap_nnz = 0;
    spg_csr view{};
    DevCsr() = default;
    DevCsr(const DevCsr&) = delete;
    DevCsr& operator=(const DevCsr&) = delete;
    ~DevCsr()
    {
        cudaFree(ro);
        cudaFree(ci);
        cudaFree(v);
    }
    void upload(const CsrMatrix& m, Staging& stg, cudaStream_t st, bool values_only)
    {
        const int64_t nnz = m.nnz();
        const size_t rows = static_cast<size_t>(m.num_rows) + 1;
        const size_t n = static_cast<size_t>(nnz > 0 ? nnz : 1);
        if (rows > cap_rows) {
            cudaFree(ro);
            cuda(cudaMalloc(&ro, sizeof(int64_t) * rows));
            cap_rows = rows;
            values_only = false;
        }
        if (n > cap_nnz) {
            cudaFree(ci);
            cudaFree(v);
            cuda(cudaMalloc(&ci, sizeof(int32_t) * n));
            cuda(cudaMalloc(&v, sizeof(double) * n));
            cap_nnz = n;
            values_only = false;
        }
        if (!values_only) {
            if (m.row_offsets.empty())
                cuda(cudaMemsetAsync(ro, 0, sizeof(int64_t), st));
            else
                stg.up(ro, m.row_offsets.data(), sizeof(int64_t) * m.row_offsets.size(), st);
            if (nnz > 0)
                stg.up(ci, m.col_indices.data(), sizeof(int32_t) * nnz, st);
        }
        if (nnz > 0)
            stg.up(v, m.values.data(), sizeof(double) * nnz, st);
        view = spg_csr{m.num_rows, m.num_cols, nnz, ro, ci, v};
    }
};

spg_config to_c(const SpgemmConfig& c)
{
    spg_config o{};
    o.scheme = static_cast<int32_t>(c.scheme);
    o.accumulator = static_cast<int32_t>(c.accumulator);
    o.l1_capacity = c.l1_capacity;
    o.dense_cutoff_k = c.dense_cutoff_k;
    o.avg_flops_cutoff = c.avg_flops_cutoff;
    o.lp_max_occupancy = c.lp_max_occupancy;
    o.compression_gate = c.compression_gate;
    o.compression = static_cast<int32_t>(c.compression);
    o.collapse_divisor = c.collapse_divisor;
    o.worker_count = c.worker_count;
    o.sort_output = c.sort_output ? 1 : 0;
    o.row_block = c.row_block;
    o.pool_mode = static_cast<int32_t>(c.pool_mode);
    o.pool_budget_bytes = c.pool_budget_bytes;
    return o;
}

ResolvedConfig from_c(const spg_resolved& r)
{
    ResolvedConfig o;
    o.accumulator = static_cast<AccumulatorKind>(r.accumulator);
    o.scheme = static_cast<Scheme>(r.scheme);
    o.l1_capacity = r.l1_capacity;
    o.effective_k = r.effective_k;
    o.l2_capacity = r.l2_capacity;
    return o;
}

spg_resolved to_c(const ResolvedConfig& r)
{
    return spg_resolved{static_cast<int32_t>(r.accumulator), static_cast<int32_t>(r.scheme), r.l1_capacity,
                        r.effective_k, r.l2_capacity};
}

spg_flops_stats to_c(const FlopsStats& s)
{
    return spg_flops_stats{s.total_flops, s.max_row_flops, s.avg_degree_a, s.avg_row_flops};
}

spg_compression_report to_c(const CompressionReport& r)
{
    return spg_compression_report{r.cf, r.cmrf, r.compressed_flops, r.compressed_max_row_flops,
                                  r.applied ? 1 : 0};
}

struct HandleGuard {
    spg_handle_t h = nullptr;
    ~HandleGuard() { spg_handle_destroy(h); }
};

// ---- device-handle cache ------------------------------------------------------
uint64_t mix(uint64_t h, uint64_t x)
{
    h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    return h;
}

uint64_t bytes_digest(uint64_t h, const void* p, size_t n)
{
    const unsigned char* b = static_cast<const unsigned char*>(p);
    size_t q = 0;
    for (; q + 8 <= n; q += 8) {
        uint64_t x;
        std::memcpy(&x, b + q, 8);
        h = mix(h, x);
    }
    for (; q < n; ++q)
        h = mix(h, b[q]);
    return h;
}

// every host field the device plan depends on
uint64_t handle_digest(const SpgemmHandle& h)
{
    uint64_t d = 0x6B6B7370;
    for (int64_t x : {int64_t{h.m}, int64_t{h.n}, int64_t{h.k}, h.nnz_a, h.nnz_b, h.max_row_size})
        d = mix(d, static_cast<uint64_t>(x));
    const spg_config c = to_c(h.config);
    const spg_resolved r = to_c(h.numeric_choice);
    d = bytes_digest(d, &c, sizeof(c));
    d = bytes_digest(d, &r, sizeof(r));
    return bytes_digest(d, h.c_row_offsets.data(), sizeof(int64_t) * h.c_row_offsets.size());
}

struct Entry {
    const void* key = nullptr;   // the host handle's c_row_offsets buffer
    uint64_t digest = 0;
    spg_handle_t h = nullptr;
    DevCsr a, b;
    bool b_is_a = false;
    const CsrMatrix* fresh_a = nullptr; // operands symbolic() just uploaded
    const CsrMatrix* fresh_b = nullptr;
    int32_t* dc = nullptr;
    double* dv = nullptr;
    size_t cap_c = 0;
    Staging* stg = nullptr; // the cache's (used under its mutex)
    uint64_t last_use = 0;
    Entry() = default;
    Entry(const Entry&) = delete;
    Entry& operator=(const Entry&) = delete;
    ~Entry()
    {
        spg_handle_destroy(h);
        cudaFree(dc);
        cudaFree(dv);
    }
    const spg_csr* bview() const { return b_is_a ? &a.view : &b.view; }
    void upload(const CsrMatrix& x, const CsrMatrix& y)
    {
        a.upload(x, *stg, nullptr, false);
        b_is_a = &x == &y;
        if (!b_is_a)
            b.upload(y, *stg, nullptr, false);
    }
};

class Cache {
public:
    static Cache& get()
    {
        static Cache c;
        return c;
    }
    std::mutex mu;
    // one pinned staging pair for every transfer (pinned allocation is slow
    // and synchronises the device: never per call)
    Staging& staging()
    {
        if (!stg)
            stg = std::make_unique<Staging>();
        return *stg;
    }
    // a few entries: every one holds the operands and C on the device
    size_t capacity() const
    {
        const char* e = std::getenv("KK_SHIM_CACHE");
        return e ? static_cast<size_t>(std::max(0, std::atoi(e))) : 2;
    }
    Entry* find(const void* key, uint64_t digest)
    {
        for (auto& e : entries)
            if (e->key == key && e->digest == digest) {
                e->last_use = ++clock;
                return e.get();
            }
        return nullptr;
    }
    Entry* insert(std::unique_ptr<Entry> e)
    {
        for (auto it = entries.begin(); it != entries.end();)
            if ((*it)->key == e->key)
                it = entries.erase(it); // a stale entry of the same buffer
            else
                ++it;
        const size_t cap = capacity();
        if (cap == 0) {
            scratch = std::move(e);
            return scratch.get();
        }
        while (entries.size() >= cap) {
            auto lru = std::min_element(entries.begin(), entries.end(),
                                        [](const auto& x, const auto& y) { return x->last_use < y->last_use; });
            entries.erase(lru);
        }
        e->last_use = ++clock;
        entries.push_back(std::move(e));
        return entries.back().get();
    }

private:
    std::unique_ptr<Staging> stg;
    std::vector<std::unique_ptr<Entry>> entries;
    std::unique_ptr<Entry> scratch; // the uncached entry of the last call (KK_SHIM_CACHE=0)
    uint64_t clock = 0;
};

std::unique_ptr<Entry> import_entry(const SpgemmHandle& handle)
{
    spg_handle_desc d{};
    d.m = handle.m;
    d.n = handle.n;
    d.k = handle.k;
    d.nnz_a = handle.nnz_a;
    d.nnz_b = handle.nnz_b;
    d.c_row_offsets = handle.c_row_offsets.data();
    d.flops = to_c(handle.flops);
    d.compression = to_c(handle.compression);
    d.max_row_size = handle.max_row_size;
    d.avg_row_size = handle.avg_row_size;
    d.avg_row_size_estimate = handle.avg_row_size_estimate;
    d.symbolic_choice = to_c(handle.symbolic_choice);
    d.numeric_choice = to_c(handle.numeric_choice);
    d.config = to_c(handle.config);
    d.symbolic_stats = spg_phase_stats{handle.symbolic_stats.ms, handle.symbolic_stats.pool_allocations,
                                       handle.symbolic_stats.l2_inserts};
    d.compress_ms = handle.compress_ms;
    d.per_row_flops = handle.flops.per_row_flops.size() == static_cast<size_t>(handle.m)
        ? handle.flops.per_row_flops.data()
        : nullptr;
    auto e = std::make_unique<Entry>();
    check(spg_handle_import(&d, &e->h, nullptr));
    return e;
}

} // namespace

std::pair<index_t, flops_t> flat_position(std::span<const flops_t> prefix, flops_t t)
{
    int32_t seg = 0;
    int64_t off = 0;
    check(spg_flat_position(prefix.data(), static_cast<int64_t>(prefix.size()), t, &seg, &off));
    return {seg, off};
}

ResolvedConfig resolve_config(Phase phase, index_t k, const FlopsStats& stats, const CompressionReport& report,
                              const SpgemmConfig& cfg, flops_t row_upper_bound)
{
    const spg_flops_stats s = to_c(stats);
    const spg_compression_report r = to_c(report);
    const spg_config c = to_c(cfg);
    spg_resolved out{};
    check(spg_resolve_config(static_cast<int32_t>(phase), k, &s, &r, &c, row_upper_bound, &out));
    return from_c(out);
}

SpgemmHandle symbolic(const CsrMatrix& a, const CsrMatrix& b, const SpgemmConfig& cfg)
{
    if (a.num_cols != b.num_rows)
        throw ContractError("symbolic: inner dimensions do not match");
    Cache& cache = Cache::get();
    std::lock_guard<std::mutex> lk(cache.mu);
    auto e = std::make_unique<Entry>();
    e->stg = &cache.staging();
    e->upload(a, b);
    const spg_config c = to_c(cfg);
    check(spg_symbolic(&e->a.view, e->bview(), &c, &e->h, nullptr));
    spg_handle_info info{};
    check(spg_handle_info_get(e->h, &info));

    SpgemmHandle h;
    h.config = cfg;
    h.m = info.m;
    h.n = info.n;
    h.k = info.k;
    h.nnz_a = info.nnz_a;
    h.nnz_b = info.nnz_b;
    h.c_row_offsets.resize(static_cast<size_t>(info.m) + 1);
    check(spg_handle_copy_row_offsets(e->h, h.c_row_offsets.data()));
    h.flops.per_row_flops.resize(static_cast<size_t>(info.m));
    if (info.m > 0)
        check(spg_handle_copy_per_row_flops(e->h, h.flops.per_row_flops.data()));
    h.flops.total_flops = info.flops.total_flops;
    h.flops.max_row_flops = info.flops.max_row_flops;
    h.flops.avg_degree_a = info.flops.avg_degree_a;
    h.flops.avg_row_flops = info.flops.avg_row_flops;
    h.compression.cf = info.compression.cf;
    h.compression.cmrf = info.compression.cmrf;
    h.compression.compressed_flops = info.compression.compressed_flops;
    h.compression.compressed_max_row_flops = info.compression.compressed_max_row_flops;
    h.compression.applied = info.compression.applied != 0;
    h.max_row_size = info.max_row_size;
    h.avg_row_size = info.avg_row_size;
    h.avg_row_size_estimate = info.avg_row_size_estimate;
    h.symbolic_choice = from_c(info.symbolic_choice);
    h.numeric_choice = from_c(info.numeric_choice);
    h.symbolic_stats.ms = info.symbolic_stats.ms;
    h.symbolic_stats.pool_allocations = info.symbolic_stats.pool_allocations;
    h.symbolic_stats.l2_inserts = info.symbolic_stats.l2_inserts;
    h.compress_ms = info.compress_ms;
    // keep the device handle and the uploaded operands for numeric() on this
    // handle (the vector's buffer moves with the returned handle)
    e->key = h.c_row_offsets.data();
    e->digest = handle_digest(h);
    e->fresh_a = &a;
    e->fresh_b = &b;
    cache.insert(std::move(e));
    return h;
}

namespace {

// same_call: a multiply() running numeric right after its own symbolic, so the
// operands symbolic() uploaded are still the caller's (numeric() alone always
// uploads: the caller may have changed values or structure since)
CsrMatrix numeric_impl(const CsrMatrix& a, const CsrMatrix& b, const SpgemmHandle& handle, PhaseStats* stats,
                       bool same_call)
{
    // engine.cpp:451-453, checked before any device work
    if (a.num_rows != handle.m || a.num_cols != handle.n || b.num_rows != handle.n || b.num_cols != handle.k
        || a.nnz() != handle.nnz_a || b.nnz() != handle.nnz_b)
        throw ReuseError("numeric: operands do not match the symbolic handle");

    // C's owning vectors are value-initialised by resize (the reference's
    // NumericSink pays the same zero-fill, engine.cpp:456-461): done on two
    // threads while the operands upload and the GPU computes
    const int64_t nnz = handle.nnz_c();
    CsrMatrix c;
    c.num_rows = handle.m;
    c.num_cols = handle.k;
    std::thread fill_c([&] { fill_fresh(c.col_indices, static_cast<size_t>(nnz)); });
    std::thread fill_v([&] { fill_fresh(c.values, static_cast<size_t>(nnz)); });
    struct Join {
        std::thread& a;
        std::thread& b;
        ~Join()
        {
            if (a.joinable())
                a.join();
            if (b.joinable())
                b.join();
        }
    } join{fill_c, fill_v};
    Cache& cache = Cache::get();
    std::lock_guard<std::mutex> lk(cache.mu);
    const uint64_t dig = handle_digest(handle);
    Entry* e = cache.find(handle.c_row_offsets.data(), dig);
    if (!e) {
        auto ne = import_entry(handle);
        ne->stg = &cache.staging();
        ne->key = handle.c_row_offsets.data();
        ne->digest = dig;
        e = cache.insert(std::move(ne));
    }
    if (!(same_call && e->fresh_a == &a && e->fresh_b == &b))
        e->upload(a, b);
    e->fresh_a = e->fresh_b = nullptr;
    const size_t need = static_cast<size_t>(nnz > 0 ? nnz : 1);
    if (need > e->cap_c) {
        cudaFree(e->dc);
        cudaFree(e->dv);
        e->dc = nullptr;
        e->dv = nullptr;
        cuda(cudaMalloc(&e->dc, sizeof(int32_t) * need));
        cuda(cudaMalloc(&e->dv, sizeof(double) * need));
        e->cap_c = need;
    }
    spg_phase_stats st{};
    check(spg_numeric(e->h, &e->a.view, e->bview(), e->dc, e->dv, stats ? &st : nullptr, nullptr));
    c.row_offsets = handle.c_row_offsets;
    fill_c.join();
    fill_v.join();
    if (nnz > 0) {
        e->stg->down(c.col_indices.data(), e->dc, sizeof(int32_t) * nnz, nullptr);
        e->stg->down(c.values.data(), e->dv, sizeof(double) * nnz, nullptr);
    }
    check(spg_handle_check(e->h)); // errors of an asynchronous pass (the reference's logic_error)
    c.sorted_rows = handle.config.sort_output;
    if (stats) {
        stats->ms = st.ms;
        stats->pool_allocations = st.pool_allocations;
        stats->l2_inserts = st.l2_inserts;
    }
    return c;
}

} // namespace

CsrMatrix numeric(const CsrMatrix& a, const CsrMatrix& b, const SpgemmHandle& handle, PhaseStats* stats)
{
    return numeric_impl(a, b, handle, stats, false);
}

MultiplyResult multiply(const CsrMatrix& a, const CsrMatrix& b, const SpgemmConfig& cfg)
{
    MultiplyResult r;
    r.handle = symbolic(a, b, cfg);
    r.c = numeric_impl(a, b, r.handle, &r.numeric_stats, true);
    return r;
}

} // namespace spgemm
