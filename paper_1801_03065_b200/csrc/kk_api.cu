// C ABI of libkkspgemm.so (include/kkspgemm.h) and the host orchestration of
// the two phases.  The host takes exactly the decisions the reference takes
// on the host (compression gate compression.cpp:131-147, resolve_config
// engine.cpp:367-395, scans' totals engine.cpp:434-441); everything that
// touches matrix data runs in the kernels of kk_kernels.cu.
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstddef>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kkspgemm.h"
#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {
long long launch_count();
}

using namespace kk;

namespace {

thread_local std::string g_err;

struct ApiError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError{code, msg}; }

void cuda_check(cudaError_t e, const char* what)
{
    if (e == cudaSuccess)
        return;
    if (e == cudaErrorMemoryAllocation)
        fail(SPG_ERR_NOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(SPG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F> int guarded(F&& f)
{
    try {
        f();
        g_err.clear();
        return SPG_OK;
    } catch (const ApiError& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SPG_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPG_ERR_INTERNAL;
    }
}

void require_device()
{
    static int ok = [] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            return 0;
        // keep freed stream-ordered memory in the pool: repeated phases then
        // allocate without touching the driver
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        return 1;
    }();
    if (!ok)
        fail(SPG_ERR_CUDA, "no CUDA device: libkkspgemm has no CPU path");
}

int ceil_pow2_i(int64_t x)
{
    int64_t p = 1;
    while (p < x)
        p <<= 1;
    return static_cast<int>(p);
}

int log2_i(int64_t p)
{
    int l = 0;
    while ((int64_t{1} << l) < p)
        ++l;
    return l;
}

int host_bucket(unsigned long long x)
{
    if (x == 0)
        return 0;
    if (x == 1)
        return 1;
    return std::min(65 - __builtin_clzll(x - 1), 63);
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

constexpr uint64_t kWarpSmemMax = 48 * 1024; // L1 accumulator budget per warp
constexpr double kTinyMaxAvgArow = 8.0;        // thread-per-row classes only for short A rows
#ifndef KK_HEAVY_SYM_WORDS
#define KK_HEAVY_SYM_WORDS 49152
#endif
constexpr int32_t kHeavySymWords = KK_HEAVY_SYM_WORDS; // dense bitmap words per CTA (heavy symbolic)
constexpr int32_t kHeavyBucketKeys = 256;     // numeric heavy rows: ~distinct columns per hashed bucket
constexpr int32_t kHeavyMaxBuckets = 1536;    // buckets per row (shared-memory histogram bound)
constexpr int64_t kHeavyMaxRow = int64_t{kHeavyMaxBuckets} * 320; // <= 62.5% load of the 512-slot tables
constexpr uint64_t kCtaSmem = 96 * 1024;     // two CTAs per SM

// device-side allocation helper (stream ordered)
template <class T> T* dalloc(size_t count, cudaStream_t st, const char* what)
{
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, std::max<size_t>(count * sizeof(T), 16), st), what);
    return static_cast<T*>(p);
}

// Key capacity of the reference's level-1 accumulator for a resolved choice:
// LlAccumulator holds l1_capacity keys (accumulators.hpp:63-151), the owning
// LpAccumulator max_new = min(ceil(occ * cap), cap - 1) with cap =
// ceil_pow2(ceil(l1 / occ)) (accumulators.hpp:158-190), Dense is single-level.
// Used only for the reference's PhaseStats (pool_allocations, l2_inserts).
int32_t ref_l1_keys(const spg_resolved& rc, double occ)
{
    const int64_t l1 = std::max<int64_t>(rc.l1_capacity, 1);
    if (rc.accumulator == SPG_ACC_LL)
        return static_cast<int32_t>(l1);
    if (rc.accumulator == SPG_ACC_LP) {
        const double o = std::max(occ, 1e-6);
        const int64_t cap = ceil_pow2_i(static_cast<int64_t>(std::ceil(static_cast<double>(l1) / o)));
        return static_cast<int32_t>(std::min<int64_t>(static_cast<int64_t>(std::ceil(occ * cap)), cap - 1));
    }
    return INT32_MAX;
}

// plan_pool's PoolSizingError (memory_pool.cpp:97-99): the reference sizes a
// pool for every LL/LP phase, one chunk = l2_capacity slots rounded to a
// 64-byte line (32 bytes per slot); a chunk above the budget is an error even
// when no row would spill.
void check_pool_budget(const spg_resolved& rc, int64_t budget)
{
    if (rc.accumulator != SPG_ACC_LL && rc.accumulator != SPG_ACC_LP)
        return;
    const int64_t bound = std::max<int64_t>(rc.l2_capacity, 1);
    const int64_t chunk = (bound + 1) / 2 * 2 * 32;
    if (chunk > budget)
        fail(SPG_ERR_POOL_SIZING, "plan_pool: a single chunk exceeds the memory budget");
}

} // namespace

namespace kk {

TabLayout make_layout(int acc, int variant, int32_t S, int32_t domain, double occupancy,
                      bool external_rows)
{
    TabLayout L;
    L.acc = acc;
    L.S = std::max<int32_t>(S, 1);
    const uint64_t pb = variant == kVarNumeric ? 8 : 4;
    L.has_ids = !external_rows;
    L.has_pay = !external_rows && variant != kVarSymRaw;
    uint64_t map_bytes = 0, aux_bytes = 0;
    if (acc == kAccLP) {
        const double occ = std::clamp(occupancy, 1e-6, 1.0);
        const int64_t need = static_cast<int64_t>(std::ceil(L.S / occ));
        L.T = std::max({ceil_pow2_i(need), ceil_pow2_i(int64_t{L.S} + 1), 32});
        L.shift = 32 - log2_i(L.T);
        map_bytes = 8ull * L.T;
        aux_bytes = 4ull * L.S;
    } else if (acc == kAccLL) {
        L.T = std::max(ceil_pow2_i(L.S), 32);
        L.shift = 32 - log2_i(L.T);
        map_bytes = 4ull * L.T;
        aux_bytes = 4ull * L.S;
    } else {
        L.T = std::max<int32_t>(domain, 1);
        map_bytes = 4ull * L.T;
    }
    L.off_map = 0;
    L.off_aux = static_cast<uint32_t>(align_up(map_bytes, 16));
    L.off_ids = static_cast<uint32_t>(align_up(L.off_aux + aux_bytes, 16));
    L.off_pay = static_cast<uint32_t>(align_up(L.off_ids + (L.has_ids ? 4ull * L.S : 0), 16));
    L.bytes = align_up(L.off_pay + (L.has_pay ? pb * L.S : 0), 16);
    return L;
}

} // namespace kk

// ---------------------------------------------------------------------------
// plans: row classes of one phase
// ---------------------------------------------------------------------------
namespace {

struct PhaseClass {
    TabLayout lay;
    bool l2 = false;
    bool fast = false;
    bool tiny = false; // a thread per row (kk_tiny.cu)
    int wpb = 8;
    int grid = 0;
    int64_t count = 0;
    int64_t off = 0;
};

// level-2 (HBM pool) launch shape for rows whose bound is s_true
struct L2Spec {
    bool valid = false;
    TabLayout lay;
    uint64_t chunk_bytes = 0;
    int32_t num_chunks = 0;
    int pool_mode = 0;
    int wpb = 8;
    int grid = 0;
};

struct PhasePlan {
    int acc = kAccLP;
    bool flat = false;
    bool fast = false;      // fast kernels (kk_fast.cu) for the L1 classes
    bool optimistic = false; // L1 tables sized below the bound; overflow rows retry in L2
    int variant = kVarNumeric;
    int32_t domain = 0;
    std::vector<PhaseClass> classes;
    BinParams bp{};
    bool need_list = false; // more than one class: rows are binned
    L2Spec l2;
    int l2_class = -1;
    bool short_rows = false; // symbolic fast kernel: rows pipelined 32 at a time
};

// GPU meta-algorithm (PAPER.md:849-852 and Table tab:methods): kkmem (LL,
// Thread-Sequential) when the average row flops are below the cutoff, kklp
// (two-level LP, Thread-Flat-Parallel) otherwise.  A dense accumulator is used
// when its map over the column domain is no larger than the hash table the
// row bound needs and it fits the warp's L1 budget (column count vs max row
// flops).  Forced configurations use the resolved choice as is.
void device_choice(bool forced, const spg_resolved& rc, const spg_config& cfg, double avg_row_flops,
                   int variant, int32_t domain, int64_t umax, int* acc, bool* flat)
{
    if (forced) {
        *acc = rc.accumulator == SPG_ACC_LL ? kAccLL : rc.accumulator == SPG_ACC_DENSE ? kAccDense : kAccLP;
        *flat = rc.scheme == SPG_SCHEME_FLAT_PARALLEL;
        return;
    }
    if (avg_row_flops < cfg.avg_flops_cutoff) {
        *acc = kAccLL;
        *flat = false;
    } else {
        *acc = kAccLP;
        *flat = true;
    }
    const int32_t s = static_cast<int32_t>(std::max<int64_t>(std::min<int64_t>(umax, domain), 1));
    const TabLayout dense = make_layout(kAccDense, variant, s, domain, cfg.lp_max_occupancy, false);
    const TabLayout hashed = make_layout(*acc, variant, s, domain, cfg.lp_max_occupancy, false);
    if (dense.bytes <= hashed.bytes && dense.bytes <= kWarpSmemMax)
        *acc = kAccDense;
}

// fast-kernel layouts (kk_fast.cu): numeric slots {key,pos,val} 16 B + slot_of;
// symbolic slots {key,word} 8 B
TabLayout make_layout_fast(int variant, int32_t S, double occupancy)
{
    TabLayout L;
    L.acc = kAccLP;
    L.S = std::max<int32_t>(S, 1);
    const double occ = std::clamp(occupancy, 1e-6, 1.0);
    const int64_t need = static_cast<int64_t>(std::ceil(L.S / occ));
    L.T = std::max({ceil_pow2_i(need), ceil_pow2_i(int64_t{L.S} + 1), 64});
    L.shift = 32 - log2_i(L.T); // hash shift (kk_fast.cu)
    if (variant == kVarNumeric) {
        L.off_map = 0;                                          // vals  [T] double
        L.off_ids = static_cast<uint32_t>(8ull * L.T);          // keys  [T] int32
        L.off_aux = static_cast<uint32_t>(12ull * L.T);         // slot_of [S]
        L.off_pay = static_cast<uint32_t>(align_up(12ull * L.T + 4ull * L.S, 16)); // step stage
        L.bytes = L.off_pay + 768; // StepStage
    } else {
        L.off_ids = 0;                                          // keys  [T]
        L.off_map = static_cast<uint32_t>(4ull * L.T);          // words [T]
        L.off_pay = static_cast<uint32_t>(8ull * L.T);          // flat-map scratch (kk_fast.cu)
        L.bytes = 8ull * L.T + 640;
    }
    L.has_ids = false;
    L.has_pay = false;
    return L;
}

L2Spec plan_l2(int acc, int variant, int64_t s_true, int32_t domain, int64_t rows, const spg_config& cfg)
{
    L2Spec S;
    S.valid = true;
    const int32_t s = static_cast<int32_t>(std::max<int64_t>(std::min<int64_t>(s_true, std::max<int32_t>(domain, 1)), 1));
    S.lay = make_layout(acc, variant, s, domain, cfg.lp_max_occupancy, variant == kVarNumeric);
    S.chunk_bytes = align_up(S.lay.bytes, 256);
    if (static_cast<int64_t>(S.chunk_bytes) > cfg.pool_budget_bytes)
        fail(SPG_ERR_POOL_SIZING, "plan_pool: a single chunk exceeds the memory budget");
    const int64_t workers = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)sm_count() * 16));
    // memory_pool.cpp:83-109: one chunk per worker (one2one) or 2x (many2many),
    // halved while over the budget, falling back to many2many below the
    // worker count
    int64_t chunks = cfg.pool_mode == SPG_POOL_ONE2ONE ? workers : 2 * workers;
    S.pool_mode = cfg.pool_mode == SPG_POOL_ONE2ONE ? 0 : 1;
    while (chunks * static_cast<int64_t>(S.chunk_bytes) > cfg.pool_budget_bytes && chunks > 1)
        chunks = std::max<int64_t>(1, chunks / 2);
    if (chunks < workers)
        S.pool_mode = 1;
    S.num_chunks = static_cast<int32_t>(chunks);
    S.wpb = 8;
    const int64_t warps = S.pool_mode == 0 ? chunks : workers;
    S.grid = static_cast<int>((warps + S.wpb - 1) / S.wpb);
    return S;
}

// hist: bucket counts of the unclamped row bounds; umax: exact max bound.
// fast: L1 classes run the kk_fast.cu kernels; opt_div > 0 sizes their tables
// optimistically at 2*bound/opt_div keys (the reference's row-size estimate
// flops/collapse_divisor, engine.cpp:410-411, with 2x headroom).
PhasePlan plan_phase(int acc, bool flat, int variant, int32_t domain, const unsigned long long* hist,
                     int64_t umax, const spg_config& cfg, bool fast = false, int opt_div = 0,
                     bool short_rows = false, double avg_a_row = 0.0)
{
    PhasePlan P;
    P.acc = acc;
    P.flat = flat;
    P.short_rows = short_rows;
    P.fast = fast;
    P.variant = variant;
    P.domain = domain;
    std::fill(std::begin(P.bp.bucket_class), std::end(P.bp.bucket_class), int8_t(-1));
    const int dom_bucket = host_bucket(static_cast<unsigned long long>(std::max<int32_t>(domain, 0)));
    const int64_t l1cap = cfg.l1_capacity > 0 ? cfg.l1_capacity : INT64_MAX;
    auto layout_of = [&](int32_t c) {
        return fast ? make_layout_fast(variant, c, cfg.lp_max_occupancy)
                    : make_layout(acc, variant, c, domain, cfg.lp_max_occupancy, false);
    };

    // candidate L1 capacities (powers of two, the smallest covering 32 keys)
    std::vector<int32_t> caps;
    if (l1cap < 32) {
        int32_t c = 1;
        while (int64_t{c} * 2 <= l1cap)
            c *= 2;
        caps.push_back(c);
    } else {
        for (int32_t c = 32; int64_t{c} <= l1cap && c <= (1 << 20); c *= 2)
            caps.push_back(c);
    }
    std::vector<int32_t> l1caps;
    for (int32_t c : caps)
        if (layout_of(c).bytes <= kWarpSmemMax)
            l1caps.push_back(c);

    // bucket -> class: [l1caps..., L2, tiny]; rows whose bound (exact row size
    // for the numeric phase, flops / compressed flops for the symbolic one)
    // is at most kTinyKeys run a thread per row (kk_tiny.cu)
    // (only when A rows are short: a thread walks its A row's entries serially)
    const bool tiny_ok = fast && l1cap >= 32 && avg_a_row <= kTinyMaxAvgArow && getenv("KK_NO_TINY") == nullptr;
    const int tiny_c = static_cast<int>(l1caps.size()) + 1;
    std::vector<int64_t> cls_count(l1caps.size() + 2, 0);
    int8_t bc[64];
    for (int b = 0; b < 64; ++b) {
        bc[b] = -1;
        const int be = std::min(b, dom_bucket);
        if (be == 0)
            continue;
        int64_t need = std::min<int64_t>(int64_t{1} << (be - 1), std::max<int32_t>(domain, 1));
        if (tiny_ok && need <= (variant == kVarNumeric ? kTinyKeys : kTinySymKeys)) {
            bc[b] = static_cast<int8_t>(tiny_c);
            cls_count[tiny_c] += static_cast<int64_t>(hist[b]);
            continue;
        }
        if (fast && opt_div > 0) {
            const int64_t est = std::max<int64_t>(32, ceil_pow2_i((2 * need + opt_div - 1) / opt_div));
            if (est < need) {
                need = est;
                P.optimistic = true;
            }
        }
        int c = static_cast<int>(l1caps.size()); // L2
        for (size_t q = 0; q < l1caps.size(); ++q)
            if (l1caps[q] >= need) {
                c = static_cast<int>(q);
                break;
            }
        bc[b] = static_cast<int8_t>(c);
        cls_count[c] += static_cast<int64_t>(hist[b]);
    }
    // compact to non-empty classes
    std::vector<int> remap(cls_count.size(), -1);
    int64_t off = 0, l2_rows = 0;
    for (size_t c = 0; c < cls_count.size(); ++c) {
        if (cls_count[c] == 0)
            continue;
        PhaseClass pc;
        pc.count = cls_count[c];
        pc.off = off;
        off += pc.count;
        pc.l2 = c == l1caps.size();
        pc.tiny = static_cast<int>(c) == tiny_c;
        if (pc.tiny) {
            pc.fast = true;
        } else if (!pc.l2) {
            pc.fast = fast;
            pc.lay = layout_of(l1caps[c]);
            pc.wpb = static_cast<int>(std::clamp<uint64_t>(kCtaSmem / pc.lay.bytes, 1, 8));
            const uint64_t smem = pc.wpb * pc.lay.bytes;
            int per_sm;
            if (!fast)
                per_sm = row_kernel_max_blocks_per_sm(acc, flat, variant, false, pc.wpb, smem);
            else if (variant == kVarNumeric)
                per_sm = flat ? numeric_flat_fast_blocks_per_sm(pc.wpb, smem)
                              : numeric_fast_blocks_per_sm(pc.wpb, smem);
            else
                per_sm = symbolic_fast_blocks_per_sm(variant == kVarSymCompressed, short_rows, pc.wpb, smem);
            const int64_t want = (pc.count + pc.wpb - 1) / pc.wpb;
            pc.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sm_count())));
        } else {
            l2_rows = pc.count;
            P.l2_class = static_cast<int>(P.classes.size());
        }
        remap[c] = static_cast<int>(P.classes.size());
        P.classes.push_back(pc);
    }
    if (P.l2_class >= 0 || P.optimistic) {
        // the HBM path runs the generic kernels (LP when the L1 ran the fast ones)
        const int l2acc = fast ? kAccLP : acc;
        P.l2 = plan_l2(l2acc, variant, umax, domain, P.optimistic ? std::max<int64_t>(l2_rows, sm_count() * 16) : l2_rows, cfg);
        if (P.l2_class >= 0) {
            PhaseClass& pc = P.classes[P.l2_class];
            pc.lay = P.l2.lay;
            pc.wpb = P.l2.wpb;
            pc.grid = P.l2.grid;
        }
    }
    for (int b = 0; b < 64; ++b)
        P.bp.bucket_class[b] = bc[b] >= 0 ? static_cast<int8_t>(remap[bc[b]]) : int8_t(-1);
    for (size_t c = 0; c < P.classes.size() && c < 32; ++c)
        P.bp.class_off[c] = P.classes[c].off;
    P.need_list = P.classes.size() > 1;
    if (P.classes.size() > 32)
        fail(SPG_ERR_INTERNAL, "too many accumulator classes");
    return P;
}

struct DevPool {
    char* base = nullptr;
    int* states = nullptr;
    uint64_t bytes = 0;
    int32_t chunks = 0;
};

void ensure_pool(DevPool& pool, const L2Spec& P, cudaStream_t st)
{
    if (!P.valid)
        return;
    const uint64_t need = P.chunk_bytes * static_cast<uint64_t>(P.num_chunks);
    if (pool.base && pool.bytes >= need && pool.chunks >= P.num_chunks)
        return;
    if (pool.base) {
        cudaFreeAsync(pool.base, st);
        cudaFreeAsync(pool.states, st);
    }
    pool.base = dalloc<char>(need, st, "pool");
    pool.states = dalloc<int>(P.num_chunks, st, "pool states");
    pool.bytes = need;
    pool.chunks = P.num_chunks;
    // all maps start empty (-1) and rows hand their chunk back clean
    cuda_check(cudaMemsetAsync(pool.base, 0xFF, need, st), "pool init");
    cuda_check(cudaMemsetAsync(pool.states, 0, sizeof(int) * P.num_chunks, st), "pool states");
}

// Per-thread pinned scratch for the symbolic phase's small host reads.
// Pinned allocation and release synchronise the whole device (they would wait
// for unrelated copies on other streams, e.g. an overlapped upload), so the
// buffer is allocated once per thread and kept; it is portable (valid in every
// context), freed when the thread exits, and re-allocated if the runtime no
// longer recognises it (e.g. after a device reset).  spg_symbolic synchronises
// its stream before returning on every path, so no copy into the buffer is
// still in flight when the next call reuses it.
struct PinnedCache {
    void* buf = nullptr;
    size_t cap = 0;
    ~PinnedCache()
    {
        if (buf)
            cudaFreeHost(buf); // may fail harmlessly at process teardown
    }
    bool valid() const
    {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, buf) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost;
    }
};

struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t n)
    {
        thread_local PinnedCache c;
        if (c.cap < n || (c.buf && !c.valid())) {
            if (c.buf && c.valid())
                cudaFreeHost(c.buf);
            c.buf = nullptr;
            c.cap = 0;
            if (cudaHostAlloc(&c.buf, n, cudaHostAllocPortable) != cudaSuccess)
                fail(SPG_ERR_NOMEM, "pinned host buffer");
            c.cap = n;
        }
        p = c.buf;
    }
};

void validate_csr(const spg_csr* x, const char* name, bool need_vals)
{
    if (!x)
        fail(SPG_ERR_CONTRACT, std::string(name) + ": null matrix");
    if (x->num_rows < 0 || x->num_cols < 0 || x->nnz < 0)
        fail(SPG_ERR_CONTRACT, std::string(name) + ": negative dimensions");
    if (!x->row_offsets)
        fail(SPG_ERR_CONTRACT, std::string(name) + ": null row_offsets");
    if (x->nnz > 0 && !x->col_indices)
        fail(SPG_ERR_CONTRACT, std::string(name) + ": null col_indices");
    if (need_vals && x->nnz > 0 && !x->values)
        fail(SPG_ERR_CONTRACT, std::string(name) + ": null values");
}

const char* dev_error_text(int code)
{
    switch (code) {
    case kDevRowOverflow: return "numeric row exceeds the symbolic structure";
    case kDevRowShort: return "numeric row shorter than the symbolic structure";
    case kDevKeyRange: return "DenseAccumulator: key outside the column domain";
    case kDevL2Overflow: return "level-2 accumulator overflow: chunk bound violated";
    case kDevReplay: return "slot replay does not match the structure";
    case kDevUnsorted:
        return "B row not column-sorted: the column-slab plan of this handle needs sorted B rows (run symbolic on this B)";
    default: return "device error";
    }
}

} // namespace

// ---------------------------------------------------------------------------
// the handle
// ---------------------------------------------------------------------------
struct spg_handle {
    spg_handle_info info{};
    int64_t* d_rowptr = nullptr;
    int64_t* d_prf = nullptr;
    DevCounters* d_ctr = nullptr;
    ScanTotals size_hist{};     // host copy of the row-size histogram
    bool numeric_forced = false;
    PhasePlan num;
    int32_t* d_num_list = nullptr;
    int32_t* d_empty_list = nullptr; // rows of C the structure leaves empty (checked every pass)
    int64_t n_empty = 0;
    DevPool num_pool;
    cudaStream_t stream = nullptr;
    // heavy numeric rows (kk_heavy.cu): per-CTA staging for the bucket scatter
    bool num_heavy = false;
    bool num_slab = false;      // heavy rows by column slabs (kk_slab.cu) instead of buckets
    bool b_sorted = false;      // symbolic saw every referenced B row column-sorted
    int64_t max_a_row = 0;      // longest A row (slab cursors)
    SlabPlan slab;              // work items and per-warp cursor scratch
    int heavy_nb = 0;
    int64_t heavy_stage = 0; // staging products
    int64_t heavy_cap = 0;
    void* heavy_stage_buf = nullptr; // 16-byte {column, value} records
    // structure-reuse replay (kk_replay.cu): recorded on the second numeric
    // pass, replayed from the third while the structure fingerprints match
    int numeric_calls = 0;
    bool replay_eligible = false;
    bool replay_ready = false;
    int replay_width = 0;
    void* d_map = nullptr;
    int64_t* d_prod_off = nullptr;
    int32_t* d_ccache = nullptr;
    DevCounters* d_rctr = nullptr;
    unsigned long long* d_fp = nullptr; // [4]: A, B of the current pass; A, B recorded
    unsigned long long* h_fp = nullptr; // pinned [2 + DevCounters]

    void free_slab()
    {
        for (void* p : {static_cast<void*>(slab.items), slab.scratch, static_cast<void*>(slab.split_out),
                        static_cast<void*>(slab.split_done)})
            if (p)
                cudaFreeAsync(p, stream);
        slab = SlabPlan{};
    }

    void free_replay()
    {
        // device buffers are stream-ordered (cudaMallocAsync); the pinned
        // readback needs the stream drained first
        for (void* p : {d_map, static_cast<void*>(d_prod_off), static_cast<void*>(d_ccache),
                        static_cast<void*>(d_rctr), static_cast<void*>(d_fp)})
            if (p)
                cudaFreeAsync(p, stream);
        if (h_fp) {
            cudaStreamSynchronize(stream);
            cudaFreeHost(h_fp);
        }
        d_map = nullptr;
        d_prod_off = nullptr;
        d_ccache = nullptr;
        d_rctr = nullptr;
        d_fp = nullptr;
        h_fp = nullptr;
        replay_ready = false;
    }

    // Every device buffer comes from the stream-ordered allocator and is
    // released on the handle's stream: destroying a handle neither waits for
    // the device nor synchronises it (cudaFree would), so a NoReuse multiply
    // loop keeps the GPU busy across handles.
    ~spg_handle()
    {
        free_replay();
        free_slab();
        for (void* p : {heavy_stage_buf, static_cast<void*>(d_rowptr), static_cast<void*>(d_prf),
                        static_cast<void*>(d_ctr), static_cast<void*>(d_num_list),
                        static_cast<void*>(d_empty_list), static_cast<void*>(num_pool.base),
                        static_cast<void*>(num_pool.states)})
            if (p)
                cudaFreeAsync(p, stream);
    }
};

namespace {

// Work items of the column-slab kernel (one per heavy row, long rows cut into
// column parts) and the per-warp cursor scratch.  Needs the handle's A row
// offsets only through max_a_row and the items' part counts, which are a
// performance choice: any A of the handle's shape runs correctly.
void build_slab_plan(spg_handle* h, const int64_t* a_rowptr, cudaStream_t st);

void build_numeric_plan(spg_handle* h, cudaStream_t st, const int64_t* a_rowptr = nullptr)
{
    const spg_config& cfg = h->info.config;
    int acc;
    bool flat;
    const bool forced = h->numeric_forced || cfg.accumulator != SPG_ACC_AUTO;
    device_choice(forced, h->info.numeric_choice, cfg, h->info.flops.avg_row_flops, kVarNumeric, h->info.k,
                  h->info.max_row_size, &acc, &flat);
    bool fast = false;
    if (!forced) {
        // Auto on the GPU: the partitioning follows the average B-row length —
        // Thread-Sequential (one B row per step, warp lanes over its entries)
        // when rows fill a good part of the warp, Thread-Flat otherwise.
        const double avg_b = h->info.n > 0 ? static_cast<double>(h->info.nnz_b) / h->info.n : 0.0;
        if (cfg.l1_capacity <= 0) {
            acc = kAccLP;
            flat = avg_b < 12.0;
            fast = true;
        }
    } else if (acc == kAccLP && cfg.l1_capacity <= 0) {
        fast = true; // forced LP: same algorithms, fast kernels
    }
    h->num = plan_phase(acc, flat, kVarNumeric, h->info.k, h->size_hist.hist, h->info.max_row_size, cfg, fast, 0,
                        false, h->info.m > 0 ? static_cast<double>(h->info.nnz_a) / h->info.m : 0.0);
    // Auto: rows beyond the warp tables take the bucketed CTA path (kk_heavy.cu)
    // when a row's distinct columns fit the hashed buckets and its products
    // fit 32-bit staging offsets
    h->num_heavy = false;
    h->num_slab = false;
    h->free_slab();
    if (fast && !forced && h->num.l2_class >= 0 && h->b_sorted && h->max_a_row > 0) {
        // column slabs: no row-size limit, products read once (work items are
        // built below, once the heavy rows are listed largest first)
        h->num_heavy = true;
        h->num_slab = true;
    } else if (fast && !forced && h->num.l2_class >= 0) {
        const int64_t cap = std::max<int64_t>(h->info.flops.max_row_flops, 1);
        if (h->info.max_row_size <= kHeavyMaxRow && cap < (int64_t{1} << 31)) {
            h->num_heavy = true;
            h->heavy_nb = static_cast<int>(std::clamp<int64_t>(
                (h->info.max_row_size + kHeavyBucketKeys - 1) / kHeavyBucketKeys, 1, kHeavyMaxBuckets));
            h->heavy_cap = cap;
        }
    }
    // slot replay (kk_replay.cu) for the Auto Thread-Sequential plan when all
    // rows run in warp tables and slots fit two bytes
    h->free_replay();
    h->numeric_calls = 0;
    h->replay_eligible = fast && !forced && !flat && h->num.l2_class < 0 && !h->num_heavy && h->d_prf
        && h->info.nnz_c > 0 && h->info.flops.total_flops > 0 && h->info.max_row_size <= 2048
        && getenv("KK_NO_REPLAY") == nullptr;
    h->replay_width = h->info.max_row_size <= 256 ? 1 : 2;
    if (h->d_num_list) {
        cudaFreeAsync(h->d_num_list, st);
        h->d_num_list = nullptr;
    }
    if (h->d_empty_list) {
        cudaFreeAsync(h->d_empty_list, st);
        h->d_empty_list = nullptr;
    }
    h->n_empty = static_cast<int64_t>(h->size_hist.hist[0]);
    if (h->n_empty > 0) {
        h->d_empty_list = dalloc<int32_t>(h->n_empty, st, "empty row list");
        auto* cnt = dalloc<unsigned long long>(1, st, "count");
        cuda_check(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st), "memset");
        cuda_check(launch_collect_empty_rows(h->info.m, h->d_rowptr, h->d_empty_list, cnt, st), "empty rows");
        cudaFreeAsync(cnt, st);
    }
    if (h->num_heavy)
        h->num.need_list = true; // heavy rows are queued largest first
    if (h->num.need_list) {
        h->d_num_list = dalloc<int32_t>(std::max<int64_t>(h->info.m, 1), st, "numeric row list");
        auto* fill = dalloc<unsigned long long>(32, st, "fill");
        cuda_check(cudaMemsetAsync(fill, 0, 32 * sizeof(unsigned long long), st), "fill");
        cuda_check(launch_bin_scatter(h->info.m, nullptr, h->d_rowptr, INT64_MAX, h->num.bp, fill,
                                      h->d_num_list, st),
                   "numeric binning");
        cudaFreeAsync(fill, st);
        if (h->num_heavy && h->d_prf) {
            const PhaseClass& hc = h->num.classes[h->num.l2_class];
            cuda_check(sort_rows_by_flops_desc(h->d_num_list + hc.off, hc.count, h->d_prf, st), "heavy row order");
        }
    }
    if (h->num_slab && a_rowptr)
        build_slab_plan(h, a_rowptr, st); // else at the first numeric call (its A)
}

void build_slab_plan(spg_handle* h, const int64_t* a_rowptr, cudaStream_t st)
{
    const PhaseClass& hc = h->num.classes[h->num.l2_class];
    SlabPlan& P = h->slab;
    P.max_a_row = (h->max_a_row + 3) / 4 * 4; // keeps every warp's int64 cursor arrays 8-byte aligned
    int64_t* off = dalloc<int64_t>(hc.count + 1, st, "slab item offsets");
    cuda_check(build_slab_items(h->d_num_list + hc.off, hc.count, a_rowptr, h->d_rowptr, h->info.k, off, nullptr,
                                nullptr, st),
               "slab parts");
    int64_t n_items = 0;
    cuda_check(cudaMemcpyAsync(&n_items, off + hc.count, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "items");
    cuda_check(cudaStreamSynchronize(st), "slab plan sync");
    P.n_items = n_items;
    P.items = dalloc<int4>(std::max<int64_t>(n_items, 1), st, "slab items");
    auto* nsplit = dalloc<unsigned long long>(1, st, "split count");
    cuda_check(cudaMemsetAsync(nsplit, 0, sizeof(unsigned long long), st), "memset");
    cuda_check(build_slab_items(h->d_num_list + hc.off, hc.count, a_rowptr, h->d_rowptr, h->info.k, off, P.items,
                                nsplit, st),
               "slab items");
    unsigned long long n_split = 0;
    cuda_check(cudaMemcpyAsync(&n_split, nsplit, sizeof(n_split), cudaMemcpyDeviceToHost, st), "split count");
    cuda_check(cudaStreamSynchronize(st), "slab plan sync");
    cudaFreeAsync(off, st);
    cudaFreeAsync(nsplit, st);
    P.n_split = static_cast<int64_t>(n_split);
    if (P.n_split > 0) {
        P.split_out = dalloc<unsigned long long>(P.n_split, st, "split rows");
        P.split_done = dalloc<unsigned int>(P.n_split, st, "split rows");
    }
    // resident warps, bounded so the cursor scratch takes at most a quarter of
    // the free memory
    const int per_cta = slab_warps_per_cta();
    int64_t warps = numeric_slab_warps();
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t per_warp = static_cast<size_t>(std::max<int64_t>(P.max_a_row, 1)) * slab_scratch_per_entry();
    const int64_t by_mem = static_cast<int64_t>(free_b / 4 / per_warp) / per_cta * per_cta;
    warps = std::max<int64_t>(per_cta, std::min(warps, by_mem));
    P.warps = warps;
    P.scratch = dalloc<unsigned char>(static_cast<size_t>(warps) * per_warp, st, "slab cursors");
}

ReplayLaunch replay_launch(spg_handle* h, const spg_csr* a, const spg_csr* b, int32_t* c_cols, double* c_vals)
{
    ReplayLaunch R{};
    R.a_rowptr = a->row_offsets;
    R.a_cols = a->col_indices;
    R.a_vals = a->values;
    R.b_rowptr = b->row_offsets;
    R.b_cols = b->col_indices;
    R.b_vals = b->values;
    R.c_rowptr = h->d_rowptr;
    R.c_cols = c_cols;
    R.c_vals = c_vals;
    R.ccache = h->d_ccache;
    R.map = h->d_map;
    R.prod_off = h->d_prod_off;
    R.m = h->info.m;
    R.row_lo = 0;
    R.row_hi = h->info.m;
    R.ctr = h->d_ctr;
    return R;
}

// fingerprints of A's and B's structure into h->d_fp[0..1] (stream-ordered;
// one pass when A and B are the same arrays)
void replay_fingerprints(spg_handle* h, const spg_csr* a, const spg_csr* b, cudaStream_t st)
{
    cuda_check(cudaMemsetAsync(h->d_fp, 0, 2 * sizeof(unsigned long long), st), "memset");
    const bool same = a->row_offsets == b->row_offsets && a->col_indices == b->col_indices
        && a->num_rows == b->num_rows;
    cuda_check(launch_fingerprint(a->num_rows, a->row_offsets, a->col_indices, h->d_fp, same ? h->d_fp + 1 : nullptr,
                                  st),
               "fingerprint");
    if (!same)
        cuda_check(launch_fingerprint(b->num_rows, b->row_offsets, b->col_indices, h->d_fp + 1, nullptr, st),
                   "fingerprint");
}

// record the slot map of this pass's (first-touch ordered) output; any
// failure leaves the handle on the hashing kernels
void record_replay(spg_handle* h, const spg_csr* a, const spg_csr* b, int32_t* c_cols, double* c_vals,
                   cudaStream_t st)
{
    const spg_handle_info& I = h->info;
    const uint64_t map_bytes = static_cast<uint64_t>(I.flops.total_flops) * h->replay_width;
    const uint64_t need = map_bytes + 4ull * I.nnz_c + 8ull * (int64_t{I.m} + 1);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (need > free_b / 2) {
        h->replay_eligible = false;
        return;
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, map_bytes, st) != cudaSuccess) {
        cudaGetLastError();
        h->replay_eligible = false;
        return;
    }
    h->d_map = p;
    h->d_ccache = dalloc<int32_t>(I.nnz_c, st, "replay column cache");
    h->d_prod_off = dalloc<int64_t>(int64_t{I.m} + 1, st, "replay product offsets");
    h->d_rctr = dalloc<DevCounters>(1, st, "replay counters");
    h->d_fp = dalloc<unsigned long long>(4, st, "fingerprints");
    if (cudaMallocHost(&p, 2 * sizeof(unsigned long long) + sizeof(DevCounters)) != cudaSuccess)
        fail(SPG_ERR_NOMEM, "pinned host buffer");
    h->h_fp = static_cast<unsigned long long*>(p);
    ScanTotals* d_stot = dalloc<ScanTotals>(1, st, "scan totals");
    cuda_check(cudaMemsetAsync(d_stot, 0, sizeof(ScanTotals), st), "memset");
    cuda_check(cudaMemsetAsync(h->d_prod_off, 0, sizeof(int64_t), st), "memset");
    cuda_check(cudaMemsetAsync(h->d_rctr, 0, sizeof(DevCounters), st), "memset");
    cuda_check(cudaMemcpyAsync(h->d_prod_off + 1, h->d_prf, sizeof(int64_t) * I.m, cudaMemcpyDeviceToDevice, st),
               "product offsets");
    cuda_check(scan_sizes_inplace(h->d_prod_off, I.m, d_stot, st), "product offsets");
    cudaFreeAsync(d_stot, st);
    ReplayLaunch R = replay_launch(h, a, b, c_cols, c_vals);
    R.ctr = h->d_rctr;
    R.T = static_cast<int32_t>(std::max<int64_t>(64, ceil_pow2_i(2 * I.max_row_size)));
    R.shift = 32 - log2_i(R.T);
    cuda_check(launch_replay_build(R, h->replay_width, st), "replay build");
    auto* hc = reinterpret_cast<DevCounters*>(h->h_fp + 2);
    cuda_check(cudaMemcpyAsync(hc, h->d_rctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st), "counters");
    // the recorded structure's fingerprints become the expected ones (d_fp[2..3])
    replay_fingerprints(h, a, b, st);
    cuda_check(cudaMemcpyAsync(h->d_fp + 2, h->d_fp, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st),
               "fingerprint");
    cuda_check(cudaStreamSynchronize(st), "replay record sync");
    if (hc->error) {
        h->free_replay();
        h->replay_eligible = false;
        return;
    }
    h->replay_ready = true;
}


} // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* spg_last_error(void) { return g_err.c_str(); }

int64_t spg_kernel_launch_count(void) { return kk::launch_count(); }

int spg_config_init(spg_config* c)
{
    if (!c)
        return SPG_ERR_CONTRACT;
    // engine.hpp:18-31, memory_pool.hpp:88
    c->scheme = SPG_SCHEME_SEQUENTIAL;
    c->accumulator = SPG_ACC_AUTO;
    c->l1_capacity = 0;
    c->dense_cutoff_k = 250000;
    c->avg_flops_cutoff = 256.0;
    c->lp_max_occupancy = 0.5;
    c->compression_gate = 0.15;
    c->compression = SPG_COMPRESSION_AUTO;
    c->collapse_divisor = 8;
    c->worker_count = 1;
    c->sort_output = 0;
    c->row_block = 512;
    c->pool_mode = SPG_POOL_ONE2ONE;
    c->pool_budget_bytes = int64_t{1} << 30;
    return SPG_OK;
}

int spg_resolve_config(int32_t phase, int32_t k, const spg_flops_stats* stats,
                       const spg_compression_report* report, const spg_config* cfg,
                       int64_t row_upper_bound, spg_resolved* out)
{
    return guarded([&] {
        if (!stats || !report || !cfg || !out)
            fail(SPG_ERR_CONTRACT, "resolve_config: null argument");
        // engine.cpp:367-395
        spg_resolved rc{};
        const bool compressed = phase == SPG_PHASE_SYMBOLIC && report->applied;
        rc.effective_k = compressed ? static_cast<int32_t>((int64_t{k} + 31) / 32) : k;
        if (cfg->accumulator != SPG_ACC_AUTO) {
            rc.accumulator = cfg->accumulator;
            rc.scheme = cfg->scheme;
        } else if (rc.effective_k < cfg->dense_cutoff_k) {
            rc.accumulator = SPG_ACC_DENSE;
            rc.scheme = cfg->scheme;
        } else if (stats->avg_row_flops < cfg->avg_flops_cutoff) {
            rc.accumulator = SPG_ACC_LL;
            rc.scheme = cfg->scheme;
        } else {
            rc.accumulator = SPG_ACC_LP;
            rc.scheme = SPG_SCHEME_FLAT_PARALLEL;
        }
        const int64_t bound = std::max<int64_t>(std::min<int64_t>(row_upper_bound, rc.effective_k), 1);
        rc.l2_capacity = static_cast<int32_t>(bound);
        rc.l1_capacity = cfg->l1_capacity > 0 ? cfg->l1_capacity : rc.l2_capacity;
        *out = rc;
    });
}

int spg_flat_position(const int64_t* prefix, int64_t len, int64_t t, int32_t* seg, int64_t* off)
{
    return guarded([&] {
        if (!prefix || len < 1 || !seg || !off)
            fail(SPG_ERR_CONTRACT, "flat_position: bad argument");
        // engine.cpp:360-365: seg = upper_bound(prefix, t) - 1
        const int64_t* it = std::upper_bound(prefix, prefix + len, t);
        const int64_t s = (it - prefix) - 1;
        *seg = static_cast<int32_t>(s);
        *off = t - prefix[s];
    });
}

int spg_symbolic(const spg_csr* a, const spg_csr* b, const spg_config* cfg_in, spg_handle_t* out,
                 void* stream)
{
    spg_handle* h = nullptr;
    const int rc = guarded([&] {
        if (!out)
            fail(SPG_ERR_CONTRACT, "symbolic: null output handle");
        *out = nullptr;
        validate_csr(a, "symbolic: A", false);
        validate_csr(b, "symbolic: B", false);
        if (a->num_cols != b->num_rows)
            fail(SPG_ERR_CONTRACT, "symbolic: inner dimensions do not match"); // engine.cpp:399-400
        require_device();
        spg_config cfg;
        if (cfg_in)
            cfg = *cfg_in;
        else
            spg_config_init(&cfg);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        h = new spg_handle;
        h->stream = st;
        spg_handle_info& I = h->info;
        I.config = cfg;
        I.m = a->num_rows;
        I.n = a->num_cols;
        I.k = b->num_cols;
        I.nnz_a = a->nnz;
        I.nnz_b = b->nnz;
        const int32_t m = I.m, n = I.n, k = I.k;

        cudaEvent_t ev[3];
        for (auto& e : ev)
            cuda_check(cudaEventCreate(&e), "event");
        struct EvGuard {
            cudaEvent_t* e;
            ~EvGuard()
            {
                for (int q = 0; q < 3; ++q)
                    cudaEventDestroy(e[q]);
            }
        } evg{ev};

        h->d_rowptr = dalloc<int64_t>(int64_t{m} + 1, st, "C row offsets");
        h->d_prf = dalloc<int64_t>(std::max(m, 1), st, "per-row flops");
        h->d_ctr = dalloc<DevCounters>(1, st, "counters");
        I.d_c_row_offsets = h->d_rowptr;
        I.d_per_row_flops = h->d_prf;
        int64_t* d_prcf = dalloc<int64_t>(std::max(m, 1), st, "per-row cflops");
        int32_t* d_csize = dalloc<int32_t>(std::max(n, 1), st, "csize");
        // B slots hold the compressed pairs; index them like B (base-relative)
        int2* d_cp_alloc = dalloc<int2>(std::max<int64_t>(b->nnz, 1), st, "compressed pairs");
        Totals* d_tot = dalloc<Totals>(1, st, "totals");
        ScanTotals* d_stot = dalloc<ScanTotals>(1, st, "scan totals");

        PinnedBuf pin(sizeof(Totals) + sizeof(ScanTotals) + sizeof(DevCounters) + 64 + 16);
        auto* htot = static_cast<Totals*>(pin.p);
        auto* hstot = reinterpret_cast<ScanTotals*>(htot + 1);
        auto* hctr = reinterpret_cast<DevCounters*>(hstot + 1);
        auto* hviews = reinterpret_cast<int64_t*>(hctr + 1);

        // the view offsets are read back with the flop totals (one host round
        // trip): the kernels rebase the compressed pairs on B's first offset
        // themselves, and compress only the band of B rows a row shard of A
        // references (A at most half as tall as B) from a device-side range
        cuda_check(cudaMemcpyAsync(hviews + 0, a->row_offsets, 8, cudaMemcpyDeviceToHost, st), "A view");
        cuda_check(cudaMemcpyAsync(hviews + 1, a->row_offsets + m, 8, cudaMemcpyDeviceToHost, st), "A view");
        cuda_check(cudaMemcpyAsync(hviews + 2, b->row_offsets, 8, cudaMemcpyDeviceToHost, st), "B view");
        cuda_check(cudaMemcpyAsync(hviews + 3, b->row_offsets + n, 8, cudaMemcpyDeviceToHost, st), "B view");
        int* d_crange = nullptr;
        if (int64_t{m} * 2 <= n) {
            d_crange = dalloc<int>(2, st, "column range");
            cuda_check(launch_col_range(m, a->row_offsets, a->col_indices, d_crange, st), "column range");
        }
        cuda_check(cudaEventRecord(ev[0], st), "event");
        cuda_check(cudaMemsetAsync(d_tot, 0, sizeof(Totals), st), "memset");
        cuda_check(cudaMemsetAsync(d_stot, 0, sizeof(ScanTotals), st), "memset");
        cuda_check(cudaMemsetAsync(h->d_ctr, 0, sizeof(DevCounters), st), "memset");
        int2* d_cp = d_cp_alloc; // rebased on the device (cpair_of)

        // ---- K3 + K1/K4 ----
        cuda_check(launch_compress(n, b->row_offsets, b->col_indices, d_csize, d_cp_alloc, &d_tot->nnz_bc,
                                   &d_tot->unsorted, d_crange, st),
                   "compress");
        if (d_crange)
            cudaFreeAsync(d_crange, st);
        const double avg_len = m > 0 ? static_cast<double>(a->nnz) / m : 0.0;
        cuda_check(launch_flops(m, avg_len, a->row_offsets, a->col_indices, b->row_offsets, d_csize,
                                h->d_prf, d_prcf, d_tot, st),
                   "flops");
        cuda_check(cudaMemcpyAsync(htot, d_tot, sizeof(Totals), cudaMemcpyDeviceToHost, st), "totals");
        cuda_check(cudaEventRecord(ev[1], st), "event");
        cuda_check(cudaStreamSynchronize(st), "flops sync");
        if (hviews[1] - hviews[0] != a->nnz || hviews[3] - hviews[2] != b->nnz)
            fail(SPG_ERR_CONTRACT, "symbolic: nnz does not match row_offsets");
        h->max_a_row = static_cast<int64_t>(htot->max_alen);
        h->b_sorted = htot->unsorted == 0;

        // ---- host decisions (engine.cpp:409-423, compression.cpp:118-147) ----
        I.flops.total_flops = static_cast<int64_t>(htot->total_f);
        I.flops.max_row_flops = static_cast<int64_t>(htot->max_f);
        I.flops.avg_degree_a = a->num_cols > 0 ? static_cast<double>(a->nnz) / a->num_cols : 0.0;
        I.flops.avg_row_flops = m > 0 ? static_cast<double>(I.flops.total_flops) / m : 0.0;
        I.avg_row_size_estimate = I.flops.avg_row_flops / std::max(cfg.collapse_divisor, 1);
        spg_compression_report& R = I.compression;
        R.compressed_flops = static_cast<int64_t>(htot->total_cf);
        I.compressed_nnz_b = static_cast<int64_t>(htot->nnz_bc);
        R.compressed_max_row_flops = static_cast<int64_t>(htot->max_cf);
        R.cf = I.flops.total_flops > 0 ? static_cast<double>(R.compressed_flops) / I.flops.total_flops : 1.0;
        R.cmrf = I.flops.max_row_flops > 0
            ? static_cast<double>(R.compressed_max_row_flops) / I.flops.max_row_flops
            : 1.0;
        bool apply = false;
        if (cfg.compression == SPG_COMPRESSION_ALWAYS)
            apply = true;
        else if (cfg.compression == SPG_COMPRESSION_NEVER)
            apply = false;
        else {
            const int64_t threshold_ppm =
                std::llround((1.0 - std::clamp(cfg.compression_gate, 0.0, 1.0)) * 1000000.0);
            apply = I.flops.total_flops > 0
                && R.compressed_flops * 1000000 < I.flops.total_flops * threshold_ppm;
        }
        R.applied = apply ? 1 : 0;
        const int64_t raw_bound = apply ? R.compressed_max_row_flops : I.flops.max_row_flops;
        cuda_check(spg_resolve_config(SPG_PHASE_SYMBOLIC, k, &I.flops, &R, &cfg, raw_bound, &I.symbolic_choice) == SPG_OK
                       ? cudaSuccess
                       : cudaErrorInvalidValue,
                   "resolve_config");
        check_pool_budget(I.symbolic_choice, cfg.pool_budget_bytes);
        const int32_t sym_l1_keys = ref_l1_keys(I.symbolic_choice, cfg.lp_max_occupancy);

        // ---- K5: symbolic union ----
        const int variant = apply ? kVarSymCompressed : kVarSymRaw;
        const int32_t domain = I.symbolic_choice.effective_k;
        int sacc;
        bool sflat;
        device_choice(cfg.accumulator != SPG_ACC_AUTO, I.symbolic_choice, cfg, I.flops.avg_row_flops, variant,
                      domain, raw_bound, &sacc, &sflat);
        // Auto: the order-free fast union with optimistic L1 sizing (kk_fast.cu)
        const bool sfast = cfg.accumulator == SPG_ACC_AUTO && cfg.l1_capacity <= 0;
        // short rows (the paper's kkmem side of the avg-row-flops cutoff):
        // latency-bound, so the fast kernel pipelines rows
        const bool short_rows = I.flops.avg_row_flops < cfg.avg_flops_cutoff;
        const PhasePlan S = plan_phase(sfast ? kAccLP : sacc, sfast ? true : sflat, variant, domain,
                                       apply ? htot->hist_cf : htot->hist_f, raw_bound, cfg, sfast,
                                       sfast ? std::max(cfg.collapse_divisor, 1) : 0, short_rows,
                                       m > 0 ? static_cast<double>(I.nnz_a) / m : 0.0);
        cuda_check(cudaMemsetAsync(h->d_rowptr, 0, sizeof(int64_t) * (int64_t{m} + 1), st), "memset");
        int32_t* d_list = nullptr;
        if (S.need_list) {
            d_list = dalloc<int32_t>(std::max(m, 1), st, "symbolic row list");
            auto* fill = dalloc<unsigned long long>(32, st, "fill");
            cuda_check(cudaMemsetAsync(fill, 0, 32 * sizeof(unsigned long long), st), "fill");
            cuda_check(launch_bin_scatter(m, apply ? d_prcf : h->d_prf, nullptr, domain, S.bp, fill, d_list, st),
                       "symbolic binning");
            cudaFreeAsync(fill, st);
        }
        unsigned long long* d_retry_cnt = nullptr;
        int32_t* d_retry = nullptr;
        if (S.optimistic) {
            d_retry_cnt = dalloc<unsigned long long>(1, st, "retry count");
            d_retry = dalloc<int32_t>(std::max(m, 1), st, "retry rows");
            cuda_check(cudaMemsetAsync(d_retry_cnt, 0, sizeof(unsigned long long), st), "memset");
        }
        DevPool spool;
        // Auto: heavy rows use the CTA dense-bitmap kernel when the column
        // domain (in 32-bit words) fits shared memory
        const int32_t dom_words = static_cast<int32_t>((int64_t{k} + 31) / 32);
        // (domains wider than the bitmap are walked in ranges of kHeavySymWords words)
        const int32_t heavy_words = sfast ? std::max(std::min(dom_words, kHeavySymWords), 1) : 0;
        auto sym_launch = [&](const PhaseClass& pc, const int32_t* list, int64_t nrows) {
            RowLaunch L{};
            L.a_rowptr = a->row_offsets;
            L.a_cols = a->col_indices;
            L.a_vals = nullptr;
            L.b_rowptr = b->row_offsets;
            L.b_cols = b->col_indices;
            L.csize = d_csize;
            L.cpair = d_cp;
            L.list = list;
            L.nrows = nrows;
            L.sym_sizes = h->d_rowptr + 1;
            L.ctr = h->d_ctr;
            L.l1_keys = sym_l1_keys;
            L.lay = pc.lay;
            L.wpb = pc.wpb;
            L.grid = pc.grid;
            L.l2 = pc.l2;
            if (pc.l2 && heavy_words > 0) {
                // heavy rows: CTA-wide dense bitmap over the column domain
                const int grid = static_cast<int>(std::min<int64_t>(nrows, sm_count()));
                cuda_check(launch_symbolic_heavy(L, S.variant == kVarSymCompressed, heavy_words, std::max(dom_words, 1), grid, st),
                           "symbolic heavy kernel");
            } else if (pc.l2) {
                ensure_pool(spool, S.l2, st);
                L.pool = PoolDesc{spool.base, S.l2.chunk_bytes, S.l2.num_chunks, S.l2.pool_mode, spool.states};
                cuda_check(launch_row_kernel(L, S.fast ? kAccLP : S.acc, S.fast ? false : S.flat, S.variant, st),
                           "symbolic L2 kernel");
            } else if (pc.tiny) {
                cuda_check(launch_symbolic_tiny(L, S.variant == kVarSymCompressed, d_retry_cnt, d_retry, st),
                           "symbolic tiny kernel");
            } else if (pc.fast) {
                cuda_check(launch_symbolic_fast(L, S.variant == kVarSymCompressed, S.short_rows, d_retry_cnt, d_retry, st),
                           "symbolic kernel");
            } else {
                cuda_check(launch_row_kernel(L, S.acc, S.flat, S.variant, st), "symbolic kernel");
            }
        };
        for (const PhaseClass& pc : S.classes)
            sym_launch(pc, S.need_list ? d_list + pc.off : nullptr, S.need_list ? pc.count : m);
        if (S.optimistic && heavy_words > 0) {
            // rows whose optimistic L1 table overflowed: the CTA bitmap kernel,
            // its row count read on the device (no host round trip)
            RowLaunch L{};
            L.a_rowptr = a->row_offsets;
            L.a_cols = a->col_indices;
            L.b_rowptr = b->row_offsets;
            L.b_cols = b->col_indices;
            L.csize = d_csize;
            L.cpair = d_cp;
            L.list = d_retry;
            L.nrows = m;             // upper bound; the kernel stops at *d_nrows
            L.d_nrows = d_retry_cnt;
            L.sym_sizes = h->d_rowptr + 1;
            L.ctr = h->d_ctr;
            L.l1_keys = sym_l1_keys;
            cuda_check(launch_symbolic_heavy(L, S.variant == kVarSymCompressed, heavy_words, std::max(dom_words, 1),
                                             sm_count(), st),
                       "symbolic heavy kernel (retries)");
            cudaFreeAsync(d_retry_cnt, st);
            cudaFreeAsync(d_retry, st);
        } else if (S.optimistic) {
            // rows whose optimistic L1 table overflowed: exact-size HBM tables
            unsigned long long* hretry = reinterpret_cast<unsigned long long*>(hviews + 5);
            cuda_check(cudaMemcpyAsync(hretry, d_retry_cnt, 8, cudaMemcpyDeviceToHost, st), "retry count");
            cuda_check(cudaStreamSynchronize(st), "retry sync");
            if (*hretry > 0) {
                PhaseClass rc;
                rc.l2 = true;
                rc.lay = S.l2.lay;
                rc.wpb = S.l2.wpb;
                rc.grid = S.l2.grid;
                sym_launch(rc, d_retry, static_cast<int64_t>(*hretry));
            }
            cudaFreeAsync(d_retry_cnt, st);
            cudaFreeAsync(d_retry, st);
        }
        // ---- K2: scan ----
        cuda_check(scan_sizes_inplace(h->d_rowptr, m, d_stot, st), "scan");
        cuda_check(cudaMemcpyAsync(hstot, d_stot, sizeof(ScanTotals), cudaMemcpyDeviceToHost, st), "scan totals");
        cuda_check(cudaMemcpyAsync(hctr, h->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st), "counters");
        int64_t* hnnz = hviews + 4;
        cuda_check(cudaMemcpyAsync(hnnz, h->d_rowptr + m, 8, cudaMemcpyDeviceToHost, st), "nnz");
        cuda_check(cudaEventRecord(ev[2], st), "event");
        if (d_list)
            cudaFreeAsync(d_list, st);
        cudaFreeAsync(d_prcf, st);
        cudaFreeAsync(d_csize, st);
        cudaFreeAsync(d_cp_alloc, st);
        cudaFreeAsync(d_tot, st);
        cudaFreeAsync(d_stot, st);
        if (spool.base) {
            cudaFreeAsync(spool.base, st);
            cudaFreeAsync(spool.states, st);
        }
        cuda_check(cudaStreamSynchronize(st), "symbolic sync");
        if (hctr->error)
            fail(SPG_ERR_INTERNAL, std::string("symbolic: ") + dev_error_text(hctr->error));

        I.nnz_c = *hnnz;
        I.max_row_size = static_cast<int64_t>(hstot->max_size);
        I.avg_row_size = m > 0 ? static_cast<double>(I.nnz_c) / m : 0.0;
        h->size_hist = *hstot;
        float ms01 = 0.f, ms12 = 0.f;
        cudaEventElapsedTime(&ms01, ev[0], ev[1]);
        cudaEventElapsedTime(&ms12, ev[1], ev[2]);
        I.compress_ms = ms01;
        I.symbolic_stats.ms = ms12;
        I.symbolic_stats.pool_allocations = static_cast<int64_t>(hctr->pool_allocations);
        I.symbolic_stats.l2_inserts = static_cast<int64_t>(hctr->l2_inserts);
        spg_resolve_config(SPG_PHASE_NUMERIC, k, &I.flops, &R, &cfg, I.max_row_size, &I.numeric_choice);
        build_numeric_plan(h, st, a->row_offsets);
        *out = h;
    });
    if (rc != SPG_OK) {
        // copies into the per-thread pinned scratch may still be in flight
        cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        cudaGetLastError();
        delete h;
        if (out)
            *out = nullptr;
    }
    return rc;
}

static int numeric_impl(spg_handle_t h, const spg_csr* a, const spg_csr* b, int32_t row_lo, int32_t row_hi,
                        int32_t* c_cols, double* c_vals, spg_phase_stats* stats, void* stream)
{
    return guarded([&] {
        if (!h)
            fail(SPG_ERR_CONTRACT, "numeric: null handle");
        validate_csr(a, "numeric: A", true);
        validate_csr(b, "numeric: B", true);
        const spg_handle_info& I = h->info;
        // engine.cpp:451-453
        if (a->num_rows != I.m || a->num_cols != I.n || b->num_rows != I.n || b->num_cols != I.k
            || a->nnz != I.nnz_a || b->nnz != I.nnz_b)
            fail(SPG_ERR_REUSE, "numeric: operands do not match the symbolic handle");
        if (I.nnz_c > 0 && (!c_cols || !c_vals))
            fail(SPG_ERR_CONTRACT, "numeric: null output buffers");
        if (row_lo < 0 || row_hi > I.m || row_lo > row_hi)
            fail(SPG_ERR_CONTRACT, "numeric: bad row range");
        const bool full = row_lo == 0 && row_hi == I.m;
        check_pool_budget(I.numeric_choice, I.config.pool_budget_bytes); // raised by numeric (run_phase)
        const int32_t num_l1_keys = ref_l1_keys(I.numeric_choice, I.config.lp_max_occupancy);
        require_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        h->stream = st;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (stats) {
            cuda_check(cudaEventCreate(&e0), "event");
            cuda_check(cudaEventCreate(&e1), "event");
            cuda_check(cudaEventRecord(e0, st), "event");
        }
        // per-call counters and queue heads restart every call; the error word
        // restarts only with a pass that begins at row 0, so a caller running
        // a pass as row blocks (host.multiply_host) sees an error raised by
        // any block when it checks after the last one
        if (row_lo == 0) {
            cuda_check(cudaMemsetAsync(h->d_ctr, 0, sizeof(DevCounters), st), "memset");
        } else {
            cuda_check(cudaMemsetAsync(h->d_ctr, 0, offsetof(DevCounters, error), st), "memset");
            cuda_check(cudaMemsetAsync(&h->d_ctr->next_row, 0, sizeof(h->d_ctr->next_row), st), "memset");
        }
        const PhasePlan& P = h->num;
        if (full)
            ++h->numeric_calls;
        bool replayed = false;
        const unsigned long long* gate = nullptr;
        if (h->replay_ready) {
            // both paths are launched; each reads the fingerprints and exactly
            // one of them does the work (no host round trip)
            replay_fingerprints(h, a, b, st);
            gate = h->d_fp;
            ReplayLaunch R = replay_launch(h, a, b, c_cols, c_vals);
            R.row_lo = row_lo;
            R.row_hi = row_hi;
            R.gate = gate;
            cuda_check(launch_replay_numeric(R, h->replay_width, static_cast<int32_t>(I.max_row_size), st),
                       "replay numeric");
            replayed = true;
        }
        if (h->num_slab && !h->slab.items)
            build_slab_plan(h, a->row_offsets, st); // handle re-planned without A (set_numeric)
        if (h->n_empty > 0 && row_hi > row_lo)
            cuda_check(launch_check_empty_rows(h->d_empty_list, h->n_empty, a->row_offsets, a->col_indices,
                                               b->row_offsets, full ? 0 : row_lo, full ? 0 : row_hi, h->d_ctr, st),
                       "empty rows check");
        if (!replayed && P.l2_class >= 0 && !h->num_heavy)
            ensure_pool(h->num_pool, P.l2, st);
        for (const PhaseClass& pc : P.classes) {
            RowLaunch L{};
            L.a_rowptr = a->row_offsets;
            L.a_cols = a->col_indices;
            L.a_vals = a->values;
            L.b_rowptr = b->row_offsets;
            L.b_cols = b->col_indices;
            L.b_vals = b->values;
            L.list = P.need_list ? h->d_num_list + pc.off : nullptr;
            L.nrows = P.need_list ? pc.count : I.m;
            L.row_lo = full ? 0 : row_lo;
            L.row_hi = full ? 0 : row_hi;
            L.gate = gate;
            if (!full && row_lo == row_hi)
                break;
            L.c_rowptr = h->d_rowptr;
            L.c_cols = c_cols;
            L.c_vals = c_vals;
            L.ctr = h->d_ctr;
            L.l1_keys = num_l1_keys;
            L.lay = pc.lay;
            L.wpb = pc.wpb;
            L.grid = pc.grid;
            L.l2 = pc.l2;
            if (pc.l2 && h->num_slab) {
                cuda_check(launch_numeric_slab(L, h->slab, I.k, h->d_prf, st), "numeric slab kernel");
            } else if (pc.l2 && h->num_heavy) {
                const int64_t resident = int64_t{numeric_heavy_blocks_per_sm(h->heavy_nb)} * sm_count();
                const int64_t want = std::max<int64_t>(1, std::min<int64_t>(resident, pc.count));
                if (!h->heavy_stage_buf) {
                    // staging for the bucket scatter (16 B per product), shared by
                    // the two size classes of heavy rows below: what every
                    // resident CTA needs for the largest row, or half the free
                    // memory, whichever is smaller (at least one largest row)
                    size_t free_b = 0, total_b = 0;
                    cudaMemGetInfo(&free_b, &total_b);
                    const int64_t by_mem = static_cast<int64_t>(free_b / 2 / 16);
                    h->heavy_stage = std::max<int64_t>(std::min<int64_t>(by_mem, h->heavy_cap * want), h->heavy_cap);
                    h->heavy_stage_buf = dalloc<double>(2 * static_cast<size_t>(h->heavy_stage), st, "heavy staging");
                }
                // rows whose products fit an equal share of the staging run on
                // every resident CTA; the largest rows then run with one
                // largest-row stage per CTA
                const int64_t small_cap = std::min<int64_t>(h->heavy_cap, h->heavy_stage / want);
                cuda_check(launch_numeric_heavy(L, h->heavy_stage_buf, small_cap, kHeavyBucketKeys,
                                                h->heavy_nb, -1, small_cap, 0, static_cast<int>(want), st),
                           "numeric heavy kernel");
                if (small_cap < h->heavy_cap) {
                    const int64_t g = std::max<int64_t>(1, std::min<int64_t>(h->heavy_stage / h->heavy_cap, want));
                    cuda_check(launch_numeric_heavy(L, h->heavy_stage_buf, h->heavy_cap, kHeavyBucketKeys,
                                                    h->heavy_nb, small_cap, INT64_MAX, 1, static_cast<int>(g), st),
                               "numeric heavy kernel (largest rows)");
                }
            } else if (pc.l2) {
                L.pool = PoolDesc{h->num_pool.base, P.l2.chunk_bytes, P.l2.num_chunks, P.l2.pool_mode,
                                  h->num_pool.states};
                cuda_check(launch_row_kernel(L, P.fast ? kAccLP : P.acc, P.fast ? false : P.flat, kVarNumeric, st),
                           "numeric L2 kernel");
            } else if (pc.tiny) {
                cuda_check(launch_numeric_tiny(L, st), "numeric tiny kernel");
            } else if (pc.fast) {
                cuda_check(P.flat ? launch_numeric_flat_fast(L, st) : launch_numeric_fast(L, st), "numeric kernel");
            } else {
                cuda_check(launch_row_kernel(L, P.acc, P.flat, kVarNumeric, st), "numeric kernel");
            }
        }
        if (full && !replayed && h->replay_eligible && !h->replay_ready && h->numeric_calls >= 2)
            record_replay(h, a, b, c_cols, c_vals, st);
        if (I.config.sort_output && row_hi > row_lo)
            cuda_check(launch_sort_rows(row_hi - row_lo, h->d_rowptr + row_lo, c_cols, c_vals, I.max_row_size, st),
                       "sort_output");
        if (stats) {
            DevCounters hc{};
            cuda_check(cudaEventRecord(e1, st), "event");
            cuda_check(cudaMemcpyAsync(&hc, h->d_ctr, sizeof(hc), cudaMemcpyDeviceToHost, st), "counters");
            cuda_check(cudaStreamSynchronize(st), "numeric sync");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            stats->ms = ms;
            stats->pool_allocations = static_cast<int64_t>(hc.pool_allocations);
            stats->l2_inserts = static_cast<int64_t>(hc.l2_inserts);
            if (hc.error)
                fail(SPG_ERR_INTERNAL, std::string("numeric: ") + dev_error_text(hc.error));
        }
    });
}

int spg_numeric(spg_handle_t h, const spg_csr* a, const spg_csr* b, int32_t* c_cols, double* c_vals,
                spg_phase_stats* stats, void* stream)
{
    if (!h)
        return guarded([&] { fail(SPG_ERR_CONTRACT, "numeric: null handle"); });
    return numeric_impl(h, a, b, 0, h->info.m, c_cols, c_vals, stats, stream);
}

int spg_numeric_rows(spg_handle_t h, const spg_csr* a, const spg_csr* b, int32_t row_begin, int32_t row_end,
                     int32_t* c_cols, double* c_vals, spg_phase_stats* stats, void* stream)
{
    if (!h)
        return guarded([&] { fail(SPG_ERR_CONTRACT, "numeric: null handle"); });
    return numeric_impl(h, a, b, row_begin, row_end, c_cols, c_vals, stats, stream);
}

int spg_handle_info_get(spg_handle_t h, spg_handle_info* out)
{
    if (!h || !out)
        return SPG_ERR_CONTRACT;
    *out = h->info;
    out->heavy_path = h->num_slab ? 2 : h->num_heavy ? 1 : 0;
    out->b_sorted = h->b_sorted ? 1 : 0;
    return SPG_OK;
}

int spg_handle_copy_row_offsets(spg_handle_t h, int64_t* host_dst)
{
    return guarded([&] {
        if (!h || !host_dst)
            fail(SPG_ERR_CONTRACT, "null argument");
        cuda_check(cudaMemcpyAsync(host_dst, h->d_rowptr, sizeof(int64_t) * (int64_t{h->info.m} + 1),
                                   cudaMemcpyDeviceToHost, h->stream),
                   "copy row offsets");
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
    });
}

int spg_handle_copy_per_row_flops(spg_handle_t h, int64_t* host_dst)
{
    return guarded([&] {
        if (!h || !host_dst)
            fail(SPG_ERR_CONTRACT, "null argument");
        if (!h->d_prf)
            fail(SPG_ERR_CONTRACT, "handle has no per-row flops (imported handle)");
        cuda_check(cudaMemcpyAsync(host_dst, h->d_prf, sizeof(int64_t) * h->info.m, cudaMemcpyDeviceToHost,
                                   h->stream),
                   "copy per-row flops");
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
    });
}

int spg_handle_copy_row_offsets_device(spg_handle_t h, int64_t* device_dst, void* stream)
{
    return guarded([&] {
        if (!h || !device_dst)
            fail(SPG_ERR_CONTRACT, "null argument");
        cuda_check(cudaMemcpyAsync(device_dst, h->d_rowptr, sizeof(int64_t) * (int64_t{h->info.m} + 1),
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)),
                   "copy row offsets");
    });
}

int spg_handle_set_numeric(spg_handle_t h, const spg_config* cfg, const spg_resolved* numeric_choice)
{
    return guarded([&] {
        if (!h)
            fail(SPG_ERR_CONTRACT, "null handle");
        if (cfg)
            h->info.config = *cfg;
        if (numeric_choice) {
            h->info.numeric_choice = *numeric_choice;
            h->numeric_forced = true;
        }
        build_numeric_plan(h, h->stream);
    });
}

int spg_handle_import(const spg_handle_desc* d, spg_handle_t* out, void* stream)
{
    spg_handle* h = nullptr;
    const int rc = guarded([&] {
        if (!d || !out || !d->c_row_offsets)
            fail(SPG_ERR_CONTRACT, "import: null argument");
        require_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        h = new spg_handle;
        h->stream = st;
        spg_handle_info& I = h->info;
        I.m = d->m;
        I.n = d->n;
        I.k = d->k;
        I.nnz_a = d->nnz_a;
        I.nnz_b = d->nnz_b;
        I.nnz_c = d->c_row_offsets[d->m] - d->c_row_offsets[0];
        I.flops = d->flops;
        I.compression = d->compression;
        I.max_row_size = d->max_row_size;
        I.avg_row_size = d->avg_row_size;
        I.avg_row_size_estimate = d->avg_row_size_estimate;
        I.symbolic_choice = d->symbolic_choice;
        I.numeric_choice = d->numeric_choice;
        I.config = d->config;
        I.symbolic_stats = d->symbolic_stats;
        I.compress_ms = d->compress_ms;
        h->d_rowptr = dalloc<int64_t>(int64_t{d->m} + 1, st, "C row offsets");
        h->d_ctr = dalloc<DevCounters>(1, st, "counters");
        I.d_c_row_offsets = h->d_rowptr;
        I.d_per_row_flops = nullptr;
        if (d->per_row_flops && d->m > 0) {
            h->d_prf = dalloc<int64_t>(d->m, st, "per-row flops");
            cuda_check(cudaMemcpyAsync(h->d_prf, d->per_row_flops, sizeof(int64_t) * d->m, cudaMemcpyHostToDevice, st),
                       "upload per-row flops");
            I.d_per_row_flops = h->d_prf;
        }
        cuda_check(cudaMemcpyAsync(h->d_rowptr, d->c_row_offsets, sizeof(int64_t) * (int64_t{d->m} + 1),
                                   cudaMemcpyHostToDevice, st),
                   "upload row offsets");
        ScanTotals* d_stot = dalloc<ScanTotals>(1, st, "hist");
        cuda_check(cudaMemsetAsync(d_stot, 0, sizeof(ScanTotals), st), "memset");
        cuda_check(launch_row_bucket_hist(d->m, h->d_rowptr, d_stot, st), "row hist");
        cuda_check(cudaMemcpyAsync(&h->size_hist, d_stot, sizeof(ScanTotals), cudaMemcpyDeviceToHost, st), "hist");
        cuda_check(cudaStreamSynchronize(st), "import sync");
        cudaFreeAsync(d_stot, st);
        I.max_row_size = std::max<int64_t>(I.max_row_size, static_cast<int64_t>(h->size_hist.max_size));
        // the reference's numeric takes its choice from the handle as is: an
        // Auto handle whose choice is the resolved one keeps the GPU plan, an
        // edited choice (acceptance_main.cpp:417-425) runs as forced
        spg_resolved auto_choice{};
        spg_resolve_config(SPG_PHASE_NUMERIC, I.k, &I.flops, &I.compression, &I.config, I.max_row_size,
                           &auto_choice);
        h->numeric_forced = !(I.config.accumulator == SPG_ACC_AUTO &&
                              std::memcmp(&auto_choice, &I.numeric_choice, sizeof(spg_resolved)) == 0);
        build_numeric_plan(h, st);
        *out = h;
    });
    if (rc != SPG_OK) {
        delete h;
        if (out)
            *out = nullptr;
    }
    return rc;
}

int spg_handle_check(spg_handle_t h)
{
    return guarded([&] {
        if (!h)
            fail(SPG_ERR_CONTRACT, "null handle");
        DevCounters hc{};
        cuda_check(cudaMemcpyAsync(&hc, h->d_ctr, sizeof(hc), cudaMemcpyDeviceToHost, h->stream), "counters");
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        if (hc.error)
            fail(SPG_ERR_INTERNAL, dev_error_text(hc.error));
    });
}

int spg_handle_replay_state(spg_handle_t h)
{
    if (!h)
        return 0;
    return h->replay_ready ? 2 : h->replay_eligible ? 1 : 0;
}

void spg_handle_destroy(spg_handle_t h)
{
    delete h; // stream-ordered release (see ~spg_handle)
}

int spg_row_flops(const spg_csr* a, const spg_csr* b, int64_t* d_out, void* stream)
{
    return guarded([&] {
        validate_csr(a, "row_flops: A", false);
        validate_csr(b, "row_flops: B", false);
        if (a->num_cols != b->num_rows)
            fail(SPG_ERR_CONTRACT, "flops_stats: inner dimensions do not match");
        if (!d_out && a->num_rows > 0)
            fail(SPG_ERR_CONTRACT, "row_flops: null output");
        require_device();
        cuda_check(launch_row_flops(a->num_rows, a->row_offsets, a->col_indices, b->row_offsets, d_out,
                                    static_cast<cudaStream_t>(stream)),
                   "row flops");
    });
}

int spg_transpose(const spg_csr* a, int64_t* d_t_row_offsets, int32_t* d_t_cols, double* d_t_vals, void* stream)
{
    return guarded([&] {
        validate_csr(a, "transpose: A", true);
        if (!d_t_row_offsets || (a->nnz > 0 && (!d_t_cols || !d_t_vals)))
            fail(SPG_ERR_CONTRACT, "transpose: null output");
        require_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        ScanTotals* d_stot = dalloc<ScanTotals>(1, st, "scan totals");
        ScanTotals hs{};
        cuda_check(cudaMemsetAsync(d_stot, 0, sizeof(ScanTotals), st), "memset");
        cuda_check(launch_transpose_count(a->num_rows, a->num_cols, a->row_offsets, a->col_indices, d_t_row_offsets,
                                          d_stot, st),
                   "transpose count");
        cuda_check(cudaMemcpyAsync(&hs, d_stot, sizeof(hs), cudaMemcpyDeviceToHost, st), "transpose totals");
        cuda_check(cudaStreamSynchronize(st), "transpose sync");
        cudaFreeAsync(d_stot, st);
        cuda_check(launch_transpose_fill(a->num_rows, a->num_cols, a->row_offsets, a->col_indices, a->values,
                                         d_t_row_offsets, d_t_cols, d_t_vals, static_cast<int64_t>(hs.max_size), st),
                   "transpose fill");
    });
}

int spg_row_digests(int32_t m, const int64_t* d_row_offsets, const int32_t* d_cols, const double* d_vals,
                    uint64_t* d_out, void* stream)
{
    return guarded([&] {
        if (m < 0 || (m > 0 && (!d_row_offsets || !d_out)))
            fail(SPG_ERR_CONTRACT, "row_digests: bad argument");
        require_device();
        cuda_check(launch_row_digests(m, d_row_offsets, d_cols, d_vals, reinterpret_cast<unsigned long long*>(d_out),
                                      static_cast<cudaStream_t>(stream)),
                   "row digests");
    });
}

int spg_sort_rows(int32_t m, const int64_t* d_row_offsets, int32_t* d_cols, double* d_vals, void* stream)
{
    return guarded([&] {
        require_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        // max row size for the kernel's path choice
        ScanTotals* d_stot = dalloc<ScanTotals>(1, st, "hist");
        ScanTotals hs{};
        cuda_check(cudaMemsetAsync(d_stot, 0, sizeof(ScanTotals), st), "memset");
        cuda_check(launch_row_bucket_hist(m, d_row_offsets, d_stot, st), "row hist");
        cuda_check(cudaMemcpyAsync(&hs, d_stot, sizeof(hs), cudaMemcpyDeviceToHost, st), "hist");
        cuda_check(cudaStreamSynchronize(st), "sync");
        cudaFreeAsync(d_stot, st);
        cuda_check(launch_sort_rows(m, d_row_offsets, d_cols, d_vals, static_cast<int64_t>(hs.max_size), st),
                   "sort rows");
    });
}

} // extern "C"
