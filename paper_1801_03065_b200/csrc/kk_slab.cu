// Heavy numeric rows by column slabs (sm_100a).
//
// Rows of C beyond the warp tables (R-MAT squares: 10^3..5*10^5 outputs per
// row, 10^4..10^7 products) run one CTA per row, rows taken largest first
// from a device queue.  The row's column domain is walked in SLABS
// [c_lo, c_hi) sized so that a slab's distinct columns fit the CTA's
// shared-memory table (~4K keys).  B's rows are column-sorted, so the part of
// B row j that falls in a slab is one contiguous RUN; per A entry a cursor
// remembers where the next slab's run starts, so every product is read once
// in total and the per-slab bookkeeping is one short run-end search per A
// entry.
//
// Left-to-right value order (bitwise the reference's sums): inside
// a slab the products are visited in the reference's (A position, B position)
// order.  A chunk of 512 products is staged, partitioned by a hash of the
// column into 8 classes with a STABLE counting sort (per-warp match ranks +
// a 64-entry scan), and warp c owns class c: it folds its products into its
// private table partition in product order (duplicates inside a 32-product
// window folded by the lowest lane, lane order = product order).  A key lives
// in exactly one partition, so every key's products are summed in product
// order, starting from the first product.
//
// Slab width is adaptive: the first guess assumes uniform column density
// (cap/k), later slabs rescale by the density just seen, and a slab whose
// partition exceeds its key budget is abandoned (tables cleared, cursors not
// advanced) and retried at half the width.  Rows come out slab by slab in
// increasing column ranges (a slab's columns in partition/slot order); the
// contract compares sorted rows.  The row's entry count is checked against
// the symbolic structure.
//
// A staged column below c_lo means a B row is not column-sorted (the run
// ended early): the kernel raises kDevUnsorted — the host plans this kernel
// only when the symbolic pass saw every referenced B row sorted.
#include <climits>
#include <cstdint>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {

constexpr int kSW = 8;                // warps per CTA = table partitions = key classes
constexpr int kST = kSW * 32;         // threads
constexpr int kTW = 1024;             // slots per partition
constexpr int kTWMax = 768;           // keys per partition before the slab is abandoned
constexpr int kXTarget = kSW * 480;   // target distinct keys per slab
constexpr int kG = kST;               // A entries per group (one per thread in the run search)
constexpr int kF = 2 * kST;           // products per staged chunk (two windows per warp)

struct __align__(16) SlabSmem {
    int32_t keys[kSW][kTW];
    double vals[kSW][kTW];
    double sval[kF];
    int32_t scol[kF];
    int64_t qst[kG];      // first B position of each non-empty run of the group
    double av[kG];        // A value of that run
    int32_t roff[kG + 1]; // flat offset of each run inside the group (compacted, strictly increasing)
    int32_t cnt[kSW][kSW]; // [staging warp][class] products of the chunk
    long long wsum[kSW];
    int32_t nkeys[kSW];
    int64_t row;
    int32_t ovf;
};

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ int key_class(int32_t key)
{
    return static_cast<int>((static_cast<uint32_t>(key) * 0x9E3779B1u) >> 29);
}

__device__ __forceinline__ uint32_t key_slot(int32_t key)
{
    return (static_cast<uint32_t>(key) * 0x85EBCA6Bu) >> 22; // 10 bits, independent of the class
}

// block-wide exclusive scan of one int64 per thread; *total = the sum
__device__ __forceinline__ long long block_scan(long long v, long long* wsum, long long* total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o)
            incl += y;
    }
    if (lane == 31)
        wsum[warp] = incl;
    __syncthreads();
    long long pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kSW; ++w) {
        const long long x = wsum[w];
        pre += w < warp ? x : 0;
        tot += x;
    }
    *total = tot;
    __syncthreads();
    return pre + incl - v;
}

// First q in [s, be) with cols[q] >= c_hi, for a column-sorted row (an
// unsorted row is caught at staging).  Runs are mostly short: eight
// independent loads first, then a galloping search.
__device__ __forceinline__ int64_t run_end(const int32_t* __restrict__ cols, int64_t s, int64_t be, int64_t c_hi)
{
    int64_t q = s;
    for (int round = 0; round < 2; ++round) {
        const int64_t n = be - q;
        if (n <= 0)
            return be;
        int32_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            c[u] = u < n ? __ldg(cols + q + u) : INT_MAX;
        int first = 8;
#pragma unroll
        for (int u = 7; u >= 0; --u)
            if (c[u] >= c_hi)
                first = u;
        if (first < 8 || n <= 8)
            return q + (first < n ? first : n);
        q += 8;
    }
    // gallop: cols[q - 1] < c_hi
    int64_t step = 16, lo = q - 1, hi = be;
    while (q + step - 1 < be) {
        if (__ldg(cols + q + step - 1) >= c_hi) {
            hi = q + step - 1;
            break;
        }
        lo = q + step - 1;
        q += step;
        step <<= 1;
    }
    // cols[lo] < c_hi, hi == be or cols[hi] >= c_hi
    while (hi - lo > 1) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(cols + mid) >= c_hi)
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

// run of flat position f inside a group: roff strictly increasing, roff[0] = 0,
// roff[nr] = total.  `hint` (warp-uniform, monotone) is the run of an earlier
// window start; fw = this window's start (<= every lane's f).
__device__ __forceinline__ int find_run(const int32_t* roff, int nr, int& hint, int32_t fw, int32_t f, int lane)
{
    for (;;) {
        const int idx = hint + 1 + lane;
        const int32_t b = idx <= nr ? roff[idx] : INT_MAX;
        const uint32_t M = __ballot_sync(kFull, b <= fw);
        hint += __popc(M);
        if (M != kFull)
            break;
    }
    // roff[hint] <= fw < roff[hint + 1]; run starts inside the window (at most
    // 31, runs are non-empty)
    const int idx = hint + 1 + lane;
    const int32_t b = idx <= nr ? roff[idx] : INT_MAX;
    uint32_t M2 = __ballot_sync(kFull, b <= fw + 31);
    int p = hint;
    while (M2) {
        const int j = __ffs(M2) - 1;
        M2 &= M2 - 1;
        if (__shfl_sync(kFull, b, j) <= f)
            ++p;
    }
    return p;
}

} // namespace

// Optional phase profile (-DKK_SLAB_PROF): thread 0 of every CTA adds clock
// deltas and event counts; read with spg_debug_slab_prof.
#ifdef KK_SLAB_PROF
__device__ unsigned long long g_slab_prof[16];
#define PROF_DECL unsigned long long prof_t = clock64();
#define PROF_MARK(idx)                                                                                   \
    do {                                                                                                 \
        if (threadIdx.x == 0) {                                                                          \
            const unsigned long long now = clock64();                                                    \
            atomicAdd(&g_slab_prof[idx], now - prof_t);                                                  \
            prof_t = now;                                                                                \
        }                                                                                                \
    } while (0)
#define PROF_RESET                                                                                       \
    do {                                                                                                 \
        if (threadIdx.x == 0)                                                                            \
            prof_t = clock64();                                                                          \
    } while (0)
#define PROF_COUNT(idx, n)                                                                               \
    do {                                                                                                 \
        if (threadIdx.x == 0)                                                                            \
            atomicAdd(&g_slab_prof[idx], (unsigned long long)(n));                                       \
    } while (0)
#else
#define PROF_DECL
#define PROF_MARK(idx)
#define PROF_RESET
#define PROF_COUNT(idx, n)
#endif

struct SlabArgs {
    int32_t* scratch;   // per CTA: cursors [max_a_row] + run ends [max_a_row] (int32, relative to the B row)
    int64_t max_a_row;  // longest A row among the planned rows
    int64_t k;          // column domain
    const int64_t* prf; // per-row flops (distinct-key estimate of the first slab), may be null
};

__global__ void __launch_bounds__(kST, 2) numeric_slab_kernel(const RowLaunch L, const SlabArgs S)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SlabSmem& sm = *reinterpret_cast<SlabSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* cur = S.scratch + (size_t)blockIdx.x * 2 * S.max_a_row;
    int32_t* endr = cur + S.max_a_row;
    int32_t* mykeys = sm.keys[warp];
    double* myvals = sm.vals[warp];

    for (int t = lane; t < kTW; t += 32)
        mykeys[t] = kEmpty;
    __syncwarp();
    PROF_DECL

    for (;;) {
        if (threadIdx.x == 0)
            sm.row = static_cast<int64_t>(atomicAdd(&L.ctr->next_row[0], 1ull));
        __syncthreads();
        const int64_t r = sm.row;
        __syncthreads();
        if (r >= L.nrows)
            break;
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int64_t cap = __ldg(L.c_rowptr + i + 1) - cbase;
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        const int64_t d = aend - abeg;
        if (d > S.max_a_row) { // plan / operand mismatch: the cursors would not fit
            if (threadIdx.x == 0)
                raise_error(L.ctr, kDevRowOverflow);
            continue;
        }
        int64_t emitted = 0;
        int64_t c_lo = 0;
        // first slab: all columns when the row fits one table, else the
        // uniform-density guess (then corrected from the slab's product count)
        int64_t W = cap <= kXTarget ? S.k : imax64(32, S.k * kXTarget / imax64(cap, 1));
        // distinct keys per product: the row's ratio first, then the last slab's
        const int64_t row_flops = S.prf ? __ldg(S.prf + i) : 0;
        double ratio = row_flops > 0 ? static_cast<double>(cap) / static_cast<double>(row_flops) : 1.0;
        bool first = true;
        bool bad = false;
        int replans = 0;
        while (c_lo < S.k && !bad) {
            const int64_t c_hi = W >= S.k - c_lo ? S.k : c_lo + W;
            const bool full = c_lo == 0 && c_hi == S.k;
            int32_t nk = 0; // this warp's keys in the slab (warp-uniform)
            if (threadIdx.x == 0)
                sm.ovf = 0;
            bool ovf = false;
            bool replan = false;
            int64_t slab_products = 0;
            for (int64_t g0 = 0; g0 < d && !ovf; g0 += kG) {
                const int ng = static_cast<int>(d - g0 < kG ? d - g0 : kG);
                PROF_RESET;
                // ---- runs of this group's A entries in [c_lo, c_hi) ----
                int64_t s = 0, e = 0;
                double a = 0.0;
                if (threadIdx.x < ng) {
                    const int64_t p = g0 + threadIdx.x;
                    const int32_t j = __ldg(L.a_cols + abeg + p);
                    a = __ldg(L.a_vals + abeg + p);
                    const int64_t bs = __ldg(L.b_rowptr + j), be = __ldg(L.b_rowptr + j + 1);
                    s = bs + (first ? 0 : cur[p]);
                    e = full ? be : run_end(L.b_cols, s, be, c_hi);
                    if (!full)
                        endr[p] = static_cast<int32_t>(e - bs);
                }
                const int64_t len = e - s;
                long long tot;
                const long long packed = block_scan((len << 20) | (len > 0 ? 1 : 0), sm.wsum, &tot);
                const int32_t nr = static_cast<int32_t>(tot & 0xFFFFF);
                const int64_t T = tot >> 20;
                if (len > 0) {
                    const int ridx = static_cast<int>(packed & 0xFFFFF);
                    sm.roff[ridx] = static_cast<int32_t>(packed >> 20);
                    sm.qst[ridx] = s;
                    sm.av[ridx] = a;
                }
                if (threadIdx.x == 0)
                    sm.roff[nr] = static_cast<int32_t>(T);
                __syncthreads();
                slab_products += T;
                if (g0 == 0 && replans < 2) {
                    // keys this slab will hold, predicted from its products
                    // (block-uniform): resize before any product is folded
                    const double est = static_cast<double>(T) * (static_cast<double>(d) / ng) * ratio;
                    const int64_t w = c_hi - c_lo;
                    if (est > 1.25 * kXTarget && w > 1) {
                        W = imax64(1, static_cast<int64_t>(w * (0.9 * kXTarget / est)));
                        replan = true;
                    } else if (est < 0.25 * kXTarget && c_hi < S.k) {
                        W = static_cast<int64_t>(w * min(8.0, 0.5 * kXTarget / fmax(est, 1.0))) + 1;
                        replan = true;
                    }
                    if (replan) {
                        ++replans;
                        break;
                    }
                }
                PROF_MARK(0);
                PROF_COUNT(8, 1);
                PROF_COUNT(9, T);
                // ---- chunks of kF products: stage, partition by class, fold ----
                int hint = 0;
                int32_t col[2];
                double v[2], va[2]; // B value and A value: multiplied at the scatter, so the
                                    // prefetched loads are not waited for before the fold
                auto load = [&](int64_t f0) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int32_t fw = static_cast<int32_t>(f0) + 64 * warp + 32 * u;
                        const int32_t f = fw + lane;
                        col[u] = -1;
                        v[u] = 0.0;
                        va[u] = 0.0;
                        if (fw < T) { // warp-uniform
                            const int p = find_run(sm.roff, nr, hint, fw, f, lane);
                            if (f < T) {
                                const int64_t q = sm.qst[p] + (f - sm.roff[p]);
                                col[u] = __ldg(L.b_cols + q);
                                v[u] = __ldg(L.b_vals + q);
                                va[u] = sm.av[p];
                            }
                        }
                    }
                };
                if (T > 0)
                    load(0);
                for (int64_t f0 = 0; f0 < T; f0 += kF) {
                    // class ranks inside this warp's two windows (stable)
                    if (lane < kSW)
                        sm.cnt[warp][lane] = 0;
                    __syncwarp();
                    int32_t pos[2], cls[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const bool valid = col[u] >= 0;
                        if (valid && col[u] < c_lo)
                            bad = true; // unsorted B row (see header)
                        cls[u] = valid ? key_class(col[u]) : kSW;
                        const uint32_t grp = __match_any_sync(kFull, cls[u]);
                        const int leader = __ffs(grp) - 1;
                        int32_t base = 0;
                        if (valid && lane == leader) {
                            base = sm.cnt[warp][cls[u]];
                            sm.cnt[warp][cls[u]] = base + __popc(grp);
                        }
                        pos[u] = __shfl_sync(kFull, base, leader) + __popc(grp & lanemask_lt());
                        __syncwarp();
                    }
                    __syncthreads(); // (A) counts visible; the previous chunk's folds are done
                    if (sm.ovf)
                        ovf = true;
                    if (ovf)
                        break;
                    // exclusive offsets in (class, staging warp) order: lane l
                    // holds entries 2l, 2l+1 of the class-major 64-vector
                    const int t0 = 2 * lane, t1 = 2 * lane + 1;
                    const int32_t x0 = sm.cnt[t0 & 7][t0 >> 3], x1 = sm.cnt[t1 & 7][t1 >> 3];
                    int32_t incl = x0 + x1;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int32_t y = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o)
                            incl += y;
                    }
                    const int32_t ex0 = incl - x0 - x1, ex1 = incl - x1;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (col[u] >= 0) {
                            const int t = cls[u] * kSW + warp;
                            const int32_t o0 = __shfl_sync(kFull, ex0, t >> 1), o1 = __shfl_sync(kFull, ex1, t >> 1);
                            const int32_t dst = ((t & 1) ? o1 : o0) + pos[u];
                            sm.scol[dst] = col[u];
                            sm.sval[dst] = __dmul_rn(va[u], v[u]);
                        } else {
                            __shfl_sync(kFull, ex0, 0);
                            __shfl_sync(kFull, ex1, 0);
                        }
                    }
                    const int32_t seg_lo = __shfl_sync(kFull, ex0, 4 * warp);
                    const int32_t seg_hi = warp + 1 < kSW ? __shfl_sync(kFull, ex0, 4 * (warp + 1))
                                                          : __shfl_sync(kFull, incl, 31);
                    __syncthreads(); // (C) staging written
                    PROF_MARK(1);
                    PROF_COUNT(10, 1);
                    if (f0 + kF < T)
                        load(f0 + kF); // next chunk's loads overlap this chunk's folds
                    // ---- fold class `warp` into partition `warp`, product order ----
                    for (int32_t x0 = seg_lo; x0 < seg_hi; x0 += 32) {
                        const bool valid = x0 + lane < seg_hi;
                        const int32_t key = valid ? sm.scol[x0 + lane] : -1 - lane;
                        const double val = valid ? sm.sval[x0 + lane] : 0.0;
                        const uint32_t grp = __match_any_sync(kFull, key);
                        const bool leader = valid && (__ffs(grp) - 1) == lane;
                        uint32_t slot = 0;
                        bool is_new = false;
                        if (leader) {
                            slot = key_slot(key);
                            for (;;) {
                                const int32_t kx = mykeys[slot];
                                if (kx == key)
                                    break;
                                if (kx == kEmpty) {
                                    const int32_t old = atomicCAS(&mykeys[slot], kEmpty, key);
                                    if (old == kEmpty) {
                                        is_new = true;
                                        break;
                                    }
                                    if (old == key)
                                        break;
                                }
                                slot = (slot + 1) & (kTW - 1);
                            }
                        }
                        double acc = val;
                        if (leader && !is_new)
                            acc = __dadd_rn(myvals[slot], val);
                        uint32_t rest = leader ? (grp & (grp - 1)) : 0u;
                        const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
                        for (int rr = 0; rr < rounds; ++rr) {
                            const int src = rest ? __ffs(rest) - 1 : lane;
                            const double xv = __shfl_sync(kFull, val, src);
                            if (rest) {
                                acc = __dadd_rn(acc, xv);
                                rest &= rest - 1;
                            }
                        }
                        if (leader)
                            myvals[slot] = acc;
                        nk += __popc(__ballot_sync(kFull, is_new));
                        __syncwarp();
                        if (nk > kTWMax) { // warp-uniform: this slab is too wide
                            if (lane == 0)
                                sm.ovf = 1;
                            break;
                        }
                    }
                    PROF_MARK(5);
                }
                PROF_MARK(2);
                __syncthreads(); // folds done before the next group's runs overwrite roff/qst/av
                PROF_MARK(3);
                if (sm.ovf)
                    ovf = true;
            }
            if (replan) {
                PROF_COUNT(14, 1);
                continue; // nothing folded, cursors unchanged: plan the slab again
            }
            if (__syncthreads_or(bad)) {
                if (threadIdx.x == 0)
                    raise_error(L.ctr, kDevUnsorted);
                bad = true;
            }
            PROF_RESET;
            if (ovf || bad) {
                PROF_COUNT(11, 1);
                // abandon the slab: clear the partitions, retry at half width
                for (int t = lane; t < kTW; t += 32)
                    mykeys[t] = kEmpty;
                __syncthreads();
                W = imax64(1, (c_hi - c_lo) / 2);
                continue;
            }
            // ---- slab done: advance cursors, emit ----
            if (!full)
                for (int64_t p = threadIdx.x; p < d; p += kST)
                    cur[p] = endr[p];
            first = false;
            if (lane == 0)
                sm.nkeys[warp] = nk;
            __syncthreads();
            int32_t before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kSW; ++w) {
                const int32_t x = sm.nkeys[w];
                before += w < warp ? x : 0;
                total += x;
            }
            int64_t o = emitted + before;
            for (int t0 = 0; t0 < kTW; t0 += 32) {
                const int32_t kx = mykeys[t0 + lane];
                const bool hit = kx != kEmpty;
                const uint32_t m = __ballot_sync(kFull, hit);
                if (hit) {
                    const int64_t dst = o + __popc(m & lanemask_lt());
                    if (dst < cap) {
                        __stcs(L.c_cols + cbase + dst, kx);
                        __stcs(L.c_vals + cbase + dst, myvals[t0 + lane]);
                    }
                    mykeys[t0 + lane] = kEmpty;
                }
                o += __popc(m);
            }
            emitted += total;
            PROF_COUNT(12, 1);
            PROF_COUNT(13, total);
            // next slab: rescale the width by the density just seen (at most 4x)
            const int64_t w_used = c_hi - c_lo;
            W = total > 0 ? imax64(1, min(4 * w_used, w_used * kXTarget / total)) : w_used * 4;
            if (slab_products > 0)
                ratio = static_cast<double>(total) / static_cast<double>(slab_products);
            replans = 0;
            c_lo = c_hi;
            __syncthreads();
            PROF_MARK(4);
        }
        if (threadIdx.x == 0 && !bad && emitted != cap)
            raise_error(L.ctr, emitted < cap ? kDevRowShort : kDevRowOverflow);
    }
}

size_t slab_smem_bytes() { return sizeof(SlabSmem); }

} // namespace kk

extern "C" int spg_debug_slab_prof(unsigned long long* out, int reset)
{
#ifdef KK_SLAB_PROF
    if (out)
        cudaMemcpyFromSymbol(out, kk::g_slab_prof, sizeof(kk::g_slab_prof));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(kk::g_slab_prof, z, sizeof(z));
    }
    return 1;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}

namespace kk {

int numeric_slab_blocks_per_sm()
{
    const void* fn = reinterpret_cast<const void*>(&numeric_slab_kernel);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SlabSmem));
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kST, sizeof(SlabSmem)) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

cudaError_t launch_numeric_slab(const RowLaunch& L, int32_t* scratch, int64_t max_a_row, int64_t k,
                                const int64_t* prf, int grid, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_slab_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SlabSmem));
    if (e != cudaSuccess)
        return e;
    SlabArgs S{scratch, max_a_row, k, prf};
    numeric_slab_kernel<<<grid, kST, sizeof(SlabSmem), st>>>(L, S);
    count_launch();
    return cudaGetLastError();
}

} // namespace kk
