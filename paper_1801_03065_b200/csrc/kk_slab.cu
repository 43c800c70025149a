// Heavy numeric rows by column slabs, one warp per slab sequence (sm_100a).
//
// Rows of C beyond the warp tables (R-MAT squares: 10^3..5*10^5 outputs per
// row, 10^4..10^7 products) are walked in column SLABS [c_lo, c_hi) sized so
// that a slab's distinct columns fit one warp's shared-memory table (~225 of
// 512 slots; 8 warps per CTA, 3 CTAs per SM).  B's rows are column-sorted, so
// the part of B row j inside a slab is one contiguous RUN; per A entry the
// warp keeps a cursor (where the next slab's run starts) and the column found
// there, so an A entry whose B row has nothing in the slab costs one
// coalesced scratch read, and every product is read exactly once.
//
// Plan: the cursors are scanned 32 at a time; entries with a run in the slab
// go into a shared queue (A order) and their run ends are searched 32 queued
// entries at a time.  Fold: a window producer keeps two mapped 32-product
// windows (their B loads) in flight ahead of the window being folded.
//
// Left-to-right value order (bitwise the reference's sums): one
// warp accumulates a slab, visiting its products in the reference's
// (A position, B position) order — runs one after another when they are long
// (lanes over a run's entries: distinct keys, no conflicts), or 32-product
// windows across several short runs with duplicate keys folded by the lowest
// lane in lane (= product) order.  Every key's products are therefore summed
// in product order starting from the first product.
//
// Slab width is adaptive: the first guess assumes uniform column density,
// each slab's product count (known before any product is folded) corrects it
// with the last slab's keys-per-product ratio, later slabs rescale by the
// density just seen, and a slab whose table overflows anyway is abandoned
// (table cleared, cursors not advanced) and retried at half the width.
//
// Rows whose slab walk would be long for one warp (A-row length x row size
// above kSplitWork) are cut into equal column PARTS walked by different warps
// (cursors start at the part's first column, found by binary search).  A
// part reserves its output block in the row when each slab completes, so the
// columns of such a row come out grouped by slab in completion order; other
// rows come out slab by slab in increasing column ranges.  The contract
// compares sorted rows; the row's entry count is checked against the
// symbolic structure.
//
// A B row that is not column-sorted makes a run end early and a later slab
// meet a column below its lower bound: kDevUnsorted (the host plans this
// kernel only when the symbolic pass saw every referenced B row sorted).
#include <algorithm>
#include <climits>
#include <cstdint>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {

#ifndef KK_SLAB_LOG2_TW
#define KK_SLAB_LOG2_TW 9 // table slots per warp (A/B builds: -DKK_SLAB_LOG2_TW=9 -DKK_SLAB_CTAS=3)
#endif
#ifndef KK_SLAB_CTAS
#define KK_SLAB_CTAS 3 // resident CTAs per SM the kernel is compiled for
#endif
constexpr int kWarps = 8;                          // independent warps per CTA
constexpr int kTW = 1 << KK_SLAB_LOG2_TW;          // table slots per warp
constexpr int kTWMax = kTW * 3 / 4;                // keys before a slab is abandoned
#ifndef KK_SLAB_XFRAC
#define KK_SLAB_XFRAC 450 // target keys per slab, per 1024 table slots
#endif
#ifndef KK_SLAB_ACCEPT
#define KK_SLAB_ACCEPT 1.6 // a planned slab predicted above ACCEPT * kX keys is re-planned narrower
#endif
constexpr int kX = kTW * KK_SLAB_XFRAC / 1024;     // target distinct keys per slab
#ifndef KK_SLAB_SPLIT
#define KK_SLAB_SPLIT 4e8
#endif
constexpr double kSplitWork = KK_SLAB_SPLIT; // A-row length x row size per part
#ifndef KK_SLAB_DEPTH
#define KK_SLAB_DEPTH 2 // mapped windows in flight ahead of the one being folded
#endif
constexpr int kDepth = KK_SLAB_DEPTH;



__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t key_slot(int32_t key)
{
    return (static_cast<uint32_t>(key) * 0x9E3779B1u) >> (32 - KK_SLAB_LOG2_TW);
}

// Run-end search, split so that two A entries' first loads are in flight
// together: probe16 loads the 16 columns at q (INT_MAX past be), finish16
// evaluates them and, for a run longer than 16, gallops.  Returns the first
// q in [s, be) with cols[q] >= c (column-sorted row) and *at = cols[q]
// (INT_MAX when q == be).
struct Probe16 {
    int32_t v[16];
};

__device__ __forceinline__ void probe16(const int32_t* __restrict__ cols, int64_t q, int64_t be, Probe16& P)
{
    const int64_t n = be - q;
#pragma unroll
    for (int u = 0; u < 16; ++u)
        P.v[u] = u < n ? __ldg(cols + q + u) : INT_MAX;
}

__device__ __forceinline__ int64_t finish16(const int32_t* __restrict__ cols, int64_t q, int64_t be, int64_t c,
                                            const Probe16& P, int32_t* at)
{
    int first = 16;
    int32_t fv = INT_MAX;
#pragma unroll
    for (int u = 15; u >= 0; --u)
        if (P.v[u] >= c) {
            first = u;
            fv = P.v[u];
        }
    if (first < 16) {
        *at = fv;
        return q + first < be ? q + first : be;
    }
    q += 16;
    if (q >= be) {
        *at = INT_MAX;
        return be;
    }
    // gallop: cols[q - 1] < c
    int64_t step = 16, lo = q - 1, hi = be;
    while (q + step - 1 < be) {
        if (__ldg(cols + q + step - 1) >= c) {
            hi = q + step - 1;
            break;
        }
        lo = q + step - 1;
        q += step;
        step <<= 1;
    }
    while (hi - lo > 1) { // cols[lo] < c, hi == be or cols[hi] >= c
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(cols + mid) >= c)
            hi = mid;
        else
            lo = mid;
    }
    *at = hi < be ? __ldg(cols + hi) : INT_MAX;
    return hi;
}

// lower_bound by plain binary search (cursor of a part that starts mid-row)
__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ cols, int64_t lo, int64_t hi, int64_t c)
{
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(cols + mid) < c)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

} // namespace

// Optional phase profile (-DKK_SLAB_PROF): lane 0 of every warp adds clock
// deltas and event counts; read with spg_debug_slab_prof.
#ifdef KK_SLAB_PROF
__device__ unsigned long long g_slab_prof[64];
#define PROF_DECL unsigned long long prof_t = clock64();
#define PROF_MARK(idx)                                                                                   \
    do {                                                                                                 \
        if (lane == 0) {                                                                                 \
            const unsigned long long now = clock64();                                                    \
            atomicAdd(&g_slab_prof[idx], now - prof_t);                                                  \
            prof_t = now;                                                                                \
        }                                                                                                \
    } while (0)
#define PROF_COUNT(idx, n)                                                                               \
    do {                                                                                                 \
        if (lane == 0)                                                                                   \
            atomicAdd(&g_slab_prof[idx], (unsigned long long)(n));                                       \
    } while (0)
#else
#define PROF_DECL
#define PROF_MARK(idx)
#define PROF_COUNT(idx, n)
#endif

struct SlabArgs {
    const int4* items;  // {row, part, parts, split slot}
    int64_t n_items;
    unsigned char* scratch; // per warp: cursor state of up to max_a_row A entries
    int64_t max_a_row;
    int64_t k;          // column domain
    const int64_t* prf; // per-row flops (first slab's keys-per-product ratio), may be null
    unsigned long long* split_out;  // per split row: output entries reserved so far
    unsigned int* split_done;       // per split row: parts finished
};

// per-warp scratch: a cursor per A entry (one 16-byte load per lane) and the
// run list of the slab being planned (non-empty runs in A order)
struct __align__(16) Cursor {
    int64_t pos; // next unconsumed B position
    int32_t rem; // B entries left in the row from pos
    int32_t nxt; // column at pos (INT_MAX when none)
};

struct WarpScratch {
    Cursor* cur;
    int64_t* rs;  // run start (B position)
    double* ra;   // A value of the run
    int32_t* rl;  // run length
    int32_t* rp;  // A entry of the run
    int32_t* rnx; // column after the run (the entry's next cursor column)
};

constexpr size_t kScratchPerEntry = 16 + 8 + 8 + 4 + 4 + 4; // 44 B; max_a_row is a multiple of 4

__device__ __forceinline__ WarpScratch warp_scratch(unsigned char* base, int64_t n)
{
    WarpScratch w;
    w.cur = reinterpret_cast<Cursor*>(base);
    w.rs = reinterpret_cast<int64_t*>(w.cur + n);
    w.ra = reinterpret_cast<double*>(w.rs + n);
    w.rl = reinterpret_cast<int32_t*>(w.ra + n);
    w.rp = w.rl + n;
    w.rnx = w.rp + n;
    return w;
}

// shared memory per warp: the table and the slots its keys occupy (for an
// O(keys) emission)
constexpr int kQueue = 64; // plan queue ring (entries with a run in the slab)
struct __align__(16) WarpSmem {
    int32_t keys[kTW];
    double vals[kTW];
    int64_t qpos[kQueue];
    int32_t qrem[kQueue];
    int32_t qp[kQueue];
    uint16_t used[kTWMax + 32];
};

// Fold one 32-product window into the warp table.  kDistinct: the window's
// keys are distinct (all from one run).  New keys get their slot recorded in
// used[nk...]; nk advances.
template <bool kDistinct>
__device__ __forceinline__ void fold(bool valid, int32_t key, double v, WarpSmem& t, int& nk, int lane)
{
    uint32_t grp = 0;
    bool leader = valid;
    if constexpr (!kDistinct) {
        grp = __match_any_sync(kFull, valid ? key : (-1 - lane));
        leader = valid && (__ffs(grp) - 1) == lane;
    }
    uint32_t slot = 0;
    bool is_new = false;
    if (leader) {
        slot = key_slot(key);
        for (;;) {
            const int32_t kx = t.keys[slot];
            if (kx == key)
                break;
            if (kx == kEmpty) {
                const int32_t old = atomicCAS(&t.keys[slot], kEmpty, key);
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
    double acc = v;
    if (leader && !is_new)
        acc = __dadd_rn(t.vals[slot], v);
    if constexpr (!kDistinct) {
        // the rest of the group in lane order: ((acc + v2) + v3) ...
        uint32_t rest = leader ? (grp & (grp - 1)) : 0u;
        const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
        for (int rr = 0; rr < rounds; ++rr) {
            const int src = rest ? __ffs(rest) - 1 : lane;
            const double xv = __shfl_sync(kFull, v, src);
            if (rest) {
                acc = __dadd_rn(acc, xv);
                rest &= rest - 1;
            }
        }
    }
    if (leader)
        t.vals[slot] = acc;
    const uint32_t nm = __ballot_sync(kFull, is_new);
    if (is_new) {
        const int q = nk + __popc(nm & lanemask_lt());
        if (q < kTWMax + 32)
            t.used[q] = static_cast<uint16_t>(slot);
    }
    nk += __popc(nm);
    __syncwarp();
}

__global__ void __launch_bounds__(kWarps * 32, KK_SLAB_CTAS) numeric_wslab_kernel(const RowLaunch L, const SlabArgs S)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem& tab = reinterpret_cast<WarpSmem*>(smem_raw)[wib];
    const int64_t gw = (int64_t)blockIdx.x * kWarps + wib;
    const WarpScratch ws = warp_scratch(S.scratch + (size_t)gw * S.max_a_row * kScratchPerEntry, S.max_a_row);
    const uint64_t pol = l2_keep_policy();
    for (int t = lane; t < kTW; t += 32)
        tab.keys[t] = kEmpty;
    __syncwarp();
    PROF_DECL

    for (;;) {
        unsigned long long itu = 0;
        if (lane == 0)
            itu = atomicAdd(&L.ctr->next_row[0], 1ull);
        const int64_t it = static_cast<int64_t>(__shfl_sync(kFull, itu, 0));
        if (it >= S.n_items)
            break;
        const int4 item = S.items[it];
        const int32_t i = item.x, part = item.y, parts = item.z, slot = item.w;
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int64_t cap = __ldg(L.c_rowptr + i + 1) - cbase;
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        const int64_t d = aend - abeg;
        if (d > S.max_a_row) { // plan / operand mismatch: the cursors would not fit
            if (lane == 0)
                raise_error(L.ctr, kDevRowOverflow);
            continue;
        }
        const int64_t C_lo = S.k * part / parts, C_hi = S.k * (part + 1) / parts;
#ifdef KK_SLAB_PROF
        const unsigned long long item_t0 = clock64();
        const int dcls = d <= 1 ? 0 : min(15, 64 - __clzll(static_cast<unsigned long long>(d - 1)));
#endif
        // ---- cursors at the part's first column ----
        for (int64_t p0 = 0; p0 < d; p0 += 32) {
            const int64_t p = p0 + lane;
            if (p < d) {
                const int32_t j = __ldg(L.a_cols + abeg + p);
                const int64_t bs = __ldg(L.b_rowptr + j), be = __ldg(L.b_rowptr + j + 1);
                const int64_t c0 = C_lo == 0 ? bs : lower_bound_col(L.b_cols, bs, be, C_lo);
                Cursor c;
                c.pos = c0;
                c.rem = static_cast<int32_t>(be - c0);
                c.nxt = c0 < be ? __ldg(L.b_cols + c0) : INT_MAX;
                ws.cur[p] = c;
            }
        }
        __syncwarp();
        PROF_MARK(0);
        const int64_t row_flops = S.prf ? __ldg(S.prf + i) : 0;
        double ratio = row_flops > 0 ? static_cast<double>(cap) / static_cast<double>(row_flops) : 1.0;
        int64_t W = imax64(1, static_cast<int64_t>(static_cast<double>(kX) * static_cast<double>(S.k) /
                                                   fmax(static_cast<double>(cap), 1.0)));
        int64_t c_lo = C_lo, emitted = 0;
        bool bad = false;
        int replans = 0;
        while (c_lo < C_hi && !bad) {
            const int64_t c_hi = W >= C_hi - c_lo ? C_hi : c_lo + W;
            // ---- plan: runs of every A entry in [c_lo, c_hi).  Cursors are
            //      scanned 32 at a time (two groups ahead in flight); the
            //      entries with a run here are queued in A order, and run ends
            //      are searched 32 queued entries at a time, every lane busy ----
            int64_t prods = 0;
            int32_t nr = 0;
            int qh = 0, qn = 0; // queue ring [qh, qh + qn) mod kQueue
            auto search = [&](int cnt) {
                const bool act = lane < cnt;
                int64_t pos = 0;
                int32_t rem = 0, p = 0;
                if (act) {
                    const int q = (qh + lane) & (kQueue - 1);
                    pos = tab.qpos[q];
                    rem = tab.qrem[q];
                    p = tab.qp[q];
                }
                Probe16 P;
                probe16(L.b_cols, pos, pos + rem, P);
                const double av = act ? __ldg(L.a_vals + abeg + p) : 0.0;
                if (act) {
                    int32_t x = INT_MAX;
                    const int64_t e = finish16(L.b_cols, pos, pos + rem, c_hi, P, &x);
                    const int r = nr + lane;
                    ws.rs[r] = pos;
                    ws.ra[r] = av;
                    ws.rl[r] = static_cast<int32_t>(e - pos);
                    ws.rp[r] = p;
                    ws.rnx[r] = x;
                    prods += e - pos;
                }
                nr += cnt;
                qh = (qh + cnt) & (kQueue - 1);
                qn -= cnt;
            };
            Cursor f1{0, 0, INT_MAX}, f2{0, 0, INT_MAX};
            if (lane < d)
                f1 = ws.cur[lane];
            if (32 + lane < d)
                f2 = ws.cur[32 + lane];
            for (int64_t p0 = 0; p0 < d; p0 += 32) {
                const int64_t p = p0 + lane;
                const Cursor c = f1;
                f1 = f2;
                f2 = Cursor{0, 0, INT_MAX};
                if (p + 64 < d)
                    f2 = ws.cur[p + 64];
                const bool na = c.nxt < c_hi; // past-the-end lanes: nxt INT_MAX
                bad = bad || (na && c.nxt < c_lo); // an earlier run ended early: unsorted B row
                const uint32_t M = __ballot_sync(kFull, na);
                if (na) {
                    const int q = (qh + qn + __popc(M & lanemask_lt())) & (kQueue - 1);
                    tab.qpos[q] = c.pos;
                    tab.qrem[q] = c.rem;
                    tab.qp[q] = static_cast<int32_t>(p);
                }
                qn += __popc(M);
                __syncwarp();
                if (qn >= 32) {
                    search(32);
                    __syncwarp();
                }
            }
            if (qn > 0)
                search(qn);
            __syncwarp();
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1)
                prods += __shfl_xor_sync(kFull, prods, o);
            PROF_COUNT(14, nr);
            PROF_COUNT(15, d);
            if (__any_sync(kFull, bad)) {
                bad = true;
                break;
            }
            __syncwarp();
            PROF_MARK(1);
            if (replans < 2) {
                // keys this slab will hold, predicted from its products: resize
                // before any product is folded
                const double est = static_cast<double>(prods) * ratio;
                const int64_t w = c_hi - c_lo;
                bool replan = false;
                if (est > KK_SLAB_ACCEPT * kX && w > 1) {
                    W = imax64(1, static_cast<int64_t>(w * (0.9 * kX / est)));
                    replan = true;
                    PROF_COUNT(12, 1);
                } else if (est < 0.2 * kX && c_hi < C_hi) {
                    W = static_cast<int64_t>(w * fmin(8.0, 0.6 * kX / fmax(est, 1.0))) + 1;
                    replan = true;
                    PROF_COUNT(13, 1);
                }
                if (replan) {
                    ++replans;
                    PROF_COUNT(10, 1);
                    continue;
                }
            }
            // ---- fold the runs in A order: batches of 32 runs, windows of 32
            //      products; the next window's loads (across batch boundaries)
            //      are in flight while a window folds ----
            int nk = 0;
            bool ovf = false, low = false; // low: a column below c_lo (unsorted B row)
            struct Batch {
                int64_t cb; // this lane's run: B start
                double ca;  //                A value
                int32_t ce; //                start in the batch's flat index
                int32_t total, nb, rank;
            };
            auto fetch = [&](int32_t r0, int64_t& s0, int32_t& l0, double& a0) {
                s0 = 0;
                l0 = 0;
                a0 = 0.0;
                if (r0 + lane < nr) {
                    s0 = ws.rs[r0 + lane];
                    l0 = ws.rl[r0 + lane];
                    a0 = ws.ra[r0 + lane];
                }
            };
            auto make = [&](int32_t r0, int64_t s0, int32_t l0, double a0) {
                Batch B;
                int32_t incl = l0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o)
                        incl += y;
                }
                B.cb = s0;
                B.ca = a0;
                B.ce = incl - l0;
                B.total = __shfl_sync(kFull, incl, 31);
                B.nb = nr - r0 < 32 ? nr - r0 : 32;
                B.rank = 0;
                return B;
            };
            // window w0 of batch B -> this lane's (key, B value, A value)
            auto map = [&](Batch& B, int32_t w0, int32_t& key, double& bv, double& a, bool& single) {
                const uint32_t bit = (lane < B.nb && B.ce >= w0 && B.ce < w0 + 32) ? (1u << (B.ce - w0)) : 0u;
                const uint32_t M = __reduce_or_sync(kFull, bit);
                int seg = B.rank + __popc(M & ((2u << lane) - 1u)) - 1;
                seg = seg < 0 ? 0 : (seg > 31 ? 31 : seg);
                const int32_t e = __shfl_sync(kFull, B.ce, seg);
                const int64_t base = __shfl_sync(kFull, B.cb, seg);
                a = __shfl_sync(kFull, B.ca, seg);
                B.rank += __popc(M);
                single = M == 0 || M == 1; // every lane in one run: distinct keys
                const int32_t t = w0 + lane;
                key = -1;
                bv = 0.0;
                if (t < B.total) {
                    key = ldg_keep(L.b_cols + base + (t - e), pol);
                    bv = ldg_keep(L.b_vals + base + (t - e), pol);
                }
            };
            if (nr > 0) {
                // window producer: batch pb at window offset pw0 (pn made, the
                // run data of the batch after it in flight); the consumer
                // keeps two mapped windows ahead of the one it folds
                int64_t s0, s1, s2;
                int32_t l0, l1, l2;
                double a0, a1, a2;
                fetch(0, s0, l0, a0);
                fetch(32, s1, l1, a1);
                fetch(64, s2, l2, a2);
                Batch pb = make(0, s0, l0, a0);
                Batch pn = make(32, s1, l1, a1);
                int32_t pr0 = 0, pw0 = 0;
                auto produce = [&](int32_t& k, double& b, double& av, bool& sg) -> bool {
                    if (pw0 >= pb.total) {
                        if (pr0 + 32 >= nr)
                            return false;
                        pr0 += 32;
                        pw0 = 0;
                        pb = pn; // not mapped yet (rank 0)
                        pn = make(pr0 + 32, s2, l2, a2);
                        fetch(pr0 + 64, s2, l2, a2);
                    }
                    map(pb, pw0, k, b, av, sg); // key -1 past the batch's products
                    pw0 += 32;
                    return true;
                };
                // ring of kDepth + 1 windows: [0] is folded, [1..kDepth] in flight
                int32_t wk[kDepth + 1];
                double wb[kDepth + 1], wx[kDepth + 1];
                bool wg[kDepth + 1], wh[kDepth + 1];
#pragma unroll
                for (int u = 0; u < kDepth; ++u) {
                    wk[u] = -1;
                    wb[u] = wx[u] = 0.0;
                    wg[u] = true;
                    wh[u] = (u == 0 || wh[u - 1]) && produce(wk[u], wb[u], wx[u], wg[u]);
                }
                while (wh[0]) {
                    wk[kDepth] = -1;
                    wb[kDepth] = wx[kDepth] = 0.0;
                    wg[kDepth] = true;
                    wh[kDepth] = wh[kDepth - 1] && produce(wk[kDepth], wb[kDepth], wx[kDepth], wg[kDepth]);
                    const bool valid = wk[0] >= 0;
                    const double v = __dmul_rn(wx[0], wb[0]);
                    low = low || (valid && wk[0] < c_lo);
                    if (wg[0])
                        fold<true>(valid, wk[0], v, tab, nk, lane);
                    else
                        fold<false>(valid, wk[0], v, tab, nk, lane);
                    if (nk > kTWMax) {
                        ovf = true;
                        break;
                    }
#pragma unroll
                    for (int u = 0; u < kDepth; ++u) {
                        wh[u] = wh[u + 1];
                        wk[u] = wk[u + 1];
                        wb[u] = wb[u + 1];
                        wx[u] = wx[u + 1];
                        wg[u] = wg[u + 1];
                    }
                }
            }
            PROF_MARK(2);
            if (__any_sync(kFull, low)) {
                bad = true;
                break;
            }
            if (ovf) {
                // abandon the slab: clear the table, retry at half width
                for (int t = lane; t < kTW; t += 32)
                    tab.keys[t] = kEmpty;
                __syncwarp();
                W = imax64(1, (c_hi - c_lo) / 2);
                PROF_COUNT(11, 1);
                continue;
            }
            // ---- slab done: advance the cursors of the runs, emit ----
            for (int32_t r = lane; r < nr; r += 32) {
                const int32_t p = ws.rp[r];
                Cursor c = ws.cur[p];
                const int32_t l = ws.rl[r];
                c.pos += l;
                c.rem -= l;
                c.nxt = ws.rnx[r];
                ws.cur[p] = c;
            }
            int64_t base = cbase + emitted;
            if (parts > 1) {
                unsigned long long b = 0;
                if (lane == 0 && nk > 0)
                    b = atomicAdd(&S.split_out[slot], static_cast<unsigned long long>(nk));
                base = cbase + static_cast<int64_t>(__shfl_sync(kFull, b, 0));
            }
            for (int q = lane; q < nk; q += 32) {
                const int sl = tab.used[q];
                const int64_t dst = base + q;
                if (dst < cbase + cap) {
                    st_stream(L.c_cols + dst, tab.keys[sl]);
                    st_stream(L.c_vals + dst, tab.vals[sl]);
                }
                tab.keys[sl] = kEmpty;
            }
            __syncwarp();
            emitted += nk;
            PROF_MARK(3);
            PROF_COUNT(8, 1);
            PROF_COUNT(9, prods);
            // next slab: rescale by the density just seen (at most 4x wider)
            const int64_t w_used = c_hi - c_lo;
            W = nk > 0 ? imax64(1, imin64(4 * w_used, w_used * kX / nk)) : 4 * w_used;
            if (prods > 0)
                ratio = static_cast<double>(nk) / static_cast<double>(prods);
            replans = 0;
            c_lo = c_hi;
        }
        if (bad) {
            for (int t = lane; t < kTW; t += 32)
                tab.keys[t] = kEmpty;
            __syncwarp();
            if (lane == 0)
                raise_error(L.ctr, kDevUnsorted);
            continue;
        }
#ifdef KK_SLAB_PROF
        if (lane == 0) {
            atomicAdd(&g_slab_prof[16 + dcls], clock64() - item_t0);
            atomicAdd(&g_slab_prof[32 + dcls], static_cast<unsigned long long>(emitted));
            atomicAdd(&g_slab_prof[48 + dcls], 1ull);
        }
#endif
        if (lane == 0) {
            if (parts == 1) {
                if (emitted != cap)
                    raise_error(L.ctr, emitted < cap ? kDevRowShort : kDevRowOverflow);
            } else {
                __threadfence();
                if (atomicAdd(&S.split_done[slot], 1u) == static_cast<unsigned>(parts - 1)) {
                    const unsigned long long tot = atomicAdd(&S.split_out[slot], 0ull);
                    if (static_cast<int64_t>(tot) != cap)
                        raise_error(L.ctr, static_cast<int64_t>(tot) < cap ? kDevRowShort : kDevRowOverflow);
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// work items: heavy rows (largest first), long ones cut into column parts
// ---------------------------------------------------------------------------
__global__ void slab_parts_kernel(const int32_t* __restrict__ list, int64_t n, const int64_t* __restrict__ a_rowptr,
                                  const int64_t* __restrict__ c_rowptr, int64_t k, int64_t* __restrict__ sizes)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = list[t];
        const double d = static_cast<double>(a_rowptr[i + 1] - a_rowptr[i]);
        const double cap = static_cast<double>(c_rowptr[i + 1] - c_rowptr[i]);
        int64_t P = static_cast<int64_t>(ceil(d * cap / kSplitWork));
        P = P < 1 ? 1 : (P > 256 ? 256 : P);
        if (P > k)
            P = k > 0 ? k : 1;
        sizes[t + 1] = P; // scanned in place into item offsets
    }
}

__global__ void slab_items_kernel(const int32_t* __restrict__ list, int64_t n, const int64_t* __restrict__ item_off,
                                  int4* __restrict__ items, unsigned long long* split_count)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = item_off[t];
        const int32_t P = static_cast<int32_t>(item_off[t + 1] - o);
        int32_t slot = -1;
        if (P > 1)
            slot = static_cast<int32_t>(atomicAdd(split_count, 1ull));
        for (int32_t q = 0; q < P; ++q)
            items[o + q] = make_int4(list[t], q, P, slot);
    }
}

} // namespace kk

extern "C" int spg_debug_slab_prof(unsigned long long* out, int reset)
{
#ifdef KK_SLAB_PROF
    if (out)
        cudaMemcpyFromSymbol(out, kk::g_slab_prof, sizeof(kk::g_slab_prof));
    if (reset) {
        unsigned long long z[64] = {};
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

size_t slab_scratch_per_entry() { return kScratchPerEntry; }

int numeric_slab_warps()
{
    const void* fn = reinterpret_cast<const void*>(&numeric_wslab_kernel);
    const int smem = static_cast<int>(sizeof(WarpSmem) * kWarps);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kWarps * 32, smem) != cudaSuccess || b < 1)
        b = 1;
    return b * sm_count() * kWarps;
}

int slab_warps_per_cta() { return kWarps; }

// Work items from the sorted heavy-row list.  Pass 1 (items == nullptr):
// item_off[0..n] = exclusive offsets of each row's parts (item_off[n] =
// item count).  Pass 2: items[] and the split-row slots.
cudaError_t build_slab_items(const int32_t* list, int64_t n, const int64_t* a_rowptr, const int64_t* c_rowptr,
                             int64_t k, int64_t* item_off, int4* items, unsigned long long* split_count,
                             cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4);
    if (!items) {
        cudaError_t e = cudaMemsetAsync(item_off, 0, sizeof(int64_t), st);
        if (e != cudaSuccess)
            return e;
        slab_parts_kernel<<<blocks, 256, 0, st>>>(list, n, a_rowptr, c_rowptr, k, item_off);
        count_launch();
        ScanTotals* tot = nullptr;
        e = cudaMallocAsync(&tot, sizeof(ScanTotals), st);
        if (e == cudaSuccess)
            e = cudaMemsetAsync(tot, 0, sizeof(ScanTotals), st);
        if (e == cudaSuccess)
            e = scan_sizes_inplace(item_off, n, tot, st); // exclusive offsets, item_off[n] = total
        if (tot)
            cudaFreeAsync(tot, st);
        if (e != cudaSuccess)
            return e;
    } else {
        slab_items_kernel<<<blocks, 256, 0, st>>>(list, n, item_off, items, split_count);
        count_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_numeric_slab(const RowLaunch& L, const SlabPlan& P, int64_t k, const int64_t* prf,
                                cudaStream_t st)
{
    if (P.n_items <= 0)
        return cudaSuccess;
    const int smem = static_cast<int>(sizeof(WarpSmem) * kWarps);
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_wslab_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
        return e;
    if (P.n_split > 0) {
        e = cudaMemsetAsync(P.split_out, 0, sizeof(unsigned long long) * P.n_split, st);
        if (e == cudaSuccess)
            e = cudaMemsetAsync(P.split_done, 0, sizeof(unsigned int) * P.n_split, st);
        if (e != cudaSuccess)
            return e;
    }
    SlabArgs S{P.items, P.n_items, static_cast<unsigned char*>(P.scratch), P.max_a_row, k, prf, P.split_out,
               P.split_done};
    const int grid = static_cast<int>(std::max<int64_t>(1, P.warps / kWarps));
    numeric_wslab_kernel<<<grid, kWarps * 32, smem, st>>>(L, S);
    count_launch();
    return cudaGetLastError();
}

} // namespace kk
