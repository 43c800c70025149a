// Fast paths of the two row kernels (sm_100a), used by the default (Auto)
// device plan.  Same semantics as the generic row_kernel in kk_kernels.cu —
// the parity tests run both — with the per-product instruction count cut down:
//
// numeric_lp_seq_kernel   Thread-Sequential numeric Gustavson (engine.cpp:259-267)
//     with a linear-probing L1 table in shared memory (keys[T], vals[T] by
//     slot, slot_of[] by first-touch position, Fibonacci hash).  New keys
//     claim slots with one shared CAS (a write-then-verify variant exists,
//     KK_NUM_VERIFY, measured slower).  Per-step scalars of the A chunk are
//     staged in shared memory and B rows of step q+2 are prefetched into
//     registers while step q accumulates.  Positions are assigned in lane
//     (= first-touch) order and values summed left to right with unfused
//     mul/add, so C is bitwise the reference's output.
//
// numeric_lp_flat_kernel  Thread-Flat-Parallel numeric for short B rows: 32-product
//     windows, duplicate keys grouped with __match_any_sync and folded by the
//     lowest lane in lane (= product) order onto the running sum.  Rows are
//     short and latency-bound, so a warp takes 32 rows at a time and
//     pipelines their dependent loads across rows (A entries two rows ahead,
//     B-row descriptors one row ahead).  A row whose products fit one window
//     skips the table: its key groups are the row's keys and the leaders'
//     lane ranks their first-touch positions.
//
// symbolic_flat_kernel    Thread-Flat-Parallel structure union (engine.cpp:268-286
//     with SymbolicSink :210-221) over the compressed graph (or raw columns).
//     The union is order-independent, so duplicate keys inside a 32-product
//     window are resolved with shared-memory CAS/OR instead of a warp fold,
//     and the row size is the popcount of the table (no position bookkeeping).
//     Tables are sized optimistically from the row bound; a row whose probe
//     sequence exceeds kSymMaxProbe (an over-full table) is re-queued to the
//     exact-size path.  A row of at most 32 pairs skips the table (its size
//     comes from the window's key groups).  Chunks of very short
//     compressed rows run as segmented steps (several whole B rows per 32
//     lanes); plans of short rows use the same row pipeline as the flat
//     numeric kernel.
//
// The flattened-window map (FlatMap) compacts a chunk's non-empty segments
// through shared memory and locates each lane's segment from a bitmask of
// segment starts (REDUX.OR + popc) instead of a per-window binary search.
#include <cstdint>
#include <cstdlib>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

// ---------------------------------------------------------------------------
// numeric: LP + Thread-Sequential
// ---------------------------------------------------------------------------
// Slot hash: Fibonacci (multiplicative) hash, linear probing.  (A
// low-bit-preserving hash would keep B-row runs in distinct banks, but on
// n = 160 stencils every run of a C row shares its low 5 bits — the same
// pathology as the reference's key & mask hash, SURVEY §7 — and clusters.)
constexpr uint32_t kProbeStep = 1;
__device__ __forceinline__ uint32_t loc_hash(int32_t key, int shift)
{
    return hash_slot(key, shift);
}

// Claim empty slots for this step's new keys (distinct keys, first probe
// already stopped at an empty slot `s`): write, re-read, losers move to the
// next empty slot.  No shared-memory atomics.
__device__ __forceinline__ uint32_t claim_slots(bool is_new, int32_t key, uint32_t s, int32_t* keys,
                                                uint32_t tmask)
{
    bool pending = is_new;
    for (;;) {
        if (pending)
            keys[s] = key;
        __syncwarp();
        if (pending && keys[s] == key)
            pending = false;
        if (!__any_sync(kFull, pending))
            break;
        if (pending)
            do {
                s = (s + kProbeStep) & tmask;
            } while (keys[s] != kEmpty);
        __syncwarp();
    }
    return s;
}

// one Thread-Sequential step: lanes hold distinct keys of one B row.
// kCas: claim new slots with shared-memory CAS (else write-then-verify).
template <bool kCas>
__device__ __forceinline__ void num_step(bool valid, int32_t key, double v, int32_t* keys, double* vals,
                                         int32_t* slot_of, uint32_t tmask, int shift, int32_t cap,
                                         int32_t& cnt)
{
    uint32_t s = 0;
    bool is_new = false;
    if (valid) {
        s = loc_hash(key, shift);
        int32_t k = keys[s];
        while (k != key && k != kEmpty) {
            s = (s + kProbeStep) & tmask;
            k = keys[s];
        }
        if (k == key) // running sum: ((first + v2) + v3) ...
            vals[s] = __dadd_rn(vals[s], v);
        else
            is_new = true;
    }
    const uint32_t nm = __ballot_sync(kFull, is_new);
    if (nm) {
        // keys beyond the symbolic row size are never inserted (the row is in
        // error, reported at its end): the table keeps free slots, probes end
        const int32_t pos = cnt + __popc(nm & lanemask_lt());
        const bool claim = is_new && pos < cap;
        if constexpr (kCas) {
            if (claim)
                while (atomicCAS(&keys[s], kEmpty, key) != kEmpty)
                    s = (s + kProbeStep) & tmask;
        } else {
            __syncwarp();
            s = claim_slots(claim, key, s, keys, tmask);
        }
        if (claim) {
            vals[s] = v;
            slot_of[pos] = static_cast<int32_t>(s);
        }
        cnt += __popc(nm);
    }
    __syncwarp();
}

// per-warp staging of one A chunk: the step scalars are read back with
// broadcast LDS (one 16-byte {B row offset, length} read for the prefetch of
// step q+2, one 8-byte read of A(i,j) for step q)
struct StepStage {
    longlong2 row[32]; // x = B row offset, y = B row length
    double a[32];
};

template <bool kCas>
__global__ void __launch_bounds__(256) numeric_lp_seq_kernel(const RowLaunch L)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t pol = l2_keep_policy(); // B stays in L2 while C streams out
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* region = smem + (size_t)wib * L.lay.bytes;
    double* vals = reinterpret_cast<double*>(region + L.lay.off_map);
    int32_t* keys = reinterpret_cast<int32_t*>(region + L.lay.off_ids);
    int32_t* slot_of = reinterpret_cast<int32_t*>(region + L.lay.off_aux);
    StepStage* stage = reinterpret_cast<StepStage*>(region + L.lay.off_pay);
    if (L.gate && L.gate[0] == L.gate[2] && L.gate[1] == L.gate[3])
        return; // the slot replay (kk_replay.cu) computed this pass
    const uint32_t tmask = static_cast<uint32_t>(L.lay.T - 1);
    const int shift = L.lay.shift;
    for (int t = lane; t < L.lay.T; t += 32)
        keys[t] = kEmpty;
    __syncwarp();

    const int64_t nwarps = (int64_t)gridDim.x * L.wpb;
    const int64_t* __restrict__ a_rowptr = L.a_rowptr;
    const int32_t* __restrict__ a_cols = L.a_cols;
    const double* __restrict__ a_vals = L.a_vals;
    const int64_t* __restrict__ b_rowptr = L.b_rowptr;

    for (int64_t r = (int64_t)blockIdx.x * L.wpb + wib; r < L.nrows; r += nwarps) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - cbase);
        if (cap == 0)
            continue;
        const int64_t abeg = __ldg(a_rowptr + i), aend = __ldg(a_rowptr + i + 1);
        int32_t cnt = 0;
        for (int64_t p0 = abeg; p0 < aend; p0 += 32) {
            const int na = static_cast<int>(aend - p0 < 32 ? aend - p0 : 32);
            int32_t bl = 0;
            if (lane < na) {
                const int32_t j = __ldg(a_cols + p0 + lane);
                const int64_t b0 = __ldg(b_rowptr + j);
                bl = static_cast<int32_t>(__ldg(b_rowptr + j + 1) - b0);
                stage->row[lane] = make_longlong2(b0, bl);
                stage->a[lane] = __ldg(a_vals + p0 + lane);
            } else {
                stage->row[lane] = make_longlong2(0, 0);
            }
            const bool long_rows = __any_sync(kFull, bl > 32);
            __syncwarp();
            if (long_rows) {
                // B rows longer than a warp: plain stepping
                for (int q = 0; q < na; ++q) {
                    const longlong2 rq = stage->row[q];
                    const int32_t len = static_cast<int32_t>(rq.y);
                    const double a = stage->a[q];
                    for (int32_t t0 = 0; t0 < len; t0 += 32) {
                        const bool valid = t0 + lane < len;
                        int32_t key = 0;
                        double v = 0.0;
                        if (valid) {
                            key = ldg_keep(L.b_cols + rq.x + t0 + lane, pol);
                            v = __dmul_rn(a, ldg_keep(L.b_vals + rq.x + t0 + lane, pol));
                        }
                        num_step<kCas>(valid, key, v, keys, vals, slot_of, tmask, shift, cap, cnt);
                    }
                }
                __syncwarp();
                continue;
            }
            // depth-2 register pipeline over the steps of the chunk (rows of
            // the stage past na have length 0)
            int32_t k0 = 0, k1 = 0, len0, len1;
            double v0 = 0.0, v1 = 0.0;
            {
                const longlong2 r0 = stage->row[0];
                const longlong2 r1 = stage->row[1];
                len0 = static_cast<int32_t>(r0.y);
                len1 = static_cast<int32_t>(r1.y);
                if (lane < len0) {
                    k0 = ldg_keep(L.b_cols + r0.x + lane, pol);
                    v0 = ldg_keep(L.b_vals + r0.x + lane, pol);
                }
                if (lane < len1) {
                    k1 = ldg_keep(L.b_cols + r1.x + lane, pol);
                    v1 = ldg_keep(L.b_vals + r1.x + lane, pol);
                }
            }
            for (int q = 0; q < na; ++q) {
                int32_t k2 = 0, len2 = 0;
                double v2 = 0.0;
                if (q + 2 < 32) {
                    const longlong2 r2 = stage->row[q + 2];
                    len2 = static_cast<int32_t>(r2.y);
                    if (lane < len2) {
                        k2 = ldg_keep(L.b_cols + r2.x + lane, pol);
                        v2 = ldg_keep(L.b_vals + r2.x + lane, pol);
                    }
                }
                num_step<kCas>(lane < len0, k0, __dmul_rn(stage->a[q], v0), keys, vals, slot_of, tmask, shift,
                               cap, cnt);
                k0 = k1;
                v0 = v1;
                len0 = len1;
                k1 = k2;
                v1 = v2;
                len1 = len2;
            }
            __syncwarp();
        }
        if (cnt != cap && lane == 0)
            raise_error(L.ctr, cnt < cap ? kDevRowShort : kDevRowOverflow);
        // flush in first-touch order and clear the table for the next row
        const int32_t used = cnt < cap ? cnt : cap;
        for (int32_t q = lane; q < used; q += 32) {
            const int32_t s = slot_of[q];
            st_stream(L.c_cols + cbase + q, keys[s]);
            st_stream(L.c_vals + cbase + q, vals[s]);
            keys[s] = kEmpty;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Thread-Flat-Parallel index mapping.  For one chunk of <= 32 A entries the
// flattened product index t maps to (segment, offset) = flat_position(prefix, t)
// (engine.cpp:360-365).  Instead of a 5-step shuffle binary search per window,
// the non-empty segments are compacted once per chunk (their starts are then
// strictly increasing) and, per 32-product window, the segment starts falling
// inside the window form a bit mask M: lane x's segment is (segments started
// before the window) + popc(M & lanes<=x) - 1.
// ---------------------------------------------------------------------------
// per-warp scratch for the compaction (shared memory, 640 B)
struct FlatScratch {
    int64_t base[32];
    double a[32];
    int32_t excl[32];
};
static_assert(sizeof(FlatScratch) == 640, "layouts reserve 640 B (symbolic) / 768 B (numeric)");

template <bool kWithA>
struct FlatMap {
    int64_t cbase;  // compacted: lane c holds B-row base - start of the c-th non-empty segment
    double ca;      // ... its A value
    int32_t cexcl;  // ... its start in the flattened index space
    int32_t nne;    // non-empty segments
    int32_t rank;   // non-empty segments starting before the current window
    int32_t total;  // products of the chunk

    // non-empty segments scatter their data to their rank in `sc` and every
    // lane reads back entry `lane` (a shared-memory compaction: cheaper than
    // locating the lane-th set bit of the mask)
    __device__ __forceinline__ void init(int64_t bb, int32_t bl, double av, int lane, FlatScratch* sc)
    {
        int32_t incl = bl;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, incl, off);
            if (lane >= off)
                incl += y;
        }
        const int32_t excl = incl - bl;
        total = __shfl_sync(kFull, incl, 31);
        const uint32_t ne = __ballot_sync(kFull, bl > 0);
        nne = __popc(ne);
        if (bl > 0) {
            const int r = __popc(ne & lanemask_lt());
            sc->base[r] = bb;
            sc->excl[r] = excl;
            if constexpr (kWithA)
                sc->a[r] = av;
        }
        __syncwarp();
        cbase = 0;
        ca = 0.0;
        cexcl = 0;
        if (lane < nne) {
            cexcl = sc->excl[lane];
            cbase = sc->base[lane] - cexcl; // product t of the segment: B position cbase + t
            if constexpr (kWithA)
                ca = sc->a[lane];
        }
        __syncwarp();
        rank = 0;
    }

    // segment data of this lane's product in window [w0, w0+32): the B
    // position of product w0 + lane is pos0 + lane; advances rank
    __device__ __forceinline__ void window(int32_t w0, int lane, int64_t& pos0, double& a)
    {
        const uint32_t bit = (lane < nne && cexcl >= w0 && cexcl < w0 + 32) ? (1u << (cexcl - w0)) : 0u;
        const uint32_t M = __reduce_or_sync(kFull, bit);
        int seg = rank + __popc(M & ((2u << lane) - 1u)) - 1;
        seg = seg < 0 ? 0 : (seg > 31 ? 31 : seg);
        pos0 = __shfl_sync(kFull, cbase, seg) + w0;
        if constexpr (kWithA)
            a = __shfl_sync(kFull, ca, seg);
        rank += __popc(M);
    }
};

// ---------------------------------------------------------------------------
// numeric: LP + Thread-Flat-Parallel (short B rows)
// ---------------------------------------------------------------------------
// One 32-product window of the row's flattened multiplications (engine.cpp:
// 268-286).  Duplicate keys inside the window come from different A entries:
// __match_any_sync groups them, the lowest lane (first touch) probes/claims,
// and folds the group's products in lane (= product) order onto the running
// sum, so values stay the reference's left-to-right sums.
__device__ __forceinline__ void num_window(bool valid, int32_t key, double v, int32_t* keys, double* vals,
                                           int32_t* slot_of, uint32_t tmask, int shift, int32_t cap,
                                           int32_t& cnt, int lane)
{
    const uint32_t grp = __match_any_sync(kFull, valid ? key : (-1 - lane));
    const bool leader = valid && (__ffs(grp) - 1) == lane;
    uint32_t s = 0;
    bool is_new = false;
    double acc = v;
    if (leader) {
        s = loc_hash(key, shift);
        int32_t k = keys[s];
        while (k != key && k != kEmpty) {
            s = (s + kProbeStep) & tmask;
            k = keys[s];
        }
        if (k == key)
            acc = __dadd_rn(vals[s], v);
        else
            is_new = true;
    }
    const uint32_t nm = __ballot_sync(kFull, is_new);
    bool claimed = false;
    if (nm) {
        const int32_t pos = cnt + __popc(nm & lanemask_lt());
        if (is_new && pos < cap) { // beyond the symbolic row size: never inserted
            while (atomicCAS(&keys[s], kEmpty, key) != kEmpty)
                s = (s + kProbeStep) & tmask;
            slot_of[pos] = static_cast<int32_t>(s);
            claimed = true;
        }
        cnt += __popc(nm);
    }
    uint32_t rest = leader ? (grp & (grp - 1)) : 0u;
    const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
    for (int r = 0; r < rounds; ++r) {
        const int src = rest ? __ffs(rest) - 1 : lane;
        const double x = __shfl_sync(kFull, v, src);
        if (rest) {
            acc = __dadd_rn(acc, x);
            rest &= rest - 1;
        }
    }
    if (leader && (!is_new || claimed))
        vals[s] = acc;
    __syncwarp();
}

__global__ void __launch_bounds__(256) numeric_lp_flat_kernel(const RowLaunch L)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t pol = l2_keep_policy(); // B stays in L2 while C streams out
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* region = smem + (size_t)wib * L.lay.bytes;
    double* vals = reinterpret_cast<double*>(region + L.lay.off_map);
    int32_t* keys = reinterpret_cast<int32_t*>(region + L.lay.off_ids);
    int32_t* slot_of = reinterpret_cast<int32_t*>(region + L.lay.off_aux);
    FlatScratch* scratch = reinterpret_cast<FlatScratch*>(region + L.lay.off_pay);
    const uint32_t tmask = static_cast<uint32_t>(L.lay.T - 1);
    const int shift = L.lay.shift;
    for (int t = lane; t < L.lay.T; t += 32)
        keys[t] = kEmpty;
    __syncwarp();

    const int64_t nwarps = (int64_t)gridDim.x * L.wpb;
    const int64_t* __restrict__ b_rowptr = L.b_rowptr;

    // One row's accumulation over a chunk of <= 32 A entries whose B-row
    // descriptors (bb, bl) and A values are already in registers.
    auto chunk = [&](int64_t bb, int32_t bl, double av, int32_t cap, int32_t& cnt, FlatMap<true>* pre = nullptr) {
        // flattened prefix of this chunk's B-row lengths (32-bit: one chunk of
        // a flat-scheme row never holds 2^31 products)
        FlatMap<true> fm;
        if (pre)
            fm = *pre;
        else
            fm.init(bb, bl, av, lane, scratch);
        const int32_t total = fm.total;
        for (int32_t w0 = 0; w0 < total; w0 += 32) {
            const int32_t t = w0 + lane;
            int64_t pos0;
            double a;
            fm.window(w0, lane, pos0, a);
            const bool valid = t < total;
            int32_t key = 0;
            double v = 0.0;
            if (valid) {
                const int64_t q = pos0 + lane;
                key = ldg_keep(L.b_cols + q, pol);
                v = __dmul_rn(a, ldg_keep(L.b_vals + q, pol));
            }
            num_window(valid, key, v, keys, vals, slot_of, tmask, shift, cap, cnt, lane);
        }
    };
    // A row whose products fit one window needs no table: the window's key
    // groups (in lane = product order) are the row's keys, their leaders in
    // lane order the first-touch positions, each group folded left to right.
    auto direct = [&](const FlatMap<true>& fm0, int64_t cbase, int32_t cap) {
        FlatMap<true> fm = fm0;
        int64_t pos0;
        double a;
        fm.window(0, lane, pos0, a);
        const bool valid = lane < fm.total;
        int32_t key = 0;
        double v = 0.0;
        if (valid) {
            const int64_t q = pos0 + lane;
            key = ldg_keep(L.b_cols + q, pol);
            v = __dmul_rn(a, ldg_keep(L.b_vals + q, pol));
        }
        const uint32_t grp = __match_any_sync(kFull, valid ? key : (-1 - lane));
        const bool leader = valid && (__ffs(grp) - 1) == lane;
        double acc = v;
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
        const uint32_t lm = __ballot_sync(kFull, leader);
        const int32_t n = __popc(lm);
        if (n != cap && lane == 0)
            raise_error(L.ctr, n < cap ? kDevRowShort : kDevRowOverflow);
        const int32_t pos = __popc(lm & lanemask_lt());
        if (leader && pos < cap) {
            st_stream(L.c_cols + cbase + pos, key);
            st_stream(L.c_vals + cbase + pos, acc);
        }
    };
    auto finish = [&](int64_t cbase, int32_t cap, int32_t cnt) {
        if (cnt != cap && lane == 0)
            raise_error(L.ctr, cnt < cap ? kDevRowShort : kDevRowOverflow);
        const int32_t used = cnt < cap ? cnt : cap;
        for (int32_t q = lane; q < used; q += 32) {
            const int32_t s = slot_of[q];
            st_stream(L.c_cols + cbase + q, keys[s]);
            st_stream(L.c_vals + cbase + q, vals[s]);
            keys[s] = kEmpty;
        }
        __syncwarp();
    };

    // Rows are taken 32 at a time (one load of their A and C ranges).  Their
    // dependent loads are software-pipelined across rows: while row k
    // accumulates, row k+1's B-row descriptors and row k+2's A entries are in
    // flight (three register sets, unrolled by three, so no in-flight load is
    // copied between registers).  Rows of more than 32 A entries are walked
    // chunk by chunk in place.
    for (int64_t r0 = ((int64_t)blockIdx.x * L.wpb + wib) * 32; r0 < L.nrows; r0 += nwarps * 32) {
        const int nr = static_cast<int>(L.nrows - r0 < 32 ? L.nrows - r0 : 32);
        int64_t rab = 0, rcb = 0;
        int32_t ralen = 0, rcap = 0;
        if (lane < nr) {
            const int32_t i = L.list ? __ldg(L.list + r0 + lane) : static_cast<int32_t>(r0 + lane);
            const bool in_range = !(L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi)); // spg_numeric_rows
            if (in_range) {
                rab = __ldg(L.a_rowptr + i);
                ralen = static_cast<int32_t>(__ldg(L.a_rowptr + i + 1) - rab);
                rcb = __ldg(L.c_rowptr + i);
                rcap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - rcb);
            }
        }
        uint32_t todo = __ballot_sync(kFull, lane < nr && rcap > 0);
        auto pop = [&]() {
            const int q = todo ? __ffs(todo) - 1 : -1;
            todo &= todo - 1;
            return q;
        };
        // stage 1: A entries of row q (short rows only)
        auto s1 = [&](int q, int32_t& j, double& av) {
            j = 0;
            av = 0.0;
            if (q < 0)
                return;
            const int32_t len = __shfl_sync(kFull, ralen, q);
            const int64_t ab = __shfl_sync(kFull, rab, q);
            if (len <= 32 && lane < len) {
                j = __ldg(L.a_cols + ab + lane);
                av = __ldg(L.a_vals + ab + lane);
            }
        };
        // stage 2: B-row descriptors of row q's entries
        auto s2 = [&](int q, int32_t j, int64_t& bb, int32_t& bl) {
            bb = 0;
            bl = 0;
            if (q < 0)
                return;
            const int32_t len = __shfl_sync(kFull, ralen, q);
            if (len <= 32 && lane < len) {
                bb = __ldg(b_rowptr + j);
                bl = static_cast<int32_t>(__ldg(b_rowptr + j + 1) - bb);
            }
        };
        // stage 3: the row itself
        auto s3 = [&](int q, int64_t bb, int32_t bl, double av) {
            const int32_t len = __shfl_sync(kFull, ralen, q);
            const int64_t cb = __shfl_sync(kFull, rcb, q);
            const int32_t cap = __shfl_sync(kFull, rcap, q);
            int32_t cnt = 0;
            if (len <= 32) {
                FlatMap<true> fm;
                fm.init(bb, bl, av, lane, scratch);
                if (fm.total <= 32) {
                    direct(fm, cb, cap);
                    return;
                }
                chunk(bb, bl, av, cap, cnt, &fm);
            } else {
                const int64_t ab = __shfl_sync(kFull, rab, q);
                for (int64_t p0 = ab; p0 < ab + len; p0 += 32) {
                    const int na = static_cast<int>(ab + len - p0 < 32 ? ab + len - p0 : 32);
                    int64_t cbb = 0;
                    int32_t cbl = 0;
                    double cav = 0.0;
                    if (lane < na) {
                        const int32_t jj = __ldg(L.a_cols + p0 + lane);
                        cav = __ldg(L.a_vals + p0 + lane);
                        cbb = __ldg(b_rowptr + jj);
                        cbl = static_cast<int32_t>(__ldg(b_rowptr + jj + 1) - cbb);
                    }
                    chunk(cbb, cbl, cav, cap, cnt);
                }
            }
            finish(cb, cap, cnt);
        };
        int32_t jA, jB, jC;
        double aA, aB, aC;
        int64_t bA = 0, bB = 0, bC = 0;
        int32_t lA = 0, lB = 0, lC = 0;
        int qA = pop(), qB = pop(), qC = -1;
        s1(qA, jA, aA);
        s1(qB, jB, aB);
        s2(qA, jA, bA, lA);
        while (qA >= 0) {
            qC = pop();
            s1(qC, jC, aC);
            s2(qB, jB, bB, lB);
            s3(qA, bA, lA, aA);
            if (qB < 0)
                break;
            qA = pop();
            s1(qA, jA, aA);
            s2(qC, jC, bC, lC);
            s3(qB, bB, lB, aB);
            if (qC < 0)
                break;
            qB = pop();
            s1(qB, jB, aB);
            s2(qA, jA, bA, lA);
            s3(qC, bC, lC, aC);
        }
    }
}

cudaError_t launch_numeric_flat_fast(const RowLaunch& L, cudaStream_t st)
{
    if (L.nrows <= 0 || L.grid <= 0)
        return cudaSuccess;
    const size_t smem = (size_t)L.wpb * L.lay.bytes;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_lp_flat_kernel),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    numeric_lp_flat_kernel<<<L.grid, L.wpb * 32, smem, st>>>(L);
    count_launch();
    return cudaGetLastError();
}

int numeric_flat_fast_blocks_per_sm(int wpb, size_t smem)
{
    const void* fn = reinterpret_cast<const void*>(&numeric_lp_flat_kernel);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, wpb * 32, smem) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

// ---------------------------------------------------------------------------
// symbolic: order-free union, LP table of {key, word} slots
// ---------------------------------------------------------------------------
constexpr int kSymMaxProbe = 32;
template <bool kCompressed, bool kPipe>
__global__ void __launch_bounds__(256) symbolic_flat_kernel(const RowLaunch L, unsigned long long* retry_count,
                                                            int32_t* retry_list)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int2* __restrict__ cpair = cpair_of(L);
    unsigned char* region = smem + (size_t)wib * L.lay.bytes;
    int32_t* keys = reinterpret_cast<int32_t*>(region + L.lay.off_ids);
    uint32_t* words = reinterpret_cast<uint32_t*>(region + L.lay.off_map);
    FlatScratch* scratch = reinterpret_cast<FlatScratch*>(region + L.lay.off_pay);
    const int T = L.lay.T;
    const uint32_t tmask = static_cast<uint32_t>(T - 1);
    const int pshift = L.lay.shift;
    const int maxp = T < kSymMaxProbe ? T : kSymMaxProbe;
    for (int t = lane; t < T; t += 32) {
        keys[t] = kEmpty;
        words[t] = 0u;
    }
    __syncwarp();

    const int64_t nwarps = (int64_t)gridDim.x * L.wpb;
    const int64_t* __restrict__ b_rowptr = L.b_rowptr;
    bool overflow = false; // the current row's table filled up

    // one chunk of <= 32 A entries of the current row, B-row descriptors in registers
    auto chunk = [&](int na, int64_t bb, int32_t bl) {
            // probe / claim / OR one (key, word); false when the probe sequence
            // exceeds kSymMaxProbe slots (the table is over-full: the row's size
            // was underestimated) — the row is then handed to the exact-size
            // path.  No per-window claim count is needed.
            auto insert = [&](int32_t key, uint32_t word) -> bool {
                if (key == kEmpty)
                    return true;
                uint32_t s = loc_hash(key, pshift);
                for (int probes = 0; probes < maxp; ++probes) {
                    const int32_t k = keys[s];
                    bool hit = k == key;
                    if (k == kEmpty) {
                        const int32_t old = atomicCAS(&keys[s], kEmpty, key);
                        hit = old == kEmpty || old == key;
                    }
                    if (hit) {
                        if constexpr (kCompressed)
                            atomicOr(&words[s], word);
                        return true;
                    }
                    s = (s + kProbeStep) & tmask;
                }
                return false;
            };
            auto full = [&](bool ok) { return __any_sync(kFull, !ok); };
            auto load = [&](int64_t q, int32_t& key, uint32_t& word) {
                if constexpr (kCompressed) {
                    const int2 pr = __ldg(cpair + q);
                    key = pr.x;
                    word = static_cast<uint32_t>(pr.y);
                } else {
                    key = __ldg(L.b_cols + q);
                    word = 1u;
                }
            };
            const int32_t maxbl = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<unsigned>(bl)));
            const int lg = maxbl <= 1 ? 0 : 32 - __clz(maxbl - 1);
            const int G = 32 >> lg;
            const int32_t csum = static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<unsigned>(bl)));
            if (!L.no_segments && maxbl <= 16 && ((na + G - 1) >> (5 - lg)) <= ((csum + 31) >> 5)) {
                // short (compressed) B rows: segmented steps — G = 32/Lw B rows
                // per step, Lw = pow2 >= the longest, lane = (row, entry); the
                // union is order-free, so no flattened-index mapping is needed.
                // Taken when it needs no more steps than 32-product windows.
                const int sub = lane >> lg;
                const int t = lane & ((1 << lg) - 1);
                auto sfetch = [&](int q0, int32_t& key, uint32_t& word) {
                    const int q = q0 + sub;
                    const int qs = q < 32 ? q : 31;
                    const int64_t b = __shfl_sync(kFull, bb, qs);
                    const int32_t l = __shfl_sync(kFull, bl, qs);
                    key = kEmpty;
                    word = 0u;
                    if (q < na && t < l)
                        load(b + t, key, word);
                };
                int32_t nkey;
                uint32_t nword;
                sfetch(0, nkey, nword);
                for (int q0 = 0; q0 < na; q0 += G) {
                    const int32_t key = nkey;
                    const uint32_t word = nword;
                    if (q0 + G < na)
                        sfetch(q0 + G, nkey, nword);
                    if (full(insert(key, word))) {
                        overflow = true;
                        break;
                    }
                }
                return;
            }
            FlatMap<false> fm;
            fm.init(bb, bl, 0.0, lane, scratch);
            const int32_t total = fm.total;
            // window w0's (key, word) are loaded one window ahead
            auto fetch = [&](int32_t w0, int32_t& key, uint32_t& word) {
                const int32_t t = w0 + lane;
                int64_t pos0;
                double a_unused;
                fm.window(w0, lane, pos0, a_unused);
                key = kEmpty;
                word = 0u;
                if (t < total)
                    load(pos0 + lane, key, word);
            };
            int32_t nkey;
            uint32_t nword;
            fetch(0, nkey, nword);
            for (int32_t w0 = 0; w0 < total; w0 += 32) {
                const int32_t key = nkey;
                const uint32_t word = nword;
                if (w0 + 32 < total)
                    fetch(w0 + 32, nkey, nword);
                if (full(insert(key, word))) {
                    overflow = true;
                    break;
                }
            }
    };
    // A row of at most 32 (key, word) pairs needs no table: the window's key
    // groups are its distinct keys (size = their count, or the popcount of
    // each group's OR).  Returns -1 when the row has more pairs.
    auto direct_size = [&](int64_t bb, int32_t bl) -> int64_t {
        const int32_t csum = static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<unsigned>(bl)));
        if (csum > 32)
            return -1;
        FlatMap<false> fm;
        fm.init(bb, bl, 0.0, lane, scratch);
        int64_t pos0;
        double a_unused;
        fm.window(0, lane, pos0, a_unused);
        const bool valid = lane < csum;
        int32_t key = 0;
        uint32_t word = 0u;
        if (valid) {
            if constexpr (kCompressed) {
                const int2 pr = __ldg(cpair + pos0 + lane);
                key = pr.x;
                word = static_cast<uint32_t>(pr.y);
            } else {
                key = __ldg(L.b_cols + pos0 + lane);
            }
        }
        const uint32_t grp = __match_any_sync(kFull, valid ? key : (-1 - lane));
        const bool leader = valid && (__ffs(grp) - 1) == lane;
        if constexpr (!kCompressed) {
            return __popc(__ballot_sync(kFull, leader));
        } else {
            uint32_t orv = word;
            uint32_t rest = leader ? (grp & (grp - 1)) : 0u;
            const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
            for (int rr = 0; rr < rounds; ++rr) {
                const int src = rest ? __ffs(rest) - 1 : lane;
                const uint32_t x = __shfl_sync(kFull, word, src);
                if (rest) {
                    orv |= x;
                    rest &= rest - 1;
                }
            }
            return __reduce_add_sync(kFull, leader ? static_cast<unsigned>(__popc(orv)) : 0u);
        }
    };
    // size of the finished row (or its hand-off to the L2 path); table reset
    auto finish = [&](int32_t i) {
        __syncwarp();
        int64_t size = 0;
        for (int t = lane; t < T; t += 32) {
            if (keys[t] != kEmpty) {
                size += kCompressed ? __popc(words[t]) : 1;
                keys[t] = kEmpty;
                words[t] = 0u;
            }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            size += __shfl_xor_sync(kFull, size, off);
        if (lane == 0) {
            if (overflow)
                retry_list[atomicAdd(retry_count, 1ull)] = i;
            else
                L.sym_sizes[i] = size;
        }
        __syncwarp();
        overflow = false;
    };

    if constexpr (!kPipe) {
        // rows with many products: one row at a time
        for (int64_t r = (int64_t)blockIdx.x * L.wpb + wib; r < L.nrows; r += nwarps) {
            const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
            const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
            for (int64_t p0 = abeg; p0 < aend && !overflow; p0 += 32) {
                const int na = static_cast<int>(aend - p0 < 32 ? aend - p0 : 32);
                int64_t bb = 0;
                int32_t bl = 0;
                if (lane < na) {
                    const int32_t j = __ldg(L.a_cols + p0 + lane);
                    bb = __ldg(b_rowptr + j);
                    bl = kCompressed ? __ldg(L.csize + j) : static_cast<int32_t>(__ldg(b_rowptr + j + 1) - bb);
                }
                if (aend - abeg <= 32) {
                    const int64_t sz = direct_size(bb, bl);
                    if (sz >= 0) {
                        if (lane == 0)
                            L.sym_sizes[i] = sz;
                        goto next_row;
                    }
                }
                chunk(na, bb, bl);
            }
            finish(i);
        next_row:;
        }
        // (the pipelined short-row loop below is the kPipe instantiation)
    } else {
        // Short rows: taken 32 at a time and their dependent loads pipelined
        // across rows (A entries two rows ahead, B-row descriptors one ahead;
        // three register sets unrolled by three), as in numeric_lp_flat_kernel.
        for (int64_t r0 = ((int64_t)blockIdx.x * L.wpb + wib) * 32; r0 < L.nrows; r0 += nwarps * 32) {
            const int nr = static_cast<int>(L.nrows - r0 < 32 ? L.nrows - r0 : 32);
            int32_t rrow = 0, ralen = 0;
            int64_t rab = 0;
            if (lane < nr) {
                rrow = L.list ? __ldg(L.list + r0 + lane) : static_cast<int32_t>(r0 + lane);
                rab = __ldg(L.a_rowptr + rrow);
                ralen = static_cast<int32_t>(__ldg(L.a_rowptr + rrow + 1) - rab);
            }
            uint32_t todo = nr == 32 ? kFull : ((1u << nr) - 1u);
            auto pop = [&]() {
                const int q = todo ? __ffs(todo) - 1 : -1;
                todo &= todo - 1;
                return q;
            };
            auto s1 = [&](int q, int32_t& j) {
                j = 0;
                if (q < 0)
                    return;
                const int32_t len = __shfl_sync(kFull, ralen, q);
                const int64_t ab = __shfl_sync(kFull, rab, q);
                if (len <= 32 && lane < len)
                    j = __ldg(L.a_cols + ab + lane);
            };
            auto s2 = [&](int q, int32_t j, int64_t& bb, int32_t& bl) {
                bb = 0;
                bl = 0;
                if (q < 0)
                    return;
                const int32_t len = __shfl_sync(kFull, ralen, q);
                if (len <= 32 && lane < len) {
                    bb = __ldg(b_rowptr + j);
                    bl = kCompressed ? __ldg(L.csize + j) : static_cast<int32_t>(__ldg(b_rowptr + j + 1) - bb);
                }
            };
            auto s3 = [&](int q, int64_t bb, int32_t bl) {
                const int32_t len = __shfl_sync(kFull, ralen, q);
                const int32_t i = __shfl_sync(kFull, rrow, q);
                if (len <= 32) {
                    const int64_t sz = direct_size(bb, bl);
                    if (sz >= 0) {
                        if (lane == 0)
                            L.sym_sizes[i] = sz;
                        return;
                    }
                    chunk(len, bb, bl);
                } else {
                    const int64_t ab = __shfl_sync(kFull, rab, q);
                    for (int64_t p0 = ab; p0 < ab + len && !overflow; p0 += 32) {
                        const int na = static_cast<int>(ab + len - p0 < 32 ? ab + len - p0 : 32);
                        int64_t cbb = 0;
                        int32_t cbl = 0;
                        if (lane < na) {
                            const int32_t jj = __ldg(L.a_cols + p0 + lane);
                            cbb = __ldg(b_rowptr + jj);
                            cbl = kCompressed ? __ldg(L.csize + jj) : static_cast<int32_t>(__ldg(b_rowptr + jj + 1) - cbb);
                        }
                        chunk(na, cbb, cbl);
                    }
                }
                finish(i);
            };
            int32_t jA, jB, jC;
            int64_t bA = 0, bB = 0, bC = 0;
            int32_t lA = 0, lB = 0, lC = 0;
            int qA = pop(), qB = pop(), qC = -1;
            s1(qA, jA);
            s1(qB, jB);
            s2(qA, jA, bA, lA);
            while (qA >= 0) {
                qC = pop();
                s1(qC, jC);
                s2(qB, jB, bB, lB);
                s3(qA, bA, lA);
                if (qB < 0)
                    break;
                qA = pop();
                s1(qA, jA);
                s2(qC, jC, bC, lC);
                s3(qB, bB, lB);
                if (qC < 0)
                    break;
                qB = pop();
                s1(qB, jB);
                s2(qA, jA, bA, lA);
                s3(qC, bC, lC);
            }
        }
    }
}

// ---------------------------------------------------------------------------
cudaError_t launch_numeric_fast(const RowLaunch& L, cudaStream_t st)
{
    if (L.nrows <= 0 || L.grid <= 0)
        return cudaSuccess;
    const size_t smem = (size_t)L.wpb * L.lay.bytes;
    const bool cas = getenv("KK_NUM_VERIFY") == nullptr; // CAS claims by default (measured faster)
    const void* fn = cas ? reinterpret_cast<const void*>(&numeric_lp_seq_kernel<true>)
                         : reinterpret_cast<const void*>(&numeric_lp_seq_kernel<false>);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    if (cas)
        numeric_lp_seq_kernel<true><<<L.grid, L.wpb * 32, smem, st>>>(L);
    else
        numeric_lp_seq_kernel<false><<<L.grid, L.wpb * 32, smem, st>>>(L);
    count_launch();
    return cudaGetLastError();
}

int numeric_fast_blocks_per_sm(int wpb, size_t smem)
{
    const void* fn = reinterpret_cast<const void*>(&numeric_lp_seq_kernel<false>);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_lp_seq_kernel<true>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, wpb * 32, smem) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

namespace {
const void* symbolic_flat_fn(bool compressed, bool pipe)
{
    return compressed ? (pipe ? reinterpret_cast<const void*>(&symbolic_flat_kernel<true, true>)
                              : reinterpret_cast<const void*>(&symbolic_flat_kernel<true, false>))
                      : (pipe ? reinterpret_cast<const void*>(&symbolic_flat_kernel<false, true>)
                              : reinterpret_cast<const void*>(&symbolic_flat_kernel<false, false>));
}
} // namespace

cudaError_t launch_symbolic_fast(const RowLaunch& L, bool compressed, bool pipe, unsigned long long* retry_count,
                                 int32_t* retry_list, cudaStream_t st)
{
    if (L.nrows <= 0 || L.grid <= 0)
        return cudaSuccess;
    const size_t smem = (size_t)L.wpb * L.lay.bytes;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(symbolic_flat_fn(compressed, pipe),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    RowLaunch Lx = L;
    Lx.no_segments = getenv("KK_SYM_NOSEG") != nullptr;
    if (compressed && pipe)
        symbolic_flat_kernel<true, true><<<L.grid, L.wpb * 32, smem, st>>>(Lx, retry_count, retry_list);
    else if (compressed)
        symbolic_flat_kernel<true, false><<<L.grid, L.wpb * 32, smem, st>>>(Lx, retry_count, retry_list);
    else if (pipe)
        symbolic_flat_kernel<false, true><<<L.grid, L.wpb * 32, smem, st>>>(Lx, retry_count, retry_list);
    else
        symbolic_flat_kernel<false, false><<<L.grid, L.wpb * 32, smem, st>>>(Lx, retry_count, retry_list);
    count_launch();
    return cudaGetLastError();
}

int symbolic_fast_blocks_per_sm(bool compressed, bool pipe, int wpb, size_t smem)
{
    const void* fn = symbolic_flat_fn(compressed, pipe);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, wpb * 32, smem) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

} // namespace kk
