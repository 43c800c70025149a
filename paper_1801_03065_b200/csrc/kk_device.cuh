// Device building blocks of the kkSpGEMM hot path for sm_100a.
//
// Row-private accumulation follows Alg. 3 of the paper and
// the reference's process_row (src/engine.cpp:251-290): one warp owns one row
// of C; work items are either one B row at a time (Thread-Sequential,
// engine.cpp:259-267) or a 32-product window of the row's flattened
// multiplications (Thread-Flat-Parallel, engine.cpp:268-286, mapped through
// the same upper_bound as flat_position engine.cpp:360-365).
//
// Determinism contract: keys receive positions in first-touch
// order ((A-row position, B-row position) order, the order the reference's
// accumulators' for_each reports), and each value is the left-to-right sum of
// its products starting from the first one, with unfused multiply and add.
// Within a Thread-Sequential step keys are distinct (one B row), so no value
// update needs an atomic; in a Flat window duplicate keys are grouped with
// __match_any_sync and the group leader folds them in lane (= product) order.
// The output is therefore bitwise identical to the reference's raw output.
#pragma once

#include <cstdint>
#include <type_traits>

namespace kk {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int32_t kEmpty = -1;

// device error codes (mapped to the C ABI's status codes on the host)
enum DevError : int {
    kDevOk = 0,
    kDevRowOverflow = 1,  // numeric row exceeds the symbolic structure (engine.cpp:238-239)
    kDevRowShort = 2,     // numeric row shorter than the structure (engine.cpp:244-245)
    kDevKeyRange = 3,     // key outside the dense domain (accumulators.hpp:308-309)
    kDevL2Overflow = 4,   // level-2 bound violated (engine.cpp:83-84)
    kDevReplay = 5,       // slot-replay map does not match the structure (kk_replay.cu)
    kDevUnsorted = 6,     // column-slab path met a B row that is not column-sorted (kk_slab.cu)
};

struct DevCounters {
    unsigned long long pool_allocations;
    unsigned long long l2_inserts;
    int error;
    int pad;
    unsigned long long next_row[2]; // heavy numeric launches: dynamic row queue heads
};

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void raise_error(DevCounters* c, int code)
{
    atomicCAS(&c->error, 0, code);
}

// ---- cache policy for the numeric kernels ------------------------------------
// B rows are re-read by every A row that references them (27 times on a 3D
// stencil) within a short window of rows, while C (6 GB on config 2) is
// written once: B's loads carry an L2 evict_last hint and C's stores are
// streaming (evict-first), so the C stream does not push B's working band out
// of L2.  -DKK_NO_CACHE_HINTS builds the plain variant (A/B measurements).
#ifndef KK_NO_CACHE_HINTS
__device__ __forceinline__ uint64_t l2_keep_policy()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ldg_keep(const int32_t* ptr, uint64_t pol)
{
    int32_t v;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ double ldg_keep(const double* ptr, uint64_t pol)
{
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
}
template <class T> __device__ __forceinline__ void st_stream(T* p, T v) { __stcs(p, v); }
#else
__device__ __forceinline__ uint64_t l2_keep_policy() { return 0; }
__device__ __forceinline__ int32_t ldg_keep(const int32_t* ptr, uint64_t) { return __ldg(ptr); }
__device__ __forceinline__ double ldg_keep(const double* ptr, uint64_t) { return __ldg(ptr); }
template <class T> __device__ __forceinline__ void st_stream(T* p, T v) { *p = v; }
#endif

// Multiplicative (Fibonacci) hash.  The reference hashes with key & mask
// (accumulators.hpp:92,197), which degenerates on stencils (10-27 probes per
// insert); the accumulated sets and values do not depend on it.
__device__ __forceinline__ uint32_t hash_slot(int32_t key, int shift)
{
    return (static_cast<uint32_t>(key) * 0x9E3779B1u) >> shift;
}

// ---- row sources (engine.cpp:32-60) ------------------------------------------
struct NumericSource { // NumericSource: payload a_val * b.values[t]
    using Payload = double;
    const int64_t* __restrict__ rowptr;
    const int32_t* __restrict__ cols;
    const double* __restrict__ vals;
    __device__ __forceinline__ int64_t base(int32_t j) const { return __ldg(rowptr + j); }
    __device__ __forceinline__ int64_t len(int32_t j) const
    {
        return __ldg(rowptr + j + 1) - __ldg(rowptr + j);
    }
    __device__ __forceinline__ int32_t key(int64_t q) const { return __ldg(cols + q); }
    __device__ __forceinline__ double payload(int64_t q, double a) const
    {
        return __dmul_rn(a, __ldg(vals + q));
    }
};

struct RawStructSource { // RawStructSource: payload 1u, key = column
    using Payload = uint32_t;
    const int64_t* __restrict__ rowptr;
    const int32_t* __restrict__ cols;
    __device__ __forceinline__ int64_t base(int32_t j) const { return __ldg(rowptr + j); }
    __device__ __forceinline__ int64_t len(int32_t j) const
    {
        return __ldg(rowptr + j + 1) - __ldg(rowptr + j);
    }
    __device__ __forceinline__ int32_t key(int64_t q) const { return __ldg(cols + q); }
    __device__ __forceinline__ uint32_t payload(int64_t, double) const { return 1u; }
};

// CompressedSource (engine.cpp:53-60).  The compressed graph is stored in B's
// own slots: row j's pairs live at [rowptr[j], rowptr[j] + csize[j]).
struct CompressedSource {
    using Payload = uint32_t;
    const int64_t* __restrict__ rowptr;
    const int32_t* __restrict__ csize;
    const int2* __restrict__ cp; // {word index, bits}
    __device__ __forceinline__ int64_t base(int32_t j) const { return __ldg(rowptr + j); }
    __device__ __forceinline__ int64_t len(int32_t j) const { return __ldg(csize + j); }
    __device__ __forceinline__ int32_t key(int64_t q) const { return __ldg(&cp[q].x); }
    __device__ __forceinline__ uint32_t payload(int64_t q, double) const
    {
        return static_cast<uint32_t>(__ldg(&cp[q].y));
    }
};

// ---- key -> first-touch position maps ------------------------------------------
// All three map a key to its position in the row's first-touch order; values
// (or column-set words) live in a payload array indexed by that position and
// the keys themselves in `ids` (the row's column list).  insert() is only
// ever called concurrently for DISTINCT keys, and never concurrently with
// lookup() (the caller separates the phases with __syncwarp).

// LP: linear probing, ids/positions in one 64-bit slot (accumulators.hpp:158-273)
struct LPMap {
    int2* slots;      // [T]: x = key (kEmpty = free), y = position
    int32_t* slot_of; // [S]: position -> slot, for O(used) reset (the reference's slots_)
    uint32_t tmask;
    int shift;

    __device__ __forceinline__ int32_t lookup(int32_t key) const
    {
        uint32_t s = hash_slot(key, shift);
        for (;;) {
            const int2 e = slots[s];
            if (e.x == key)
                return e.y;
            if (e.x == kEmpty)
                return -1;
            s = (s + 1) & tmask;
        }
    }
    __device__ __forceinline__ void insert(int32_t key, int32_t pos)
    {
        uint32_t s = hash_slot(key, shift);
        for (;;) {
            if (atomicCAS(&slots[s].x, kEmpty, key) == kEmpty) {
                slots[s].y = pos;
                slot_of[pos] = static_cast<int32_t>(s);
                return;
            }
            s = (s + 1) & tmask;
        }
    }
    __device__ __forceinline__ void reset(int32_t pos, const int32_t*) { slots[slot_of[pos]].x = kEmpty; }
};

// LL: linked-list hashmap of KKMEM (accumulators.hpp:63-151):
// begins[pow2], nexts, ids; position == entry index; lock-free prepend.
struct LLMap {
    int32_t* begins; // [T]
    int32_t* nexts;  // [S]
    const int32_t* ids;
    int shift;

    __device__ __forceinline__ int32_t lookup(int32_t key) const
    {
        for (int32_t s = begins[hash_slot(key, shift)]; s != kEmpty; s = nexts[s])
            if (ids[s] == key)
                return s;
        return -1;
    }
    __device__ __forceinline__ void insert(int32_t key, int32_t pos)
    {
        nexts[pos] = atomicExch(&begins[hash_slot(key, shift)], pos);
    }
    __device__ __forceinline__ void reset(int32_t pos, const int32_t* ids_)
    {
        begins[hash_slot(ids_[pos], shift)] = kEmpty;
    }
};

// Dense: direct position map over the column domain (accumulators.hpp:279-349).
struct DenseMap {
    int32_t* map; // [domain], kEmpty = untouched
    int32_t domain;
    DevCounters* ctr;

    __device__ __forceinline__ int32_t lookup(int32_t key) const
    {
        if (static_cast<uint32_t>(key) >= static_cast<uint32_t>(domain)) {
            raise_error(ctr, kDevKeyRange);
            return -2;
        }
        return map[key];
    }
    __device__ __forceinline__ void insert(int32_t key, int32_t pos) { map[key] = pos; }
    __device__ __forceinline__ void reset(int32_t pos, const int32_t* ids_) { map[ids_[pos]] = kEmpty; }
};

template <class P> __device__ __forceinline__ P combine(P a, P b);
template <> __device__ __forceinline__ double combine<double>(double a, double b)
{
    return __dadd_rn(a, b); // SumCombine, unfused (accumulators.hpp:19-21)
}
template <> __device__ __forceinline__ uint32_t combine<uint32_t>(uint32_t a, uint32_t b)
{
    return a | b; // BitOrCombine (accumulators.hpp:23-25)
}

// One work item: every lane holds at most one (key, payload) product.
// Returns nothing; advances the warp-uniform first-touch counter `cnt`.
// kCountOnly: payload is the constant 1 (raw symbolic) and is not stored.
// spill counts the products whose key's first-touch rank is >= l1_keys: the
// products the reference's two-level accumulators send to level 2
// (engine.cpp:78-87 — a key outside the first l1_keys distinct keys of the row
// finds L1 full), i.e. PhaseStats::l2_inserts.
template <bool kFlat, bool kCountOnly, class Map, class P>
__device__ __forceinline__ void accumulate_item(bool valid, int32_t key, P v, Map& map,
                                                int32_t* ids, P* pay, int32_t cap,
                                                int32_t& cnt, DevCounters* ctr, int lane,
                                                int32_t l1_keys, int64_t& spill)
{
    bool active = valid;
    uint32_t rest = 0;
    if constexpr (kFlat) {
        // duplicate keys inside one window come from different A entries;
        // the lowest lane is the first touch and owns the update.
        const uint32_t grp = __match_any_sync(kFull, valid ? key : (-1 - lane));
        active = valid && (__ffs(grp) - 1) == lane;
        rest = grp & (grp - 1);
    }
    int32_t pos = active ? map.lookup(key) : -1;
    if (pos == -2) { // dense key out of range: drop the product, error already raised
        active = false;
        pos = -1;
    }
    __syncwarp();
    const bool is_new = active && pos < 0;
    const uint32_t nm = __ballot_sync(kFull, is_new);
    bool ok = active;
    if (is_new) {
        pos = cnt + __popc(nm & lanemask_lt());
        if (pos < cap) {
            ids[pos] = key;
            map.insert(key, pos);
        } else {
            raise_error(ctr, kDevRowOverflow);
            ok = false;
        }
    }
    cnt += __popc(nm);
    if (ok && pos >= l1_keys)
        spill += 1 + __popc(rest);
    if constexpr (kCountOnly) {
        __syncwarp();
        return;
    } else {
        P acc = P(0);
        if (ok)
            acc = is_new ? v : combine<P>(pay[pos], v);
        if constexpr (kFlat) {
            // fold the rest of the group in lane order: ((acc + v2) + v3) ...
            const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
            uint32_t m = rest;
            for (int r = 0; r < rounds; ++r) {
                const int src = m ? __ffs(m) - 1 : lane;
                const P x = __shfl_sync(kFull, v, src);
                if (m) {
                    acc = combine<P>(acc, x);
                    m &= m - 1;
                }
            }
        }
        if (ok)
            pay[pos] = acc;
        __syncwarp();
    }
}

// Process row i of C = A*B with the warp.  Returns the number of distinct keys.
template <bool kFlat, bool kCountOnly, class Src, class Map, class P>
__device__ __forceinline__ int32_t warp_row(const int64_t* __restrict__ a_rowptr,
                                            const int32_t* __restrict__ a_cols,
                                            const double* __restrict__ a_vals, int32_t i,
                                            const Src& src, Map& map, int32_t* ids, P* pay,
                                            int32_t cap, DevCounters* ctr, int lane,
                                            int32_t l1_keys, int64_t& spill)
{
    constexpr bool kNumeric = std::is_same<P, double>::value;
    const int64_t abeg = __ldg(a_rowptr + i);
    const int64_t aend = __ldg(a_rowptr + i + 1);
    int32_t cnt = 0;
    for (int64_t p0 = abeg; p0 < aend; p0 += 32) {
        const int na = static_cast<int>(aend - p0 < 32 ? aend - p0 : 32);
        int64_t bbase = 0, blen = 0;
        double av = 0.0;
        if (lane < na) {
            const int32_t j = __ldg(a_cols + p0 + lane);
            if constexpr (kNumeric)
                av = __ldg(a_vals + p0 + lane);
            bbase = src.base(j);
            blen = src.len(j);
        }
        if constexpr (!kFlat) {
            for (int q = 0; q < na; ++q) {
                const int64_t base = __shfl_sync(kFull, bbase, q);
                const int64_t len = __shfl_sync(kFull, blen, q);
                const double a = __shfl_sync(kFull, av, q);
                for (int64_t t0 = 0; t0 < len; t0 += 32) {
                    const int64_t t = t0 + lane;
                    const bool valid = t < len;
                    int32_t key = 0;
                    P v = P(0);
                    if (valid) {
                        key = src.key(base + t);
                        if constexpr (!kCountOnly)
                            v = src.payload(base + t, a);
                    }
                    accumulate_item<false, kCountOnly>(valid, key, v, map, ids, pay, cap, cnt,
                                                       ctr, lane, l1_keys, spill);
                }
            }
        } else {
            int64_t incl = blen;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t y = __shfl_up_sync(kFull, incl, off);
                if (lane >= off)
                    incl += y;
            }
            const int64_t excl = incl - blen;
            const int64_t total = __shfl_sync(kFull, incl, 31);
            for (int64_t w0 = 0; w0 < total; w0 += 32) {
                const int64_t t = w0 + lane;
                const bool valid = t < total;
                // seg = upper_bound(prefix, t) - 1 (flat_position, engine.cpp:360-365)
                int seg = 0;
#pragma unroll
                for (int s = 16; s >= 1; s >>= 1) {
                    const int64_t y = __shfl_sync(kFull, incl, seg + s - 1);
                    if (y <= t)
                        seg += s;
                }
                const int64_t e = __shfl_sync(kFull, excl, seg);
                const int64_t base = __shfl_sync(kFull, bbase, seg);
                const double a = __shfl_sync(kFull, av, seg);
                int32_t key = 0;
                P v = P(0);
                if (valid) {
                    key = src.key(base + (t - e));
                    if constexpr (!kCountOnly)
                        v = src.payload(base + (t - e), a);
                }
                accumulate_item<true, kCountOnly>(valid, key, v, map, ids, pay, cap, cnt, ctr,
                                                  lane, l1_keys, spill);
            }
        }
    }
    return cnt;
}

} // namespace kk
