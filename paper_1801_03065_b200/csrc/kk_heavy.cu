// Heavy rows: rows of C whose accumulator does not fit a warp's shared-memory
// table (R-MAT squares have rows of 10^4..5*10^5 outputs, SURVEY §7 "c4's
// numeric phase is dominated by the HBM L2 path").  One CTA per row.
//
// symbolic_heavy_kernel: the structure union is order-independent, so the CTA
//   ORs every (word index, word) of the row into a DENSE bitmap over the whole
//   column domain in shared memory (the Dense accumulator, accumulators.hpp:
//   279-349, with effective_k = ceil(k/32) words when compressed) and pops the
//   words it touched (a one-bit-per-word summary lists them).  Chunks with many
//   products are split into windows over all 32 warps.
//
// numeric_heavy_kernel: values must be summed left to right per key
//   (bit-exact vs the reference), so products are first scattered STABLY into
//   hashed column buckets (~256 distinct columns each; counting sort: per-warp
//   tile histograms, bucket-major scan, match-ranked scatter in product order),
//   then each warp accumulates one bucket at a time into a 512-slot shared
//   hash table with the ordered in-window fold and emits it compacted.  Every
//   product is read/written a bounded number of times (streaming); the only
//   random accesses are to shared memory; per-row overhead is proportional to
//   the row's output, not to the column domain.  Heavy rows therefore come out
//   in bucket/slot order (the contract compares sorted rows); their values are
//   bitwise the reference's.
#include <cstdint>

#include <cub/device/device_radix_sort.cuh>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {

constexpr int kHeavyThreads = 256; // numeric: 8 warps
constexpr int kHeavyWarps = kHeavyThreads / 32;

// flat mapping of one chunk of <= 32 A entries (see FlatMap in kk_fast.cu;
// restated here so the heavy kernels are self-contained)
struct HMap {
    int64_t cbase;
    double ca;
    int32_t cexcl, nne, rank, total;
    __device__ __forceinline__ void init(int64_t bb, int32_t bl, double av, int lane)
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
        const int src = lane < nne ? static_cast<int>(__fns(ne, 0, lane + 1)) : lane;
        cbase = __shfl_sync(kFull, bb, src);
        ca = __shfl_sync(kFull, av, src);
        cexcl = __shfl_sync(kFull, excl, src);
        rank = 0;
    }
    __device__ __forceinline__ void window(int32_t w0, int lane, int32_t& e, int64_t& base, double& a)
    {
        const uint32_t bit = (lane < nne && cexcl >= w0 && cexcl < w0 + 32) ? (1u << (cexcl - w0)) : 0u;
        const uint32_t M = __reduce_or_sync(kFull, bit);
        int seg = rank + __popc(M & ((2u << lane) - 1u)) - 1;
        seg = seg < 0 ? 0 : (seg > 31 ? 31 : seg);
        e = __shfl_sync(kFull, cexcl, seg);
        base = __shfl_sync(kFull, cbase, seg);
        a = __shfl_sync(kFull, ca, seg);
        rank += __popc(M);
    }
};

// walk products [p_lo, p_hi) of A's row in flattened (p, t) order, 32 at a
// time: fn(valid, key, value) once per window, warp-converged
template <bool kNumeric, bool kCompressed, class F>
__device__ __forceinline__ void walk_products(const RowLaunch& L, int64_t p_lo, int64_t p_hi, int lane, F&& fn)
{
    const int2* __restrict__ cpair = kCompressed ? cpair_of(L) : nullptr;
    for (int64_t p0 = p_lo; p0 < p_hi; p0 += 32) {
        const int na = static_cast<int>(p_hi - p0 < 32 ? p_hi - p0 : 32);
        int64_t bb = 0;
        int32_t bl = 0;
        double av = 0.0;
        if (lane < na) {
            const int32_t j = __ldg(L.a_cols + p0 + lane);
            if constexpr (kNumeric)
                av = __ldg(L.a_vals + p0 + lane);
            bb = __ldg(L.b_rowptr + j);
            if constexpr (kCompressed)
                bl = __ldg(L.csize + j);
            else
                bl = static_cast<int32_t>(__ldg(L.b_rowptr + j + 1) - bb);
        }
        HMap fm;
        fm.init(bb, bl, av, lane);
        // window loads are issued one window ahead of their use (latency hiding:
        // these kernels run at two CTAs of 8 warps per SM)
        auto load = [&](int32_t w0, int32_t& key, uint32_t& word, double& v) {
            int32_t e;
            int64_t base;
            double a;
            fm.window(w0, lane, e, base, a);
            const int32_t t = w0 + lane;
            key = 0;
            word = 0;
            v = 0.0;
            if (t < fm.total) {
                const int64_t q = base + (t - e);
                if constexpr (kCompressed) {
                    const int2 pr = __ldg(cpair + q);
                    key = pr.x;
                    word = static_cast<uint32_t>(pr.y);
                } else {
                    key = __ldg(L.b_cols + q); // raw column: its word bit is set at use
                    if constexpr (kNumeric)
                        v = __dmul_rn(a, __ldg(L.b_vals + q));
                }
            }
        };
        int32_t nkey;
        uint32_t nword;
        double nv;
        if (fm.total > 0)
            load(0, nkey, nword, nv);
        for (int32_t w0 = 0; w0 < fm.total; w0 += 32) {
            const int32_t key = nkey;
            uint32_t word = nword;
            const double v = nv;
            const bool valid = w0 + lane < fm.total;
            if (w0 + 32 < fm.total)
                load(w0 + 32, nkey, nword, nv);
            if constexpr (!kCompressed)
                word = 1u << (key & 31);
            fn(valid, key, word, v);
        }
    }
}

} // namespace

// ---------------------------------------------------------------------------
// symbolic: dense bitmap over the column domain, CTA per row
// ---------------------------------------------------------------------------
template <bool kCompressed>
// words: bitmap words in shared memory; dom_words: words of the whole column
// domain.  A domain wider than the bitmap is walked in ranges of `words`
// words, the row's pairs filtered per range (no size limit on k).
__global__ void __launch_bounds__(1024) symbolic_heavy_kernel(const RowLaunch L, int32_t words, int32_t dom_words)
{
    extern __shared__ __align__(16) unsigned char smem[];
    // bm: dense bitmap of the column domain; sm: one bit per bm word, set on
    // the word's first touch, so the count-and-clear pass visits touched words
    // only (O(touched), not O(domain), per row)
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem);
    const int32_t swords = (words + 31) >> 5;
    uint32_t* sm = bm + words;
    __shared__ unsigned long long red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int2* __restrict__ cpair = kCompressed ? cpair_of(L) : nullptr;
    for (int t = threadIdx.x; t < words + swords; t += blockDim.x)
        bm[t] = 0u;
    __syncthreads();
    int32_t r0 = 0; // first word of the current range
    auto add = [&](int32_t w, uint32_t word) {
        w -= r0;
        if (static_cast<uint32_t>(w) >= static_cast<uint32_t>(words))
            return; // another range's word
        if (atomicOr(&bm[w], word) == 0u)
            atomicOr(&sm[w >> 5], 1u << (w & 31));
    };
    const int64_t nrows = L.d_nrows ? static_cast<int64_t>(*L.d_nrows) : L.nrows;
    for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        unsigned long long row_cnt = 0; // (thread 0)
        for (r0 = 0; r0 < dom_words; r0 += words) {
            // chunks of 32 A entries: a chunk with many products is split into
            // 32-product windows over all warps, a small one goes to one warp
            // (the union is order-free)
            for (int64_t c = abeg, ci = 0; c < aend; c += 32, ++ci) {
                const int na = static_cast<int>(aend - c < 32 ? aend - c : 32);
                int64_t bb = 0;
                int32_t bl = 0;
                if (lane < na) {
                    const int32_t j = __ldg(L.a_cols + c + lane);
                    bb = __ldg(L.b_rowptr + j);
                    bl = kCompressed ? __ldg(L.csize + j) : static_cast<int32_t>(__ldg(L.b_rowptr + j + 1) - bb);
                }
                const int32_t tot = static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<unsigned>(bl)));
                const bool split = tot >= 8 * 32;
                if (!split && (ci % nw) != warp)
                    continue;
                HMap fm;
                fm.init(bb, bl, 0.0, lane);
                const int32_t w_first = split ? 32 * warp : 0, w_step = split ? 32 * nw : 32;
                for (int32_t w0 = w_first; w0 < tot; w0 += w_step) {
                    // segments that start before the window (windows are strided)
                    fm.rank = __popc(__ballot_sync(kFull, lane < fm.nne && fm.cexcl < w0));
                    int32_t e;
                    int64_t base;
                    double a_unused;
                    fm.window(w0, lane, e, base, a_unused);
                    const int32_t t = w0 + lane;
                    if (t < tot) {
                        const int64_t q = base + (t - e);
                        if constexpr (kCompressed) {
                            const int2 pr = __ldg(cpair + q);
                            add(pr.x, static_cast<uint32_t>(pr.y));
                        } else {
                            const int32_t key = __ldg(L.b_cols + q);
                            add(key >> 5, 1u << (key & 31));
                        }
                    }
                }
            }
            __syncthreads();
            unsigned long long cnt = 0;
            for (int t = threadIdx.x; t < swords; t += blockDim.x) {
                uint32_t sw = sm[t];
                while (sw) {
                    const int b = __ffs(sw) - 1;
                    sw &= sw - 1;
                    const int32_t w = (t << 5) + b;
                    cnt += __popc(bm[w]);
                    bm[w] = 0u;
                }
                sm[t] = 0u;
            }
    #pragma unroll
            for (int off = 16; off >= 1; off >>= 1)
                cnt += __shfl_xor_sync(kFull, cnt, off);
            if (lane == 0)
                red[warp] = cnt;
            __syncthreads();
            if (threadIdx.x == 0)
                for (int w = 0; w < nw; ++w)
                    row_cnt += red[w];
            __syncthreads();
        } // column ranges
        if (threadIdx.x == 0)
            L.sym_sizes[i] = static_cast<int64_t>(row_cnt);
    }
}

// ---------------------------------------------------------------------------
// numeric: stable column-bucket scatter + ordered dense accumulation
// ---------------------------------------------------------------------------
struct HeavyArgs {
    longlong2* stage;    // [num_ctas * stage_cap] records {column, value bits}: one 16-byte store per product
    int64_t stage_cap;   // products per CTA (>= max row flops)
    int32_t bucket_keys; // target distinct columns per bucket
    int32_t nb;          // maximum buckets per row
    int64_t min_products, max_products; // rows with products in (min, max] only
    int32_t queue;                      // which DevCounters::next_row head this launch uses
};

// block-wide exclusive scan of one int32 per thread (kHeavyThreads threads);
// returns the exclusive prefix, *total gets the sum
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* sh_warp, int32_t* total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o)
            incl += y;
    }
    if (lane == 31)
        sh_warp[warp] = incl;
    __syncthreads();
    int32_t wpre = 0, tot = 0;
    for (int w = 0; w < kHeavyWarps; ++w) {
        const int32_t x = sh_warp[w];
        wpre += w < warp ? x : 0;
        tot += x;
    }
    *total = tot;
    __syncthreads();
    return wpre + incl - v;
}

// per-warp bucket table (pass 3): linear probing, keys[kHeavyT] + vals[kHeavyT]
constexpr int kHeavyT = 512;
constexpr int kHeavyTShift = 32 - 9;

__device__ __forceinline__ int heavy_bucket(int32_t key, int nb)
{
    // multiply-shift range reduction of a Fibonacci hash: buckets balance the
    // row's DISTINCT columns whatever their distribution (R-MAT hubs)
    return static_cast<int>((static_cast<uint64_t>(static_cast<uint32_t>(key) * 0x9E3779B1u) * nb) >> 32);
}

__device__ __forceinline__ uint32_t heavy_slot(int32_t key)
{
    return (static_cast<uint32_t>(key) * 0x85EBCA6Bu) >> kHeavyTShift; // independent of the bucket hash
}

__global__ void __launch_bounds__(kHeavyThreads) numeric_heavy_kernel(const RowLaunch L, const HeavyArgs H)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb_max = H.nb;
    // shared memory: bstart[nb+1] bcount[nb] outoff[nb] | union {
    //   off[kHeavyWarps][nb] int32            (passes 1-2: tile x bucket offsets)
    //   per-warp bucket tables keys[T] + vals[T] (pass 3) }
    int32_t* bstart = reinterpret_cast<int32_t*>(smem);
    int32_t* bcount = bstart + nb_max + 1;
    int32_t* outoff = bcount + nb_max;
    const size_t head = ((size_t)(3 * nb_max + 1) * 4 + 15) / 16 * 16;
    int32_t* off = reinterpret_cast<int32_t*>(smem + head);
    double* tvals = reinterpret_cast<double*>(smem + head) + (size_t)warp * kHeavyT;
    int32_t* tkeys = reinterpret_cast<int32_t*>(smem + head + (size_t)kHeavyWarps * kHeavyT * 8) + (size_t)warp * kHeavyT;
    __shared__ int32_t sh_warp[kHeavyWarps];
    __shared__ int64_t tile_lo[kHeavyWarps + 1];
    __shared__ int32_t next_bucket;
    __shared__ int64_t s_row;
    longlong2* srec = H.stage + (size_t)blockIdx.x * H.stage_cap;

    // rows are taken from a queue (the list is ordered by decreasing products,
    // so the largest rows start first and the tail is short)
    for (;;) {
        if (threadIdx.x == 0)
            s_row = static_cast<int64_t>(atomicAdd(&L.ctr->next_row[H.queue], 1ull));
        __syncthreads();
        const int64_t r = s_row;
        __syncthreads();
        if (r >= L.nrows)
            break;
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - cbase);
        // buckets for this row: about H.bucket_keys distinct columns each
        int nb = (cap + H.bucket_keys - 1) / H.bucket_keys;
        nb = nb < 1 ? 1 : (nb > nb_max ? nb_max : nb);
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        const int64_t d = aend - abeg;
        // ---- product-balanced contiguous tiles of A entries, one per warp ----
        // thread t owns A entries [abeg + d*t/T, abeg + d*(t+1)/T)
        const int64_t e_lo = abeg + d * threadIdx.x / kHeavyThreads;
        const int64_t e_hi = abeg + d * (threadIdx.x + 1) / kHeavyThreads;
        int32_t mine = 0;
        for (int64_t p = e_lo; p < e_hi; ++p) {
            const int32_t j = __ldg(L.a_cols + p);
            mine += static_cast<int32_t>(__ldg(L.b_rowptr + j + 1) - __ldg(L.b_rowptr + j));
        }
        if (threadIdx.x <= kHeavyWarps)
            tile_lo[threadIdx.x] = threadIdx.x == 0 ? abeg : aend;
        int32_t F;
        const int32_t before = block_excl_scan(mine, sh_warp, &F);
        if (F <= H.min_products || F > H.max_products)
            continue; // another launch (staging size class) takes this row
        if (threadIdx.x == 0)
            next_bucket = 0;
        // tile w starts at the first A entry p whose product prefix P(p) >= F*w/8
        for (int w = 1; w < kHeavyWarps; ++w) {
            const int64_t target = static_cast<int64_t>(F) * w / kHeavyWarps;
            long long cand = aend;
            if (before >= target) {
                cand = e_lo;
            } else if (before + mine >= target) {
                int64_t run = before;
                for (int64_t p = e_lo; p < e_hi; ++p) {
                    if (run >= target) {
                        cand = p;
                        break;
                    }
                    const int32_t j = __ldg(L.a_cols + p);
                    run += __ldg(L.b_rowptr + j + 1) - __ldg(L.b_rowptr + j);
                }
            }
            if (cand < aend)
                atomicMin(reinterpret_cast<long long*>(&tile_lo[w]), cand);
        }
        for (int t = threadIdx.x; t < kHeavyWarps * nb; t += blockDim.x)
            off[t] = 0;
        __syncthreads();
        const int64_t t_lo = tile_lo[warp], t_hi = tile_lo[warp + 1];
        // ---- pass 1: per-(tile, bucket) counts ----
        walk_products<true, false>(L, t_lo, t_hi, lane, [&](bool valid, int32_t key, uint32_t, double) {
            const int b = valid ? heavy_bucket(key, nb) : -1;
            const uint32_t grp = __match_any_sync(kFull, b);
            if (b >= 0 && (__ffs(grp) - 1) == lane)
                off[warp * nb + b] += __popc(grp);
        });
        __syncthreads();
        // ---- bucket-major exclusive scan -> stable offsets off[w][b] ----
        {
            const int per = (nb + kHeavyThreads - 1) / kHeavyThreads; // buckets per thread
            const int b0 = threadIdx.x * per;
            int32_t mysum = 0;
            for (int u = 0; u < per; ++u) {
                const int b = b0 + u;
                if (b < nb)
                    for (int w = 0; w < kHeavyWarps; ++w)
                        mysum += off[w * nb + b];
            }
            int32_t all;
            int32_t run = block_excl_scan(mysum, sh_warp, &all);
            for (int u = 0; u < per; ++u) {
                const int b = b0 + u;
                if (b < nb) {
                    bstart[b] = run;
                    for (int w = 0; w < kHeavyWarps; ++w) {
                        const int32_t c = off[w * nb + b];
                        off[w * nb + b] = run;
                        run += c;
                    }
                }
            }
            if (threadIdx.x == 0)
                bstart[nb] = all;
        }
        __syncthreads();
        // ---- pass 2: stable scatter of (col, a*b) into the CTA's staging ----
        walk_products<true, false>(L, t_lo, t_hi, lane, [&](bool valid, int32_t key, uint32_t, double v) {
            const int b = valid ? heavy_bucket(key, nb) : -1;
            const uint32_t grp = __match_any_sync(kFull, b);
            const int leader = __ffs(grp) - 1;
            int32_t base = 0;
            if (b >= 0 && lane == leader) {
                base = off[warp * nb + b];
                off[warp * nb + b] = base + __popc(grp);
            }
            base = __shfl_sync(kFull, base, leader);
            if (b >= 0) {
                const int32_t pos = base + __popc(grp & lanemask_lt());
                srec[pos] = make_longlong2(key, __double_as_longlong(v));
            }
        });
        __syncthreads();
        // ---- pass 3: warps grab buckets; ordered accumulation in a per-warp
        //      hash table, emitted compacted at the bucket's start ----
        for (int t = lane; t < kHeavyT; t += 32) // the tables aliased off[] in passes 1-2
            tkeys[t] = kEmpty;
        __syncwarp();
        for (;;) {
            int b = 0;
            if (lane == 0)
                b = atomicAdd(&next_bucket, 1);
            b = __shfl_sync(kFull, b, 0);
            if (b >= nb)
                break;
            const int32_t lo = bstart[b], hi = bstart[b + 1];
            int32_t nkey = -1 - lane;
            double nv = 0.0;
            if (lo + lane < hi) {
                const longlong2 rc = srec[lo + lane];
                nkey = static_cast<int32_t>(rc.x);
                nv = __longlong_as_double(rc.y);
            }
            bool lost = false;
            for (int32_t w0 = lo; w0 < hi; w0 += 32) {
                const int32_t q = w0 + lane;
                const bool valid = q < hi;
                const int32_t key = nkey;
                const double v = nv;
                // next window's products are loaded while this one accumulates
                nkey = -1 - lane;
                nv = 0.0;
                if (q + 32 < hi) {
                    const longlong2 rc = srec[q + 32];
                    nkey = static_cast<int32_t>(rc.x);
                    nv = __longlong_as_double(rc.y);
                }
                const uint32_t grp = __match_any_sync(kFull, key);
                const bool leader = valid && (__ffs(grp) - 1) == lane;
                double acc = v;
                uint32_t s = 0;
                if (leader) {
                    // leaders hold distinct keys; a first touch claims a slot and
                    // its running sum starts at this product
                    s = heavy_slot(key);
                    int probes = 0;
                    for (;;) {
                        const int32_t k = tkeys[s];
                        if (k == key) {
                            acc = __dadd_rn(tvals[s], v);
                            break;
                        }
                        if (k == kEmpty) {
                            const int32_t old = atomicCAS(&tkeys[s], kEmpty, key);
                            if (old == kEmpty)
                                break;
                            if (old == key) {
                                acc = __dadd_rn(tvals[s], v); // unreachable: leaders are distinct
                                break;
                            }
                        }
                        s = (s + 1) & (kHeavyT - 1);
                        if (++probes >= kHeavyT) {
                            lost = true;
                            break;
                        }
                    }
                }
                uint32_t rest = leader ? (grp & (grp - 1)) : 0u;
                const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(rest)));
                for (int rr = 0; rr < rounds; ++rr) {
                    const int src = rest ? __ffs(rest) - 1 : lane;
                    const double x = __shfl_sync(kFull, v, src);
                    if (rest) {
                        acc = __dadd_rn(acc, x);
                        rest &= rest - 1;
                    }
                }
                if (leader)
                    tvals[s] = acc;
                __syncwarp();
            }
            if (__any_sync(kFull, lost) && lane == 0)
                raise_error(L.ctr, kDevL2Overflow);
            // emit the bucket's columns (table order), compacted in place at its start
            int32_t base = lo;
            for (int t0 = 0; t0 < kHeavyT; t0 += 32) {
                const int32_t k = tkeys[t0 + lane];
                const bool hit = k != kEmpty;
                const uint32_t m = __ballot_sync(kFull, hit);
                if (hit) {
                    const int32_t pos = base + __popc(m & lanemask_lt());
                    srec[pos] = make_longlong2(k, __double_as_longlong(tvals[t0 + lane]));
                    tkeys[t0 + lane] = kEmpty;
                }
                base += __popc(m);
            }
            if (lane == 0)
                bcount[b] = base - lo;
            __syncwarp();
        }
        __syncthreads();
        // ---- output offsets of the buckets, then copy out ----
        {
            const int per = (nb + kHeavyThreads - 1) / kHeavyThreads;
            const int b0 = threadIdx.x * per;
            int32_t mysum = 0;
            for (int u = 0; u < per; ++u)
                mysum += b0 + u < nb ? bcount[b0 + u] : 0;
            int32_t all;
            int32_t run = block_excl_scan(mysum, sh_warp, &all);
            for (int u = 0; u < per; ++u) {
                const int b = b0 + u;
                if (b < nb) {
                    outoff[b] = run;
                    run += bcount[b];
                }
            }
            if (threadIdx.x == 0 && all != cap)
                raise_error(L.ctr, all < cap ? kDevRowShort : kDevRowOverflow);
        }
        __syncthreads();
        for (int b = warp; b < nb; b += kHeavyWarps) {
            const int32_t lo = bstart[b], c = bcount[b], o = outoff[b];
            for (int32_t q = lane; q < c; q += 32) {
                if (o + q < cap) {
                    const longlong2 rc = srec[lo + q];
                    L.c_cols[cbase + o + q] = static_cast<int32_t>(rc.x);
                    L.c_vals[cbase + o + q] = __longlong_as_double(rc.y);
                }
            }
        }
        __syncthreads();
    }
}

size_t heavy_numeric_smem(int nb, int /*bucket_keys*/)
{
    const size_t head = ((size_t)(3 * nb + 1) * 4 + 15) / 16 * 16;
    const size_t hist = (size_t)kHeavyWarps * nb * 4;
    const size_t tables = (size_t)kHeavyWarps * kHeavyT * 12;
    return head + (hist > tables ? hist : tables);
}

__global__ void gather_row_flops_kernel(const int32_t* __restrict__ list, int64_t n, const int64_t* __restrict__ prf,
                                        int64_t* __restrict__ keys)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        keys[t] = __ldg(prf + __ldg(list + t));
}

cudaError_t sort_rows_by_flops_desc(int32_t* list, int64_t n, const int64_t* prf, cudaStream_t st)
{
    if (n <= 1)
        return cudaSuccess;
    int64_t *k_in = nullptr, *k_out = nullptr;
    int32_t* v_out = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, k_in, k_out, list, v_out,
                                                             static_cast<int>(n), 0, 64, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&k_in, sizeof(int64_t) * n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&k_out, sizeof(int64_t) * n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&v_out, sizeof(int32_t) * n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&tmp, tmp_bytes, st);
    if (e == cudaSuccess) {
        gather_row_flops_kernel<<<sm_count() * 4, 256, 0, st>>>(list, n, prf, k_in);
        count_launch();
        e = cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, k_in, k_out, list, v_out, static_cast<int>(n),
                                                     0, 64, st);
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(list, v_out, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
    for (void* p : {static_cast<void*>(k_in), static_cast<void*>(k_out), static_cast<void*>(v_out), tmp})
        if (p)
            cudaFreeAsync(p, st);
    return e;
}

int numeric_heavy_blocks_per_sm(int32_t nb)
{
    const size_t smem = heavy_numeric_smem(nb, 0);
    const void* fn = reinterpret_cast<const void*>(&numeric_heavy_kernel);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kHeavyThreads, smem) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

cudaError_t launch_symbolic_heavy(const RowLaunch& L, bool compressed, int32_t words, int32_t dom_words, int grid,
                                  cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    const size_t smem = ((size_t)words + (words + 31) / 32) * 4;
    const void* fn = compressed ? reinterpret_cast<const void*>(&symbolic_heavy_kernel<true>)
                                : reinterpret_cast<const void*>(&symbolic_heavy_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    if (compressed)
        symbolic_heavy_kernel<true><<<grid, 1024, smem, st>>>(L, words, dom_words);
    else
        symbolic_heavy_kernel<false><<<grid, 1024, smem, st>>>(L, words, dom_words);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_numeric_heavy(const RowLaunch& L, void* stage, int64_t stage_cap,
                                 int32_t bucket_keys, int32_t nb, int64_t min_products, int64_t max_products,
                                 int queue, int grid, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    const size_t smem = heavy_numeric_smem(nb, bucket_keys);
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_heavy_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    HeavyArgs H{static_cast<longlong2*>(stage), stage_cap, bucket_keys, nb, min_products, max_products, queue};
    numeric_heavy_kernel<<<grid, kHeavyThreads, smem, st>>>(L, H);
    count_launch();
    return cudaGetLastError();
}

} // namespace kk
