// Heavy rows: rows of C whose accumulator does not fit a warp's shared-memory
// table (R-MAT squares have rows of 10^4..5*10^5 outputs, SURVEY §7 "c4's
// numeric phase is dominated by the HBM L2 path").  One CTA per row.
//
// symbolic_heavy_kernel: the structure union is order-independent, so the CTA
//   ORs every (word index, word) of the row into a DENSE bitmap over the whole
//   column domain in shared memory (the Dense accumulator, accumulators.hpp:
//   279-349, with effective_k = ceil(k/32) words when compressed) and pops it.
//
// numeric_heavy_kernel: values must be summed left to right per key
//   (bit-exact vs the reference), so products are first scattered STABLY into
//   column buckets of W columns (counting sort: per-warp-tile histograms,
//   bucket-major scan, match-ranked scatter in product order), then each warp
//   accumulates one bucket at a time into a dense shared-memory slab with the
//   ordered in-window fold, and emits the bucket's columns in ascending order.
//   Every product is read/written a bounded number of times (streaming), the
//   only random accesses are to shared memory.  Heavy rows therefore come out
//   column-sorted; their values are bitwise the reference's.
#include <cstdint>

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
        for (int32_t w0 = 0; w0 < fm.total; w0 += 32) {
            int32_t e;
            int64_t base;
            double a;
            fm.window(w0, lane, e, base, a);
            const int32_t t = w0 + lane;
            const bool valid = t < fm.total;
            int32_t key = 0;
            uint32_t word = 0;
            double v = 0.0;
            if (valid) {
                const int64_t q = base + (t - e);
                if constexpr (kCompressed) {
                    key = __ldg(L.csi + q);
                    word = __ldg(L.cs + q);
                } else {
                    key = __ldg(L.b_cols + q);
                    word = 1u << (key & 31);
                    if constexpr (kNumeric)
                        v = __dmul_rn(a, __ldg(L.b_vals + q));
                }
            }
            fn(valid, key, word, v);
        }
    }
}

} // namespace

// ---------------------------------------------------------------------------
// symbolic: dense bitmap over the column domain, CTA per row
// ---------------------------------------------------------------------------
template <bool kCompressed>
__global__ void __launch_bounds__(1024) symbolic_heavy_kernel(const RowLaunch L, int32_t words)
{
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem);
    __shared__ unsigned long long red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int t = threadIdx.x; t < words; t += blockDim.x)
        bm[t] = 0u;
    __syncthreads();
    for (int64_t r = blockIdx.x; r < L.nrows; r += gridDim.x) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        // warps take interleaved 32-entry chunks of A(i,:): the union is order-free
        for (int64_t c = abeg + 32 * warp; c < aend; c += 32 * nw)
            walk_products<false, kCompressed>(L, c, c + 32 < aend ? c + 32 : aend, lane,
                                              [&](bool valid, int32_t key, uint32_t word, double) {
                                                  if (valid)
                                                      atomicOr(&bm[kCompressed ? key : (key >> 5)], word);
                                              });
        __syncthreads();
        unsigned long long cnt = 0;
        for (int t = threadIdx.x; t < words; t += blockDim.x) {
            cnt += __popc(bm[t]);
            bm[t] = 0u;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            cnt += __shfl_xor_sync(kFull, cnt, off);
        if (lane == 0)
            red[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long s = 0;
            for (int w = 0; w < nw; ++w)
                s += red[w];
            L.sym_sizes[i] = static_cast<int64_t>(s);
            atomicAdd(&L.ctr->pool_allocations, 1ull);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// numeric: stable column-bucket scatter + ordered dense accumulation
// ---------------------------------------------------------------------------
struct HeavyArgs {
    int32_t* stage_cols; // [num_ctas * stage_cap]
    double* stage_vals;
    int64_t stage_cap;   // products per CTA (>= max row flops)
    int32_t logw;        // bucket width W = 1 << logw columns
    int32_t nb;          // buckets (k / W rounded up)
};

__global__ void __launch_bounds__(kHeavyThreads) numeric_heavy_kernel(const RowLaunch L, const HeavyArgs H)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = H.nb;
    const int W = 1 << H.logw;
    // layout: off[kHeavyWarps][nb] int32 | bstart[nb+1] int32 | bcount[nb] int32 |
    //         per-warp dense slab vals[W] double + bitmap[W/32]
    int32_t* off = reinterpret_cast<int32_t*>(smem);
    int32_t* bstart = off + kHeavyWarps * nb;
    int32_t* bcount = bstart + nb + 1;
    const size_t head = ((size_t)(kHeavyWarps * nb + 2 * nb + 1) * 4 + 15) / 16 * 16;
    double* slab = reinterpret_cast<double*>(smem + head) + (size_t)warp * W;
    uint32_t* bits = reinterpret_cast<uint32_t*>(smem + head + (size_t)kHeavyWarps * W * 8) + (size_t)warp * (W / 32);
    __shared__ int32_t s_total;
    int32_t* scols = H.stage_cols + (size_t)blockIdx.x * H.stage_cap;
    double* svals = H.stage_vals + (size_t)blockIdx.x * H.stage_cap;
    for (int t = lane; t < W / 32; t += 32)
        bits[t] = 0u;

    for (int64_t r = blockIdx.x; r < L.nrows; r += gridDim.x) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - cbase);
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        // contiguous A-entry tile per warp: tiles in warp order = product order
        const int64_t d = aend - abeg;
        const int64_t t_lo = abeg + d * warp / kHeavyWarps, t_hi = abeg + d * (warp + 1) / kHeavyWarps;
        for (int t = threadIdx.x; t < kHeavyWarps * nb; t += blockDim.x)
            off[t] = 0;
        __syncthreads();
        // pass 1: per-(tile, bucket) counts
        walk_products<true, false>(L, t_lo, t_hi, lane, [&](bool valid, int32_t key, uint32_t, double) {
            const int b = valid ? (key >> H.logw) : -1;
            const uint32_t grp = __match_any_sync(kFull, b);
            if (b >= 0 && (__ffs(grp) - 1) == lane)
                off[warp * nb + b] += __popc(grp);
        });
        __syncthreads();
        // bucket-major exclusive scan -> stable offsets off[w][b]
        if (warp == 0) {
            int32_t carry = 0;
            for (int b0 = 0; b0 < nb; b0 += 32) {
                const int b = b0 + lane;
                int32_t tot = 0;
                if (b < nb)
                    for (int w = 0; w < kHeavyWarps; ++w)
                        tot += off[w * nb + b];
                int32_t incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o)
                        incl += y;
                }
                if (b < nb) {
                    int32_t run = carry + incl - tot;
                    bstart[b] = run;
                    for (int w = 0; w < kHeavyWarps; ++w) {
                        const int32_t c = off[w * nb + b];
                        off[w * nb + b] = run;
                        run += c;
                    }
                }
                carry += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0) {
                bstart[nb] = carry;
                s_total = carry;
            }
        }
        __syncthreads();
        // pass 2: stable scatter of (col, a*b) into the CTA's staging area
        walk_products<true, false>(L, t_lo, t_hi, lane, [&](bool valid, int32_t key, uint32_t, double v) {
            const int b = valid ? (key >> H.logw) : -1;
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
                scols[pos] = key;
                svals[pos] = v;
            }
        });
        __syncthreads();
        // pass 3: each warp accumulates whole buckets, in product order
        for (int b = warp; b < nb; b += kHeavyWarps) {
            const int32_t lo = bstart[b], hi = bstart[b + 1];
            for (int32_t w0 = lo; w0 < hi; w0 += 32) {
                const int32_t q = w0 + lane;
                const bool valid = q < hi;
                int32_t key = -1 - lane;
                double v = 0.0;
                if (valid) {
                    key = scols[q] & (W - 1);
                    v = svals[q];
                }
                const uint32_t grp = __match_any_sync(kFull, key);
                const bool leader = valid && (__ffs(grp) - 1) == lane;
                double acc = v;
                if (leader) {
                    // leaders hold distinct keys but may share a bitmap word: atomic set
                    const uint32_t m = 1u << (key & 31);
                    if (atomicOr(&bits[key >> 5], m) & m)
                        acc = __dadd_rn(slab[key], v);
                    // else first touch: the running sum starts at this product
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
                    slab[key] = acc;
                __syncwarp();
            }
            // emit the bucket's columns ascending, compacted in place at its start
            int32_t base = lo;
            for (int t0 = 0; t0 < W / 32; t0 += 32) {
                const uint32_t word = t0 + lane < W / 32 ? bits[t0 + lane] : 0u;
                const int32_t c = __popc(word);
                int32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o)
                        incl += y;
                }
                int32_t pos = base + incl - c;
                uint32_t wb = word;
                while (wb) {
                    const int bit = __ffs(wb) - 1;
                    wb &= wb - 1;
                    const int32_t colw = ((t0 + lane) << 5) + bit;
                    scols[pos] = (b << H.logw) + colw;
                    svals[pos] = slab[colw];
                    ++pos;
                }
                if (t0 + lane < W / 32)
                    bits[t0 + lane] = 0u;
                base += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0)
                bcount[b] = base - lo;
            __syncwarp();
        }
        __syncthreads();
        // output offsets of the buckets; then copy out
        if (warp == 0) {
            int32_t carry = 0;
            for (int b0 = 0; b0 < nb; b0 += 32) {
                const int b = b0 + lane;
                const int32_t c = b < nb ? bcount[b] : 0;
                int32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o)
                        incl += y;
                }
                if (b < nb)
                    off[b] = carry + incl - c; // reuse: output offset of bucket b
                carry += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0 && carry != cap)
                raise_error(L.ctr, carry < cap ? kDevRowShort : kDevRowOverflow);
        }
        __syncthreads();
        for (int b = warp; b < nb; b += kHeavyWarps) {
            const int32_t lo = bstart[b], c = bcount[b], o = off[b];
            for (int32_t q = lane; q < c; q += 32) {
                if (o + q < cap) {
                    L.c_cols[cbase + o + q] = scols[lo + q];
                    L.c_vals[cbase + o + q] = svals[lo + q];
                }
            }
        }
        if (threadIdx.x == 0) {
            atomicAdd(&L.ctr->pool_allocations, 1ull);
            atomicAdd(&L.ctr->l2_inserts, static_cast<unsigned long long>(s_total));
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
size_t heavy_numeric_smem(int nb, int logw)
{
    const size_t head = ((size_t)(kHeavyWarps * nb + 2 * nb + 1) * 4 + 15) / 16 * 16;
    return head + (size_t)kHeavyWarps * ((size_t(1) << logw) * 8 + (size_t(1) << logw) / 8);
}

cudaError_t launch_symbolic_heavy(const RowLaunch& L, bool compressed, int32_t words, int grid, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    const size_t smem = (size_t)words * 4;
    const void* fn = compressed ? reinterpret_cast<const void*>(&symbolic_heavy_kernel<true>)
                                : reinterpret_cast<const void*>(&symbolic_heavy_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    if (compressed)
        symbolic_heavy_kernel<true><<<grid, 1024, smem, st>>>(L, words);
    else
        symbolic_heavy_kernel<false><<<grid, 1024, smem, st>>>(L, words);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_numeric_heavy(const RowLaunch& L, int32_t* stage_cols, double* stage_vals, int64_t stage_cap,
                                 int32_t logw, int32_t nb, int grid, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    const size_t smem = heavy_numeric_smem(nb, logw);
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&numeric_heavy_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    HeavyArgs H{stage_cols, stage_vals, stage_cap, logw, nb};
    numeric_heavy_kernel<<<grid, kHeavyThreads, smem, st>>>(L, H);
    count_launch();
    return cudaGetLastError();
}

} // namespace kk
