// sm_100a kernels of the kkSpGEMM hot path and their launchers.
//
//   compress_kernel      K3  compressed_row_sizes + compress_rows (compression.cpp:25-82)
//   flops_kernel<G>      K1+K4 flops_stats + compressed flops (csr_matrix.cpp:136-154,
//                             compression.cpp:109-117), with per-row bucket histograms
//   bin_scatter_kernel        rows -> accumulator classes (row binning by bound)
//   row_kernel<...>      K5/K6 symbolic / numeric row accumulation (engine.cpp:251-351)
//   scan kernels         K2  device exclusive scan of row sizes (engine.cpp:434-438)
//   sort kernels         K7  sort_output pass (engine.cpp:466-485)
//
// All of these are HBM/L2/latency-bound integer and fp64 scalar work; tensor
// cores have no role.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {
std::atomic<long long> g_launches{0};
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

int sm_count()
{
    static int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return sms;
}

__device__ __forceinline__ int bucket_of(unsigned long long x)
{
    // 0 for x == 0, else ceil(log2 x) + 1: bucket b holds x in (2^(b-2), 2^(b-1)]
    return x == 0 ? 0 : min(65 - __clzll(x - 1), 63);
}

// Warp-aggregated histogram increment (all 32 lanes, converged): one shared
// atomic per distinct bucket instead of one per lane (rows of a stencil all
// fall in the same bucket, which serialised the per-lane atomics).  b < 0
// contributes nothing.
__device__ __forceinline__ void warp_hist_add(unsigned long long* sh, int b, int lane)
{
    const uint32_t grp = __match_any_sync(kFull, b);
    if (b >= 0 && (__ffs(grp) - 1) == lane)
        atomicAdd(&sh[b], static_cast<unsigned long long>(__popc(grp)));
}

// OR of v over the lanes of `grp` (a __match_any_sync group), every lane
// receiving its own group's result.  Group membership is arbitrary, so the
// members are visited one by one (rounds = largest group).
__device__ __forceinline__ uint32_t group_or(uint32_t grp, uint32_t v, int lane)
{
    uint32_t acc = v;
    uint32_t m = grp & ~(1u << lane);
    const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(m)));
    for (int r = 0; r < rounds; ++r) {
        const int src = m ? __ffs(m) - 1 : lane;
        const uint32_t x = __shfl_sync(kFull, v, src);
        if (m) {
            acc |= x;
            m &= m - 1;
        }
    }
    return acc;
}

// group_or through a per-warp 32-word shared buffer (zero on entry and on
// return): members OR into their leader's word, then read it back.
__device__ __forceinline__ uint32_t group_or_smem(uint32_t grp, uint32_t v, int lane, uint32_t* buf)
{
    const int leader = __ffs(grp) - 1;
    if (v)
        atomicOr(&buf[leader], v);
    __syncwarp();
    const uint32_t r = buf[leader];
    __syncwarp();
    if (lane == leader)
        buf[lane] = 0u;
    __syncwarp();
    return r;
}

// ---------------------------------------------------------------------------
// K3: graph compression of B, written into B's own slots (pairs of row j at
// [rowptr[j], rowptr[j] + csize[j])).  Warp per row.  Pair order is the
// first-touch order of compression.cpp:67-73 for rows of <= 32 entries and
// for sorted rows; unsorted long rows use an order-insensitive merge (the
// compressed graph only feeds the order-independent bit-OR union).
// ---------------------------------------------------------------------------
// rows up to this length are compressed by one thread (aggregation/AP rows);
// longer ones (stencils: 27) by a warp, whose loads coalesce
#ifndef KK_SHORT_ROW
#define KK_SHORT_ROW 8
#endif
constexpr int32_t kShortRow = KK_SHORT_ROW;

// Thread per B row for rows of <= kShortRow entries:
// the running (word index, bits) pair stays in registers and is flushed when the word
// changes; an out-of-order word (unsorted row) merges into its earlier pair.
// Longer rows are left to the warp kernel below.
// The compressed pairs live in B's own slots relative to the VIEW's first
// offset (rowptr[0] of a row-block view need not be 0): both compress kernels
// take the unshifted allocation and rebase on the device, and work only on the
// band [band[0], band[1]] of B rows that A references when `band` is given —
// so the host never reads either value before launching.
__device__ __forceinline__ void compress_band(int32_t n_all, const int* band, int32_t& j0, int32_t& n)
{
    j0 = 0;
    n = n_all;
    if (band) {
        const int lo = __ldg(band), hi = __ldg(band + 1) + 1;
        j0 = lo < 0 ? 0 : (lo > n_all ? n_all : lo);
        const int e = hi < j0 ? j0 : (hi > n_all ? n_all : hi);
        n = e - j0;
    }
}

// One thread compresses one row, entry by entry (rc: the row's columns, in
// global or shared memory): a run of one word extends the open pair; a word
// at or below the largest seen so far may merge into an earlier pair (rows
// that are not column-sorted), first-touch order kept.  Returns the pair count.
__device__ __forceinline__ int32_t compress_row_seq(const int32_t* __restrict__ rc, int32_t len, int64_t lo,
                                                    int2* __restrict__ cp,
                                                    bool& sorted)
{
    int32_t np = 0, cur_w = -1, maxw = -1, prev_c = INT_MIN;
    uint32_t cur = 0;
    for (int32_t q = 0; q < len; ++q) {
        const int32_t c = rc[q];
        sorted = sorted && c > prev_c;
        prev_c = c;
        const int32_t w = c >> 5;
        const uint32_t bit = 1u << (c & 31);
        if (w == cur_w) {
            cur |= bit;
            continue;
        }
        int32_t found = -1;
        if (w <= maxw) // not beyond every word seen so far: maybe an earlier pair
            for (int32_t t = 0; t < np; ++t)
                if (cp[lo + t].x == w) {
                    found = t;
                    break;
                }
        if (cur_w >= 0) { // flush the running pair
            cp[lo + np - 1].y = static_cast<int>(cur);
            cur_w = -1;
        }
        if (found >= 0) { // merge into the earlier pair, in place (first-touch order kept)
            cp[lo + found].y |= static_cast<int>(bit);
            continue;
        }
        cp[lo + np].x = w;
        ++np;
        cur_w = w;
        cur = bit;
        maxw = max(maxw, w);
    }
    if (cur_w >= 0)
        cp[lo + np - 1].y = static_cast<int>(cur);
    return np;
}

__global__ void __launch_bounds__(256) compress_short_kernel(int32_t n_all, const int64_t* __restrict__ rowptr_all,
                                                             const int32_t* __restrict__ cols,
                                                             int32_t* __restrict__ csize_all,
                                                             int2* __restrict__ cp_alloc, unsigned long long* nnz_bc,
                                                             unsigned long long* unsorted, const int* band)
{
    int32_t j0, n;
    compress_band(n_all, band, j0, n);
    const int64_t* __restrict__ rowptr = rowptr_all + j0;
    int32_t* __restrict__ csize = csize_all + j0;
    int2* __restrict__ cp = cp_alloc - __ldg(rowptr_all);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long pairs = 0;
    bool sorted = true;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < n; b0 += stride) { // warp-uniform trips
        const int64_t j = b0 + threadIdx.x;
        int64_t lo = 0;
        int32_t len = 0;
        if (j < n) {
            lo = __ldg(rowptr + j);
            len = static_cast<int32_t>(__ldg(rowptr + j + 1) - lo);
        }
        // rows beyond kShortRow are the warp kernel's
        const bool is_long = j < n && len > kShortRow;
        if (j >= n || is_long)
            continue;
        const int32_t np = compress_row_seq(cols + lo, len, lo, cp, sorted);
        csize[j] = np;
        pairs += static_cast<unsigned long long>(np);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
        pairs += __shfl_xor_sync(kFull, pairs, off);
    if ((threadIdx.x & 31) == 0 && pairs)
        atomicAdd(nnz_bc, pairs);
    if (!__all_sync(kFull, sorted) && (threadIdx.x & 31) == 0)
        atomicAdd(unsorted, 1ull);
}

__device__ __forceinline__ int compress_row_short(int64_t j, int64_t lo, int64_t len, int32_t col, int lane,
                                                  int32_t* __restrict__ csize, int2* __restrict__ cp,
                                                  bool* sorted_out, uint32_t* orbuf)
{
    const bool valid = lane < len;
    const int32_t w = col >> 5;
    const int32_t key = valid ? w : -1 - lane;
    const uint32_t grp = __match_any_sync(kFull, key);
    const uint32_t orv = group_or_smem(grp, valid ? (1u << (col & 31)) : 0u, lane, orbuf);
    const bool leader = valid && (__ffs(grp) - 1) == lane;
    const uint32_t lm = __ballot_sync(kFull, leader);
    const int32_t prev = __shfl_up_sync(kFull, col, 1);
    if (!__all_sync(kFull, !valid || lane == 0 || col > prev))
        *sorted_out = false;
    if (leader)
        cp[lo + __popc(lm & lanemask_lt())] = make_int2(w, static_cast<int>(orv));
    if (lane == 0)
        csize[j] = __popc(lm);
    return __popc(lm);
}

__device__ int compress_row_long(int64_t j, int64_t lo, int64_t len, const int32_t* __restrict__ cols, int lane,
                                 int32_t* __restrict__ csize, int2* __restrict__ cp, bool* sorted_out);

// Warp kernel for rows of more than kShortRow entries.  A warp takes batches
// of 32 consecutive rows: one coalesced load of their offsets; when the
// batch's entries fit the warp's stage (kCompressStage columns) they are
// copied in with all loads in flight, and each row is compressed from shared
// memory; otherwise the long rows of the batch (ballot) go one after another,
// the next row's columns loaded while the current one is compressed.
constexpr int kCompressStage = 1024;
__global__ void __launch_bounds__(256) compress_kernel(int32_t n_all, const int64_t* __restrict__ rowptr_all,
                                                       const int32_t* __restrict__ cols,
                                                       int32_t* __restrict__ csize_all,
                                                       int2* __restrict__ cp_alloc, unsigned long long* nnz_bc,
                                                       unsigned long long* unsorted, const int* band)
{
    int32_t j0, n;
    compress_band(n_all, band, j0, n);
    const int64_t* __restrict__ rowptr = rowptr_all + j0;
    int32_t* __restrict__ csize = csize_all + j0;
    int2* __restrict__ cp = cp_alloc - __ldg(rowptr_all);
    const int lane = threadIdx.x & 31;
    __shared__ int32_t stage_all[8][kCompressStage];
    __shared__ uint32_t orbuf_all[8][32];
    int32_t* stage = stage_all[threadIdx.x >> 5];
    uint32_t* orbuf = orbuf_all[threadIdx.x >> 5];
    orbuf[lane] = 0u;
    __syncwarp();
    unsigned long long pairs = 0; // warp-uniform
    bool sorted = true;           // warp-uniform
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < n; r0 += warps * 32) {
        const int64_t jr = r0 + lane;
        int64_t blo = 0, blen = 0;
        if (jr < n) {
            blo = __ldg(rowptr + jr);
            blen = __ldg(rowptr + jr + 1) - blo;
        }
        uint32_t todo = __ballot_sync(kFull, jr < n && blen > kShortRow);
        if (!todo)
            continue;
        const int nb = n - r0 < 32 ? static_cast<int>(n - r0) : 32;
        const int64_t sbase = __shfl_sync(kFull, blo, 0);
        const int64_t stot = __shfl_sync(kFull, blo + blen, nb - 1) - sbase;
        if (stot <= kCompressStage && __all_sync(kFull, blen <= 32)) {
            // staged batch: every column load in flight at once
#pragma unroll 4
            for (int t = lane; t < stot; t += 32)
                stage[t] = __ldg(cols + sbase + t);
            __syncwarp();
            while (todo) {
                const int q = __ffs(todo) - 1;
                todo &= todo - 1;
                const int64_t lo = __shfl_sync(kFull, blo, q);
                const int64_t len = __shfl_sync(kFull, blen, q);
                const int32_t col = lane < len ? stage[lo - sbase + lane] : 0;
                pairs += compress_row_short(r0 + q, lo, len, col, lane, csize, cp, &sorted, orbuf);
            }
            __syncwarp();
            continue;
        }
        auto pop = [&]() {
            const int q = todo ? __ffs(todo) - 1 : -1;
            todo &= todo - 1;
            return q;
        };
        auto fetch = [&](int q, int64_t& lo, int64_t& len, int32_t& col) {
            lo = __shfl_sync(kFull, blo, q);
            len = __shfl_sync(kFull, blen, q);
            col = 0;
            if (len <= 32 && lane < len)
                col = __ldg(cols + lo + lane);
        };
        auto process = [&](int q, int64_t lo, int64_t len, int32_t col) {
            if (len <= 32)
                pairs += compress_row_short(r0 + q, lo, len, col, lane, csize, cp, &sorted, orbuf);
            else
                pairs += compress_row_long(r0 + q, lo, len, cols, lane, csize, cp, &sorted);
        };
        int64_t loA = 0, lenA = 0, loB = 0, lenB = 0;
        int32_t colA = 0, colB = 0;
        int qa = pop();
        if (qa >= 0)
            fetch(qa, loA, lenA, colA);
        while (qa >= 0) { // two register sets: a prefetched load is never copied
            const int qb = pop();
            if (qb >= 0)
                fetch(qb, loB, lenB, colB);
            process(qa, loA, lenA, colA);
            if (qb < 0)
                break;
            qa = pop();
            if (qa >= 0)
                fetch(qa, loA, lenA, colA);
            process(qb, loB, lenB, colB);
        }
    }
    if (lane == 0 && pairs)
        atomicAdd(nnz_bc, pairs);
    if (lane == 0 && !sorted)
        atomicAdd(unsorted, 1ull);
}

__device__ int compress_row_long(int64_t j, int64_t lo, int64_t len, const int32_t* __restrict__ cols, int lane,
                                 int32_t* __restrict__ csize, int2* __restrict__ cp, bool* sorted_out)
{
    {
        // long row: sortedness first (one extra read of the row, L1/L2 resident)
        bool sorted = true;
        int32_t prev_last = INT_MIN;
        for (int64_t t0 = 0; t0 < len; t0 += 32) {
            const bool valid = t0 + lane < len;
            const int32_t c = valid ? __ldg(cols + lo + t0 + lane) : INT_MAX;
            int32_t prev = __shfl_up_sync(kFull, c, 1);
            if (lane == 0)
                prev = prev_last;
            sorted = sorted && __all_sync(kFull, !valid || c > prev);
            prev_last = __shfl_sync(kFull, c, 31);
        }
        if (!sorted)
            *sorted_out = false;
        int32_t cnt = 0;
        if (sorted) {
            int32_t carry_w = -1;
            for (int64_t t0 = 0; t0 < len; t0 += 32) {
                const bool valid = t0 + lane < len;
                const int32_t col = valid ? __ldg(cols + lo + t0 + lane) : 0;
                const int32_t w = col >> 5;
                const int32_t key = valid ? w : -1 - lane;
                const uint32_t grp = __match_any_sync(kFull, key);
                const uint32_t orv = group_or(grp, valid ? (1u << (col & 31)) : 0u, lane);
                int32_t pw = __shfl_up_sync(kFull, w, 1);
                if (lane == 0)
                    pw = carry_w;
                const bool start = valid && w != pw;
                if (valid && lane == 0 && w == carry_w)
                    cp[lo + cnt - 1].y |= static_cast<int>(orv); // run continues from the previous chunk
                const uint32_t lm = __ballot_sync(kFull, start);
                if (start)
                    cp[lo + cnt + __popc(lm & lanemask_lt())] = make_int2(w, static_cast<int>(orv));
                cnt += __popc(lm);
                const int last = static_cast<int>(len - 1 - t0 < 31 ? len - 1 - t0 : 31);
                carry_w = __shfl_sync(kFull, w, last);
                __syncwarp();
            }
        } else {
            for (int64_t t0 = 0; t0 < len; t0 += 32) {
                const bool valid = t0 + lane < len;
                const int32_t col = valid ? __ldg(cols + lo + t0 + lane) : 0;
                const int32_t w = col >> 5;
                const int32_t key = valid ? w : -1 - lane;
                const uint32_t grp = __match_any_sync(kFull, key);
                const uint32_t orv = group_or(grp, valid ? (1u << (col & 31)) : 0u, lane);
                const bool leader = valid && (__ffs(grp) - 1) == lane;
                int32_t found = -1;
                if (leader)
                    for (int32_t q = 0; q < cnt; ++q)
                        if (cp[lo + q].x == w) {
                            found = q;
                            break;
                        }
                __syncwarp();
                const bool is_new = leader && found < 0;
                const uint32_t nm = __ballot_sync(kFull, is_new);
                if (is_new)
                    cp[lo + cnt + __popc(nm & lanemask_lt())] = make_int2(w, static_cast<int>(orv));
                else if (leader)
                    cp[lo + found].y |= static_cast<int>(orv);
                cnt += __popc(nm);
                __syncwarp();
            }
        }
        if (lane == 0)
            csize[j] = cnt;
        return cnt;
    }
}

// ---------------------------------------------------------------------------
// K1+K4: per-row flops and compressed flops, totals, maxima and bucket
// histograms (the histograms let the host size every accumulator class
// without another pass).  G lanes per A row.
// ---------------------------------------------------------------------------
template <int G>
#ifndef KK_FLOPS_MINB
#define KK_FLOPS_MINB 4 // 64 registers: no spills (c2 0.71 -> 0.57 ms vs 8)
#endif
__global__ void __launch_bounds__(256, KK_FLOPS_MINB) flops_kernel(int32_t m, const int64_t* __restrict__ a_rowptr,
                                                    const int32_t* __restrict__ a_cols,
                                                    const int64_t* __restrict__ b_rowptr,
                                                    const int32_t* __restrict__ csize,
                                                    int64_t* __restrict__ out_f,
                                                    int64_t* __restrict__ out_cf, Totals* tot)
{
    __shared__ unsigned long long sh_hist[2][64];
    for (int t = threadIdx.x; t < 128; t += blockDim.x)
        (&sh_hist[0][0])[t] = 0;
    __syncthreads();
    const int glane = threadIdx.x & (G - 1);
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    unsigned long long my_tf = 0, my_mf = 0, my_tcf = 0, my_mcf = 0, my_ma = 0;
    const int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
    // uniform trip count per warp so the group shuffles stay converged; two
    // rows per group per trip, their loads issued together (the chain
    // row offsets -> A columns -> B offsets is latency-bound)
    const int64_t iters = (m + 2 * groups - 1) / (2 * groups);
    for (int64_t it = 0; it < iters; ++it) {
        int64_t i2[2], beg[2], end[2], f2[2] = {0, 0}, cf2[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            i2[u] = first + (2 * it + u) * groups;
            beg[u] = end[u] = 0;
            if (i2[u] < m) {
                beg[u] = __ldg(a_rowptr + i2[u]);
                end[u] = __ldg(a_rowptr + i2[u] + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            int64_t p = beg[u] + glane;
            int64_t f = 0, cf = 0;
            for (; p + 3 * G < end[u]; p += 4 * G) {
                int32_t j[4];
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    j[v] = __ldg(a_cols + p + v * G);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    f += __ldg(b_rowptr + j[v] + 1) - __ldg(b_rowptr + j[v]);
                    cf += __ldg(csize + j[v]);
                }
            }
            for (; p < end[u]; p += G) {
                const int32_t j = __ldg(a_cols + p);
                f += __ldg(b_rowptr + j + 1) - __ldg(b_rowptr + j);
                cf += __ldg(csize + j);
            }
            f2[u] = f;
            cf2[u] = cf;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            int64_t f = f2[u], cf = cf2[u];
            const int64_t i = i2[u];
#pragma unroll
            for (int off = G / 2; off >= 1; off >>= 1) {
                f += __shfl_xor_sync(kFull, f, off, G);
                cf += __shfl_xor_sync(kFull, cf, off, G);
            }
            const bool owner = glane == 0 && i < m;
            if (owner) {
                my_ma = max(my_ma, (unsigned long long)(end[u] - beg[u]));
                out_f[i] = f;
                out_cf[i] = cf;
                my_tf += f;
                my_tcf += cf;
                my_mf = max(my_mf, (unsigned long long)f);
                my_mcf = max(my_mcf, (unsigned long long)cf);
            }
            warp_hist_add(sh_hist[0], owner ? bucket_of(f) : -1, threadIdx.x & 31);
            warp_hist_add(sh_hist[1], owner ? bucket_of(cf) : -1, threadIdx.x & 31);
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        my_tf += __shfl_xor_sync(kFull, my_tf, off);
        my_tcf += __shfl_xor_sync(kFull, my_tcf, off);
        my_mf = max(my_mf, __shfl_xor_sync(kFull, my_mf, off));
        my_mcf = max(my_mcf, __shfl_xor_sync(kFull, my_mcf, off));
        my_ma = max(my_ma, __shfl_xor_sync(kFull, my_ma, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&tot->total_f, my_tf);
        atomicAdd(&tot->total_cf, my_tcf);
        atomicMax(&tot->max_f, my_mf);
        atomicMax(&tot->max_cf, my_mcf);
        atomicMax(&tot->max_alen, my_ma);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 128; t += blockDim.x) {
        const unsigned long long v = (&sh_hist[0][0])[t];
        if (v)
            atomicAdd(t < 64 ? &tot->hist_f[t] : &tot->hist_cf[t - 64], v);
    }
}

// ---------------------------------------------------------------------------
// Row binning: class id from the row bound (per-row flops, compressed flops
// or, for the numeric phase, the exact row size), warp-aggregated append.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bin_scatter_kernel(int32_t m, const int64_t* __restrict__ bound,
                                                          const int64_t* __restrict__ rowptr_c,
                                                          int64_t clamp, BinParams bp,
                                                          unsigned long long* fill,
                                                          int32_t* __restrict__ list)
{
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
        const int64_t i = base + threadIdx.x;
        int c = -1;
        if (i < m) {
            int64_t u = bound ? bound[i] : rowptr_c[i + 1] - rowptr_c[i];
            u = min(u, clamp);
            c = bp.bucket_class[bucket_of((unsigned long long)u)];
        }
        const int key = c >= 0 ? c : -1 - lane;
        const uint32_t grp = __match_any_sync(kFull, key);
        const int leader = __ffs(grp) - 1;
        unsigned long long off = 0;
        if (c >= 0 && lane == leader)
            off = atomicAdd(&fill[c], (unsigned long long)__popc(grp));
        off = __shfl_sync(kFull, off, leader);
        if (c >= 0)
            list[bp.class_off[c] + (int64_t)off + __popc(grp & lanemask_lt())] = (int32_t)i;
    }
}

// ---------------------------------------------------------------------------
// K5/K6: the row accumulation kernel.  One warp per row of C; the accumulator
// (key->position map + ids + payload) lives in the warp's shared-memory
// region (L1) or in a pool chunk in HBM (L2).
// ---------------------------------------------------------------------------
template <int kAcc> struct MapOf;
template <> struct MapOf<kAccLP> {
    using type = LPMap;
    __device__ static LPMap make(unsigned char* r, const TabLayout& L, const int32_t*, DevCounters*)
    {
        return LPMap{reinterpret_cast<int2*>(r + L.off_map), reinterpret_cast<int32_t*>(r + L.off_aux),
                     static_cast<uint32_t>(L.T - 1), L.shift};
    }
    __device__ static void init(unsigned char* r, const TabLayout& L, int lane)
    {
        int2* s = reinterpret_cast<int2*>(r + L.off_map);
        for (int t = lane; t < L.T; t += 32)
            s[t] = make_int2(kEmpty, 0);
    }
};
template <> struct MapOf<kAccLL> {
    using type = LLMap;
    __device__ static LLMap make(unsigned char* r, const TabLayout& L, const int32_t* ids, DevCounters*)
    {
        return LLMap{reinterpret_cast<int32_t*>(r + L.off_map), reinterpret_cast<int32_t*>(r + L.off_aux),
                     ids, L.shift};
    }
    __device__ static void init(unsigned char* r, const TabLayout& L, int lane)
    {
        int32_t* b = reinterpret_cast<int32_t*>(r + L.off_map);
        for (int t = lane; t < L.T; t += 32)
            b[t] = kEmpty;
    }
};
template <> struct MapOf<kAccDense> {
    using type = DenseMap;
    __device__ static DenseMap make(unsigned char* r, const TabLayout& L, const int32_t*, DevCounters* c)
    {
        return DenseMap{reinterpret_cast<int32_t*>(r + L.off_map), L.T, c};
    }
    __device__ static void init(unsigned char* r, const TabLayout& L, int lane)
    {
        int32_t* b = reinterpret_cast<int32_t*>(r + L.off_map);
        for (int t = lane; t < L.T; t += 32)
            b[t] = kEmpty;
    }
};

__device__ __forceinline__ int acquire_chunk(const PoolDesc& pool, int hint, int lane)
{
    int c = -1;
    if (lane == 0) {
        for (;;) {
            for (int s = 0; s < pool.num_chunks; ++s) {
                const int cc = (hint + s) % pool.num_chunks;
                if (atomicCAS(&pool.states[cc], 0, 1) == 0) {
                    c = cc;
                    break;
                }
            }
            if (c >= 0)
                break;
            __nanosleep(200);
        }
        __threadfence(); // also invalidates this SM's L1 (stale chunk lines)
    }
    return __shfl_sync(kFull, c, 0);
}

template <int kAcc, bool kFlat, int kVar, bool kL2>
__global__ void __launch_bounds__(256) row_kernel(const RowLaunch L)
{
    extern __shared__ __align__(16) unsigned char smem[];
    using Map = typename MapOf<kAcc>::type;
    constexpr bool kNum = kVar == kVarNumeric;
    constexpr bool kCountOnly = kVar == kVarSymRaw;
    using P = typename std::conditional<kNum, double, uint32_t>::type;

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * L.wpb + wib;
    int64_t nwarps = (int64_t)gridDim.x * L.wpb;
    unsigned char* region = nullptr;
    if constexpr (!kL2) {
        region = smem + (size_t)wib * L.lay.bytes;
        MapOf<kAcc>::init(region, L.lay, lane);
        __syncwarp();
    } else {
        if (L.pool.mode == 0) {
            if (gw >= L.pool.num_chunks)
                return;
            nwarps = L.pool.num_chunks;
            region = reinterpret_cast<unsigned char*>(L.pool.base) + (size_t)gw * L.pool.chunk_bytes;
        }
    }

    // reference statistics (engine.cpp:78-87, memory_pool allocation_count):
    // rows whose distinct keys exceed the reference's L1 key capacity take one
    // pool chunk; every product of a key past that rank is an L2 insert
    unsigned long long my_alloc = 0, my_inserts = 0;
    for (int64_t r = gw; r < L.nrows; r += nwarps) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        int chunk = -1;
        if constexpr (kL2) {
            if (L.pool.mode != 0) {
                chunk = acquire_chunk(L.pool, static_cast<int>(gw % L.pool.num_chunks), lane);
                region = reinterpret_cast<unsigned char*>(L.pool.base) + (size_t)chunk * L.pool.chunk_bytes;
            }
        }
        int32_t* ids;
        P* pay;
        int32_t cap;
        int64_t cbase = 0;
        if constexpr (kNum) {
            cbase = __ldg(L.c_rowptr + i);
            cap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - cbase);
            if (cap == 0)
                continue; // empty row of C: nothing to accumulate
            if constexpr (kL2) {
                ids = L.c_cols + cbase;
                pay = reinterpret_cast<P*>(L.c_vals + cbase);
            } else {
                ids = reinterpret_cast<int32_t*>(region + L.lay.off_ids);
                pay = reinterpret_cast<P*>(region + L.lay.off_pay);
            }
        } else {
            cap = L.lay.S;
            ids = reinterpret_cast<int32_t*>(region + L.lay.off_ids);
            pay = reinterpret_cast<P*>(region + L.lay.off_pay);
        }
        Map map = MapOf<kAcc>::make(region, L.lay, ids, L.ctr);
        int64_t spill = 0;
        int32_t cnt;
        if constexpr (kVar == kVarNumeric) {
            const NumericSource src{L.b_rowptr, L.b_cols, L.b_vals};
            cnt = warp_row<kFlat, false>(L.a_rowptr, L.a_cols, L.a_vals, i, src, map, ids, pay,
                                         cap, L.ctr, lane, L.l1_keys, spill);
        } else if constexpr (kVar == kVarSymRaw) {
            const RawStructSource src{L.b_rowptr, L.b_cols};
            cnt = warp_row<kFlat, true>(L.a_rowptr, L.a_cols, nullptr, i, src, map, ids, pay,
                                        cap, L.ctr, lane, L.l1_keys, spill);
        } else {
            const CompressedSource src{L.b_rowptr, L.csize, cpair_of(L)};
            cnt = warp_row<kFlat, false>(L.a_rowptr, L.a_cols, nullptr, i, src, map, ids, pay,
                                         cap, L.ctr, lane, L.l1_keys, spill);
        }
        const int32_t used = min(cnt, cap);
        if constexpr (kNum) {
            if (cnt < cap && lane == 0)
                raise_error(L.ctr, kDevRowShort);
            if constexpr (!kL2) {
                for (int32_t q = lane; q < used; q += 32) {
                    L.c_cols[cbase + q] = ids[q];
                    L.c_vals[cbase + q] = pay[q];
                }
            }
        } else {
            int64_t size;
            if constexpr (kCountOnly) {
                size = cnt;
            } else {
                int64_t s = 0;
                for (int32_t q = lane; q < used; q += 32)
                    s += __popc(pay[q]);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    s += __shfl_xor_sync(kFull, s, off);
                size = s;
            }
            if (lane == 0)
                L.sym_sizes[i] = size;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            spill += __shfl_xor_sync(kFull, spill, off);
        my_inserts += static_cast<unsigned long long>(spill);
        my_alloc += cnt > L.l1_keys ? 1 : 0;
        __syncwarp();
        for (int32_t q = lane; q < used; q += 32)
            map.reset(q, ids);
        __syncwarp();
        if constexpr (kL2) {
            if (chunk >= 0 && lane == 0) {
                __threadfence();
                atomicExch(&L.pool.states[chunk], 0);
            }
        }
    }
    if (lane == 0 && (my_alloc || my_inserts)) {
        atomicAdd(&L.ctr->pool_allocations, my_alloc);
        atomicAdd(&L.ctr->l2_inserts, my_inserts);
    }
}

// ---------------------------------------------------------------------------
// K2: in-place scan of row sizes.  rowptr[0] = 0 and rowptr[1..m] hold the
// sizes on entry; on exit rowptr is the exclusive offset array.  Phase 1 also
// records the max row size and the size-bucket histogram.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int64_t* __restrict__ x, int64_t n,
                                                                   int64_t* __restrict__ block_sums,
                                                                   ScanTotals* tot)
{
    __shared__ unsigned long long sh_hist[64];
    __shared__ int64_t sh_red[kScanThreads / 32];
    if (tot)
        for (int t = threadIdx.x; t < 64; t += blockDim.x)
            sh_hist[t] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    int64_t s = 0;
    unsigned long long mx = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t idx = base + (int64_t)k * kScanThreads + threadIdx.x;
        int64_t v = 0;
        if (idx < n) {
            v = x[idx];
            s += v;
            mx = max(mx, (unsigned long long)v);
        }
        if (tot)
            warp_hist_add(sh_hist, idx < n ? bucket_of((unsigned long long)v) : -1, threadIdx.x & 31);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        s += __shfl_xor_sync(kFull, s, off);
        mx = max(mx, __shfl_xor_sync(kFull, mx, off));
    }
    if ((threadIdx.x & 31) == 0) {
        sh_red[threadIdx.x >> 5] = s;
        if (tot)
            atomicMax(&tot->max_size, mx);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w)
            t += sh_red[w];
        block_sums[blockIdx.x] = t;
    }
    if (tot)
        for (int t = threadIdx.x; t < 64; t += blockDim.x)
            if (sh_hist[t])
                atomicAdd(&tot->hist[t], sh_hist[t]);
}

// inclusive scan of one tile per block, plus an offset per block (or none)
__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(int64_t* __restrict__ x, int64_t n,
                                                                 const int64_t* __restrict__ block_offsets)
{
    __shared__ int64_t sh_warp[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t v[kScanItems];
    int64_t run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t idx = base + k;
        v[k] = idx < n ? x[idx] : 0;
        run += v[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t incl = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off)
            incl += y;
    }
    if (lane == 31)
        sh_warp[w] = incl;
    __syncthreads();
    int64_t wpre = 0;
    for (int q = 0; q < w; ++q)
        wpre += sh_warp[q];
    int64_t acc = incl - run + wpre + (block_offsets ? block_offsets[blockIdx.x] : 0);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t idx = base + k;
        acc += v[k];
        if (idx < n)
            x[idx] = acc;
    }
}

// exclusive -> used as block offsets: shift an inclusive scan by one
__global__ void shift_exclusive_kernel(const int64_t* __restrict__ incl, int64_t* __restrict__ excl, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        excl[i] = i == 0 ? 0 : incl[i - 1];
}

// inclusive scan of x[0..n) in place (recursive over tiles)
static cudaError_t inclusive_scan(int64_t* x, int64_t n, ScanTotals* tot, cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1 && !tot) {
        scan_tile_kernel<<<1, kScanThreads, 0, st>>>(x, n, nullptr);
        count_launch();
        return cudaGetLastError();
    }
    int64_t* sums = nullptr;
    cudaError_t e = cudaMallocAsync(&sums, sizeof(int64_t) * 2 * tiles, st);
    if (e != cudaSuccess)
        return e;
    int64_t* offs = sums + tiles;
    scan_reduce_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(x, n, sums, tot);
    count_launch();
    e = inclusive_scan(sums, tiles, nullptr, st);
    if (e == cudaSuccess) {
        shift_exclusive_kernel<<<(unsigned)std::min<int64_t>((tiles + 255) / 256, 4096), 256, 0, st>>>(sums, offs, tiles);
        scan_tile_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(x, n, offs);
        count_launch(2);
        e = cudaGetLastError();
    }
    cudaFreeAsync(sums, st);
    return e;
}

cudaError_t scan_sizes_inplace(int64_t* rowptr, int64_t m, ScanTotals* tot, cudaStream_t st)
{
    // rowptr[0] is 0 already; scan the sizes in rowptr[1..m]
    return inclusive_scan(rowptr + 1, m, tot, st);
}

// [min, max] column index of A's entries: the B rows A can reference.  A row
// block of a banded matrix (a multi-GPU shard) references a band of B, and
// only that band is compressed.
__global__ void __launch_bounds__(256) col_range_kernel(int32_t m, const int64_t* __restrict__ a_rowptr,
                                                        const int32_t* __restrict__ a_cols, int* out2)
{
    const int64_t lo = __ldg(a_rowptr), hi = __ldg(a_rowptr + m);
    int mn = INT_MAX, mx = INT_MIN;
    for (int64_t q = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += (int64_t)gridDim.x * blockDim.x) {
        const int c = __ldg(a_cols + q);
        mn = c < mn ? c : mn;
        mx = c > mx ? c : mx;
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out2, mn);
        atomicMax(out2 + 1, mx);
    }
}

cudaError_t launch_col_range(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols, int* out2, cudaStream_t st)
{
    const int init[2] = {INT_MAX, INT_MIN};
    cudaError_t e = cudaMemcpyAsync(out2, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess || m <= 0)
        return e;
    col_range_kernel<<<sm_count() * 4, 256, 0, st>>>(m, a_rowptr, a_cols, out2);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Transpose (csr_matrix.cpp:82-108): column counts, in-place scan, scatter
// through per-column cursors, then the rows of the result are sorted by
// their (original row) column index, which restores the reference's order
// (entries of a column in increasing row order).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) transpose_count_kernel(int32_t m, const int64_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ cols,
                                                              unsigned long long* __restrict__ cnt)
{
    const int64_t lo = __ldg(rowptr), hi = __ldg(rowptr + m);
    for (int64_t q = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + __ldg(cols + q), 1ull);
}

__global__ void __launch_bounds__(256) transpose_scatter_kernel(int32_t m, const int64_t* __restrict__ rowptr,
                                                                const int32_t* __restrict__ cols,
                                                                const double* __restrict__ vals,
                                                                unsigned long long* __restrict__ cursor,
                                                                int32_t* __restrict__ t_cols, double* __restrict__ t_vals)
{
    // warp per row: the row index is the transposed entry's column
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        const int64_t lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
        for (int64_t q = lo + lane; q < hi; q += 32) {
            const unsigned long long p = atomicAdd(cursor + __ldg(cols + q), 1ull);
            t_cols[p] = static_cast<int32_t>(i);
            if (vals)
                t_vals[p] = __ldg(vals + q);
        }
    }
}

// phase 1: column counts -> t_rowptr (scanned); tot->max_size = longest row of A^T
cudaError_t launch_transpose_count(int32_t m, int32_t n, const int64_t* rowptr, const int32_t* cols,
                                   int64_t* t_rowptr, ScanTotals* tot, cudaStream_t st)
{
    cudaError_t e = cudaMemsetAsync(t_rowptr, 0, sizeof(int64_t) * (static_cast<size_t>(n) + 1), st);
    if (e != cudaSuccess)
        return e;
    if (m > 0) {
        transpose_count_kernel<<<sm_count() * 4, 256, 0, st>>>(m, rowptr, cols,
                                                              reinterpret_cast<unsigned long long*>(t_rowptr + 1));
        count_launch();
    }
    return scan_sizes_inplace(t_rowptr, n, tot, st);
}

// phase 2: scatter through per-column cursors, then sort the rows of A^T
cudaError_t launch_transpose_fill(int32_t m, int32_t n, const int64_t* rowptr, const int32_t* cols,
                                  const double* vals, const int64_t* t_rowptr, int32_t* t_cols, double* t_vals,
                                  int64_t max_row, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    unsigned long long* cursor = nullptr;
    cudaError_t e = cudaMallocAsync(&cursor, sizeof(int64_t) * (static_cast<size_t>(n) + 1), st);
    if (e != cudaSuccess)
        return e;
    cudaMemcpyAsync(cursor, t_rowptr, sizeof(int64_t) * (static_cast<size_t>(n) + 1), cudaMemcpyDeviceToDevice, st);
    const int blocks = static_cast<int>(std::min<int64_t>((m + 7) / 8, (int64_t)sm_count() * 8));
    transpose_scatter_kernel<<<blocks, 256, 0, st>>>(m, rowptr, cols, vals, cursor, t_cols, t_vals);
    count_launch();
    cudaFreeAsync(cursor, st);
    if ((e = cudaGetLastError()) != cudaSuccess)
        return e;
    return launch_sort_rows(n, t_rowptr, t_cols, t_vals, max_row, st);
}

// per-row flops only (K1 without compression): the flop-balanced row
// partition of the multi-GPU path.  Warp per row.
__global__ void __launch_bounds__(256) row_flops_kernel(int32_t m, const int64_t* __restrict__ a_rowptr,
                                                        const int32_t* __restrict__ a_cols,
                                                        const int64_t* __restrict__ b_rowptr,
                                                        int64_t* __restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        int64_t f = 0;
        for (int64_t p = __ldg(a_rowptr + i) + lane; p < __ldg(a_rowptr + i + 1); p += 32) {
            const int32_t j = __ldg(a_cols + p);
            f += __ldg(b_rowptr + j + 1) - __ldg(b_rowptr + j);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            f += __shfl_xor_sync(kFull, f, off);
        if (lane == 0)
            out[i] = f;
    }
}

cudaError_t launch_row_flops(int32_t m, const int64_t* a_rowptr, const int32_t* a_cols, const int64_t* b_rowptr,
                             int64_t* out, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    const int blocks = (int)std::min<int64_t>((m + 7) / 8, (int64_t)sm_count() * 8);
    row_flops_kernel<<<blocks, 256, 0, st>>>(m, a_rowptr, a_cols, b_rowptr, out);
    count_launch();
    return cudaGetLastError();
}

__global__ void row_hist_kernel(int32_t m, const int64_t* __restrict__ rowptr, ScanTotals* tot)
{
    __shared__ unsigned long long sh_hist[64];
    for (int t = threadIdx.x; t < 64; t += blockDim.x)
        sh_hist[t] = 0;
    __syncthreads();
    unsigned long long mx = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < m; b0 += stride) { // warp-uniform trips
        const int64_t i = b0 + threadIdx.x;
        unsigned long long v = 0;
        if (i < m) {
            v = (unsigned long long)(rowptr[i + 1] - rowptr[i]);
            mx = max(mx, v);
        }
        warp_hist_add(sh_hist, i < m ? bucket_of(v) : -1, threadIdx.x & 31);
    }
    atomicMax(&tot->max_size, mx);
    __syncthreads();
    for (int t = threadIdx.x; t < 64; t += blockDim.x)
        if (sh_hist[t])
            atomicAdd(&tot->hist[t], sh_hist[t]);
}

cudaError_t launch_row_bucket_hist(int32_t m, const int64_t* rowptr, ScanTotals* tot, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 8);
    row_hist_kernel<<<blocks, 256, 0, st>>>(m, rowptr, tot);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Rows the symbolic structure left empty.  The numeric kernels never visit
// them, so a reused handle whose new operands DO produce products in such a
// row would drop them silently; the reference's NumericSink::finish throws
// "numeric row exceeds the symbolic structure" (engine.cpp:238-239).  The
// rows are collected once per plan and checked on every numeric pass.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) collect_empty_rows_kernel(int32_t m, const int64_t* __restrict__ c_rowptr,
                                                                 int32_t* __restrict__ list,
                                                                 unsigned long long* __restrict__ count)
{
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const bool e = i < m && c_rowptr[i + 1] == c_rowptr[i];
        const uint32_t b = __ballot_sync(kFull, e);
        unsigned long long off = 0;
        if (lane == 0 && b)
            off = atomicAdd(count, (unsigned long long)__popc(b));
        off = __shfl_sync(kFull, off, 0);
        if (e)
            list[off + __popc(b & lanemask_lt())] = static_cast<int32_t>(i);
    }
}

__global__ void __launch_bounds__(256) check_empty_rows_kernel(const int32_t* __restrict__ list, int64_t n,
                                                               const int64_t* __restrict__ a_rowptr,
                                                               const int32_t* __restrict__ a_cols,
                                                               const int64_t* __restrict__ b_rowptr,
                                                               int32_t row_lo, int32_t row_hi, DevCounters* ctr)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    // 32 rows per warp step: lane r owns row list[g + r]; rows with A entries
    // are then walked by the whole warp (rare: an empty C row normally has an
    // empty A row or references empty B rows only)
    for (int64_t g = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; g < n; g += warps * 32) {
        int64_t ab = 0, ae = 0;
        if (g + lane < n) {
            const int32_t i = __ldg(list + g + lane);
            if (!(row_hi > 0 && (i < row_lo || i >= row_hi))) {
                ab = __ldg(a_rowptr + i);
                ae = __ldg(a_rowptr + i + 1);
            }
        }
        uint32_t todo = __ballot_sync(kFull, ae > ab);
        while (todo) {
            const int r = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t lo = __shfl_sync(kFull, ab, r), hi = __shfl_sync(kFull, ae, r);
            bool any = false;
            for (int64_t p = lo + lane; p < hi && !any; p += 32) {
                const int32_t j = __ldg(a_cols + p);
                any = __ldg(b_rowptr + j + 1) > __ldg(b_rowptr + j);
            }
            if (__any_sync(kFull, any)) {
                if (lane == 0)
                    raise_error(ctr, kDevRowOverflow);
                return;
            }
        }
    }
}

cudaError_t launch_collect_empty_rows(int32_t m, const int64_t* c_rowptr, int32_t* list, unsigned long long* count,
                                      cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 8);
    collect_empty_rows_kernel<<<blocks, 256, 0, st>>>(m, c_rowptr, list, count);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_check_empty_rows(const int32_t* list, int64_t n, const int64_t* a_rowptr, const int32_t* a_cols,
                                    const int64_t* b_rowptr, int32_t row_lo, int32_t row_hi, DevCounters* ctr,
                                    cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4));
    check_empty_rows_kernel<<<blocks, 256, 0, st>>>(list, n, a_rowptr, a_cols, b_rowptr, row_lo, row_hi, ctr);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Per-row canonical digests (the device side of oracle.cpp:105-159's
// canonicalize + compare): an order-independent 64-bit hash of each row's
// (column, value bits) set plus its length, so a row in any column order has
// the digest of its sorted form.  The oracle computes the same function on the
// CPU (oracle/spgemm_oracle.c orc_row_digests); equal digests mean equal
// sorted columns and bitwise-equal values.  Warp per row, coalesced reads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t dg_mix(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__global__ void __launch_bounds__(256) row_digest_kernel(int32_t m, const int64_t* __restrict__ rowptr,
                                                         const int32_t* __restrict__ cols,
                                                         const double* __restrict__ vals,
                                                         unsigned long long* __restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        const int64_t lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
        uint64_t d = 0;
        for (int64_t q = lo + lane; q < hi; q += 32) {
            const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(__ldcs(vals + q)));
            const uint32_t c = static_cast<uint32_t>(__ldcs(cols + q));
            d += dg_mix((static_cast<uint64_t>(c) * 0x9E3779B97F4A7C15ull) ^ dg_mix(bits));
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            d += __shfl_xor_sync(kFull, d, off);
        if (lane == 0)
            out[i] = d + dg_mix(static_cast<uint64_t>(hi - lo) + 0x2545F4914F6CDD1Dull);
    }
}

cudaError_t launch_row_digests(int32_t m, const int64_t* rowptr, const int32_t* cols, const double* vals,
                               unsigned long long* out, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((m + 7) / 8, (int64_t)sm_count() * 8));
    row_digest_kernel<<<blocks, 256, 0, st>>>(m, rowptr, cols, vals, out);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K7: per-row column sort (sort_output).  Warp per row; rows of up to
// kSortSmem entries rank-sort in shared memory, longer rows rank-sort from a
// global copy.
// ---------------------------------------------------------------------------
constexpr int kSortSmem = 1024;
constexpr int kSortWarps = 4;

__global__ void __launch_bounds__(32 * kSortWarps) sort_rows_kernel(int32_t m, const int64_t* __restrict__ rowptr,
                                                                    int32_t* __restrict__ cols,
                                                                    double* __restrict__ vals,
                                                                    const int32_t* __restrict__ big_cols,
                                                                    const double* __restrict__ big_vals)
{
    __shared__ int32_t sh_c[kSortWarps][kSortSmem];
    __shared__ double sh_v[kSortWarps][kSortSmem];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t warps = (int64_t)gridDim.x * kSortWarps;
    for (int64_t i = (int64_t)blockIdx.x * kSortWarps + w; i < m; i += warps) {
        const int64_t lo = rowptr[i];
        const int64_t s = rowptr[i + 1] - lo;
        if (s <= 1)
            continue;
        if (s <= kSortSmem) {
            for (int64_t q = lane; q < s; q += 32) {
                sh_c[w][q] = cols[lo + q];
                sh_v[w][q] = vals[lo + q];
            }
            __syncwarp();
            for (int64_t q = lane; q < s; q += 32) {
                const int32_t c = sh_c[w][q];
                int64_t rank = 0;
                for (int64_t r = 0; r < s; ++r)
                    rank += sh_c[w][r] < c;
                cols[lo + rank] = c;
                vals[lo + rank] = sh_v[w][q];
            }
            __syncwarp();
        } else if (big_cols) {
            for (int64_t q = lane; q < s; q += 32) {
                const int32_t c = big_cols[lo + q];
                int64_t rank = 0;
                for (int64_t r = 0; r < s; ++r)
                    rank += big_cols[lo + r] < c;
                cols[lo + rank] = c;
                vals[lo + rank] = big_vals[lo + q];
            }
        }
    }
}

cudaError_t launch_sort_rows(int32_t m, const int64_t* rowptr, int32_t* cols, double* vals,
                             int64_t max_row, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    int32_t* bc = nullptr;
    double* bv = nullptr;
    int64_t nnz = 0;
    if (max_row > kSortSmem) {
        cudaMemcpyAsync(&nnz, rowptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        int64_t base = 0;
        cudaMemcpyAsync(&base, rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        nnz -= base;
        cudaError_t e = cudaMallocAsync(&bc, sizeof(int32_t) * nnz + 16, st);
        if (e != cudaSuccess)
            return e;
        e = cudaMallocAsync(&bv, sizeof(double) * nnz + 16, st);
        if (e != cudaSuccess)
            return e;
        // copies indexed like the originals (offset by the view's base)
        cudaMemcpyAsync(bc, cols + base, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(bv, vals + base, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st);
        bc -= base;
        bv -= base;
        const int blocks = (int)std::min<int64_t>((m + kSortWarps - 1) / kSortWarps, (int64_t)sm_count() * 16);
        sort_rows_kernel<<<blocks, 32 * kSortWarps, 0, st>>>(m, rowptr, cols, vals, bc, bv);
        count_launch();
        cudaFreeAsync(bc + base, st);
        cudaFreeAsync(bv + base, st);
        return cudaGetLastError();
    }
    const int blocks = (int)std::min<int64_t>((m + kSortWarps - 1) / kSortWarps, (int64_t)sm_count() * 16);
    sort_rows_kernel<<<blocks, 32 * kSortWarps, 0, st>>>(m, rowptr, cols, vals, nullptr, nullptr);
    count_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_compress(int32_t n, const int64_t* b_rowptr, const int32_t* b_cols,
                            int32_t* csize, int2* cp_alloc, unsigned long long* nnz_bc, unsigned long long* unsorted,
                            const int* band, cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    // short rows: thread per row; longer rows: warp per row in batches of 32
    const int tblocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
    compress_short_kernel<<<tblocks, 256, 0, st>>>(n, b_rowptr, b_cols, csize, cp_alloc, nnz_bc, unsorted, band);
    count_launch();
    const int64_t batches = (n + 31) / 32;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((batches + 7) / 8, (int64_t)sm_count() * 8));
    compress_kernel<<<blocks, 256, 0, st>>>(n, b_rowptr, b_cols, csize, cp_alloc, nnz_bc, unsorted, band);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_flops(int32_t m, double avg_len, const int64_t* a_rowptr, const int32_t* a_cols,
                         const int64_t* b_rowptr, const int32_t* csize, int64_t* out_f,
                         int64_t* out_cf, Totals* tot, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    // lanes per row: ~4 entries per lane so every lane has several independent
    // gathers in flight (the kernel is latency-bound, not bandwidth-bound)
    int g = 1;
    while (g < 32 && 4 * g < avg_len)
        g <<= 1;
    const int rows_per_block = 256 / g;
    const int blocks = (int)std::min<int64_t>((m + rows_per_block - 1) / rows_per_block, (int64_t)sm_count() * 8);
#define KK_FLOPS(G)                                                                                   \
    case G:                                                                                           \
        flops_kernel<G><<<blocks, 256, 0, st>>>(m, a_rowptr, a_cols, b_rowptr, csize, out_f, out_cf, tot); \
        break;
    switch (g) {
        KK_FLOPS(1)
        KK_FLOPS(2)
        KK_FLOPS(4)
        KK_FLOPS(8)
        KK_FLOPS(16)
        KK_FLOPS(32)
    }
#undef KK_FLOPS
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_bin_scatter(int32_t m, const int64_t* bound, const int64_t* rowptr_c,
                               int64_t clamp, const BinParams& bp, unsigned long long* fill,
                               int32_t* list, cudaStream_t st)
{
    if (m <= 0)
        return cudaSuccess;
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 8);
    bin_scatter_kernel<<<blocks, 256, 0, st>>>(m, bound, rowptr_c, clamp, bp, fill, list);
    count_launch();
    return cudaGetLastError();
}

namespace {
template <int kAcc, bool kFlat, int kVar, bool kL2>
const void* row_kernel_ptr()
{
    return reinterpret_cast<const void*>(&row_kernel<kAcc, kFlat, kVar, kL2>);
}

template <int kAcc, bool kFlat, int kVar>
const void* pick_l2(bool l2)
{
    return l2 ? row_kernel_ptr<kAcc, kFlat, kVar, true>() : row_kernel_ptr<kAcc, kFlat, kVar, false>();
}
template <int kAcc, bool kFlat>
const void* pick_var(int var, bool l2)
{
    switch (var) {
    case kVarNumeric: return pick_l2<kAcc, kFlat, kVarNumeric>(l2);
    case kVarSymRaw: return pick_l2<kAcc, kFlat, kVarSymRaw>(l2);
    default: return pick_l2<kAcc, kFlat, kVarSymCompressed>(l2);
    }
}
template <int kAcc>
const void* pick_flat(bool flat, int var, bool l2)
{
    return flat ? pick_var<kAcc, true>(var, l2) : pick_var<kAcc, false>(var, l2);
}
const void* pick_kernel(int acc, bool flat, int var, bool l2)
{
    switch (acc) {
    case kAccLL: return pick_flat<kAccLL>(flat, var, l2);
    case kAccDense: return pick_flat<kAccDense>(flat, var, l2);
    default: return pick_flat<kAccLP>(flat, var, l2);
    }
}
} // namespace

int row_kernel_max_blocks_per_sm(int acc, bool flat, int variant, bool l2, int wpb, size_t smem)
{
    const void* fn = pick_kernel(acc, flat, variant, l2);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, wpb * 32, smem) != cudaSuccess)
        return 1;
    return std::max(blocks, 1);
}

cudaError_t launch_row_kernel(const RowLaunch& L, int acc, bool flat, int variant, cudaStream_t st)
{
    if (L.nrows <= 0 || L.grid <= 0)
        return cudaSuccess;
    const void* fn = pick_kernel(acc, flat, variant, L.l2);
    const size_t smem = L.l2 ? 0 : (size_t)L.wpb * L.lay.bytes;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    void* args[] = {const_cast<RowLaunch*>(&L)};
    cudaError_t e = cudaLaunchKernel(fn, dim3(L.grid), dim3(L.wpb * 32), args, smem, st);
    count_launch();
    return e;
}

} // namespace kk
