// Rows of at most kTinyKeys distinct keys: one THREAD per row (sm_100a).
//
// On 2D stencils and the A*P stage of a Galerkin product a row of C has ~10
// keys from ~25 products.  A warp spends a whole 32-product window (segment
// map, match, table reset, flush) on such a row, so those kernels are bound by
// per-row instruction overhead, not by the bytes.  Here every thread owns a
// row and a kTinyKeys-entry table in shared memory, laid out [slot][thread]
// so the 32 threads of a warp touch 32 consecutive words (no bank conflicts),
// and visits the row's products in the reference's order — A position, then
// B position (engine.cpp:259-267) — with a linear search of its few keys.
//
// numeric_tiny_kernel   Keys are appended in first-touch order; values are
//     the left-to-right sums from the first product with unfused multiply and
//     add (NumericSink, engine.cpp:223-247), so columns and value bits equal
//     the warp kernels' and the reference's raw output.  A row whose
//     distinct keys differ from the symbolic count raises the reference's
//     row overflow / short errors (engine.cpp:238-245).
// symbolic_tiny_kernel  Order-free union of (word, bits) pairs (or raw
//     columns) for rows whose bound — compressed flops or flops, an exact
//     upper bound on the distinct keys — is at most kTinySymKeys
//     (SymbolicSink, engine.cpp:210-221); the size is the popcount.
#include <algorithm>
#include <cstdint>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {

#ifndef KK_TINY_THREADS
#define KK_TINY_THREADS 128
#endif
constexpr int kTinyThreads = KK_TINY_THREADS;

__global__ void __launch_bounds__(kTinyThreads) numeric_tiny_kernel(const RowLaunch L)
{
    __shared__ int32_t skeys[kTinyKeys][kTinyThreads];
    __shared__ double svals[kTinyKeys][kTinyThreads];
    if (L.gate && L.gate[0] == L.gate[2] && L.gate[1] == L.gate[3])
        return; // the slot replay (kk_replay.cu) computed this pass
    const int tid = threadIdx.x;
    const uint64_t pol = l2_keep_policy();
    const int64_t stride = (int64_t)gridDim.x * kTinyThreads;
    for (int64_t r = (int64_t)blockIdx.x * kTinyThreads + tid; r < L.nrows; r += stride) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        if (L.row_hi > 0 && (i < L.row_lo || i >= L.row_hi))
            continue; // outside the requested row range (spg_numeric_rows)
        const int64_t cbase = __ldg(L.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(L.c_rowptr + i + 1) - cbase);
        const int32_t lim = cap < kTinyKeys ? cap : kTinyKeys;
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        int32_t cnt = 0;
        bool over = false;
        for (int64_t p = abeg; p < aend; ++p) {
            const int32_t j = __ldg(L.a_cols + p);
            const double av = __ldg(L.a_vals + p);
            const int64_t b0 = __ldg(L.b_rowptr + j), b1 = __ldg(L.b_rowptr + j + 1);
            for (int64_t q0 = b0; q0 < b1; q0 += 8) {
                // a B row's entries loaded together, then folded in order
                int32_t kk[8];
                double vv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    kk[u] = -1;
                    vv[u] = 0.0;
                    if (q0 + u < b1) {
                        kk[u] = ldg_keep(L.b_cols + q0 + u, pol);
                        vv[u] = ldg_keep(L.b_vals + q0 + u, pol);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (q0 + u >= b1)
                        break;
                    const double v = __dmul_rn(av, vv[u]);
                    int t = 0;
                    while (t < cnt && skeys[t][tid] != kk[u])
                        ++t;
                    if (t < cnt) {
                        svals[t][tid] = __dadd_rn(svals[t][tid], v);
                    } else if (cnt < lim) {
                        skeys[cnt][tid] = kk[u];
                        svals[cnt][tid] = v; // the first product itself: -0.0 and NaN payloads kept
                        ++cnt;
                    } else {
                        over = true; // more distinct keys than the structure holds
                    }
                }
            }
        }
        if (over || cnt != cap)
            raise_error(L.ctr, over || cnt > cap ? kDevRowOverflow : kDevRowShort);
        for (int32_t t = 0; t < cnt; ++t) {
            st_stream(L.c_cols + cbase + t, skeys[t][tid]);
            st_stream(L.c_vals + cbase + t, svals[t][tid]);
        }
    }
}

template <bool kCompressed>
__global__ void __launch_bounds__(kTinyThreads) symbolic_tiny_kernel(const RowLaunch L,
                                                                     unsigned long long* retry_count,
                                                                     int32_t* retry_list)
{
    __shared__ int32_t skeys[kTinySymKeys][kTinyThreads];
    __shared__ uint32_t swords[kTinySymKeys][kTinyThreads];
    const int tid = threadIdx.x;
    const int2* __restrict__ cpair = cpair_of(L);
    const int64_t stride = (int64_t)gridDim.x * kTinyThreads;
    for (int64_t r = (int64_t)blockIdx.x * kTinyThreads + tid; r < L.nrows; r += stride) {
        const int32_t i = L.list ? __ldg(L.list + r) : static_cast<int32_t>(r);
        const int64_t abeg = __ldg(L.a_rowptr + i), aend = __ldg(L.a_rowptr + i + 1);
        int32_t cnt = 0;
        bool over = false;
        for (int64_t p = abeg; p < aend && !over; ++p) {
            const int32_t j = __ldg(L.a_cols + p);
            const int64_t bb = __ldg(L.b_rowptr + j);
            const int32_t bl = kCompressed ? __ldg(L.csize + j) : static_cast<int32_t>(__ldg(L.b_rowptr + j + 1) - bb);
            for (int32_t q = 0; q < bl; ++q) {
                int32_t key;
                uint32_t word;
                if constexpr (kCompressed) {
                    const int2 pr = __ldg(cpair + bb + q);
                    key = pr.x;
                    word = static_cast<uint32_t>(pr.y);
                } else {
                    key = __ldg(L.b_cols + bb + q);
                    word = 1u;
                }
                int t = 0;
                while (t < cnt && skeys[t][tid] != key)
                    ++t;
                if (t < cnt) {
                    swords[t][tid] |= word;
                } else if (cnt < kTinySymKeys) {
                    skeys[cnt][tid] = key;
                    swords[cnt][tid] = word;
                    ++cnt;
                } else {
                    over = true; // cannot happen for a row in this class (bound <= kTinySymKeys)
                    break;
                }
            }
        }
        if (over) {
            if (retry_list)
                retry_list[atomicAdd(retry_count, 1ull)] = i;
            else
                raise_error(L.ctr, kDevRowOverflow);
            continue;
        }
        int64_t size = 0;
        for (int t = 0; t < cnt; ++t)
            size += kCompressed ? __popc(swords[t][tid]) : 1;
        L.sym_sizes[i] = size;
    }
}

int tiny_grid(int64_t nrows)
{
    const int64_t want = (nrows + kTinyThreads - 1) / kTinyThreads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t{sm_count()} * 16)));
}

} // namespace

cudaError_t launch_numeric_tiny(const RowLaunch& L, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    numeric_tiny_kernel<<<tiny_grid(L.nrows), kTinyThreads, 0, st>>>(L);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_symbolic_tiny(const RowLaunch& L, bool compressed, unsigned long long* retry_count,
                                 int32_t* retry_list, cudaStream_t st)
{
    if (L.nrows <= 0)
        return cudaSuccess;
    if (compressed)
        symbolic_tiny_kernel<true><<<tiny_grid(L.nrows), kTinyThreads, 0, st>>>(L, retry_count, retry_list);
    else
        symbolic_tiny_kernel<false><<<tiny_grid(L.nrows), kTinyThreads, 0, st>>>(L, retry_count, retry_list);
    count_launch();
    return cudaGetLastError();
}

} // namespace kk
