// Structure-reuse replay of the numeric phase (sm_100a).
//
// The reference's reuse contract (engine.hpp:42-56, cli.cpp:137-151): one
// symbolic pass, then numeric passes as the values change.  Every numeric
// pass of the reference re-derives where each product lands in its C row by
// probing the accumulator (engine.cpp:259-267).  With the structure fixed,
// that slot is a function of the structure alone, so after the second numeric
// pass on a handle the slot of every product is recorded once:
//
//   slot map      one byte (rows <= 256 entries) or two bytes per product, in
//                 the product order of the Thread-Sequential walk (A entry p,
//                 then B-row entry t) — the order of the row's flops;
//   column cache  C's column indices in first-touch order (4 B per entry).
//
// Later passes run replay_numeric_kernel: per product one map byte, one B
// value and an unfused multiply + add onto acc[slot] in shared memory — no
// key loads, probes or claims.  The first product of a slot lands on -0.0
// (-0.0 + v == v bitwise, including v = +0.0 and NaN payloads) and the rest
// are added in product order, so values are bitwise those of the hashing
// kernels (and of the reference's raw output).
//
// The map is valid only for the structure it was recorded on.  The reference
// checks dimensions and nnz only (engine.cpp:451-453); the replay path also
// fingerprints A's and B's row offsets and column indices (64-bit sums of
// a non-linear hash of (position, value), relative to the row-offset base so row-block views
// fingerprint like the matrix they were cut from) on every pass.  The replay
// kernel and the hashing kernels are both launched and both read the
// fingerprints: exactly one of them does the work, with no host round trip.
#include <cstdint>

#include "kk_device.cuh"
#include "kk_internal.h"

namespace kk {

namespace {

// Order-independent sum of a NON-linear per-element hash:
//   element idx with value x contributes mix64(w(idx) ^ x)   (mod 2^64),
// w(idx) = 2K*idx + 1 an odd (bijective) position weight and mix64 the
// splitmix64 finalizer.  A moment checksum (sum of w(idx) * x) would be blind
// to edits that preserve two moments of the column array (e.g. two adjacent
// swaps with opposite column gaps in different rows); through the mixer every
// changed (position, value) pair moves the sum by an unrelated 64-bit amount,
// so a structural edit goes undetected with probability ~2^-64 whatever its
// shape.  Threads still combine partial sums in any order.
constexpr uint64_t kFpK2 = 0x3C6EF372FE94F82Aull; // 2 * 0x9E3779B97F4A7C15 (mod 2^64)

__device__ __forceinline__ uint64_t fp_weight(int64_t idx)
{
    return static_cast<uint64_t>(idx) * kFpK2 + 1ull;
}

__device__ __forceinline__ uint64_t fp_mix(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ uint64_t fp_term(uint64_t w, uint64_t x) { return fp_mix(w ^ x); }

// sum over (i, rowptr[i] - rowptr[0]) and (q, cols[rowptr[0] + q]); the row
// offsets are weighted from index nnz + 1 on so they never share weights with
// the columns.  Added into out0 (and out1 when A and B are the same arrays).
__global__ void __launch_bounds__(256) fingerprint_kernel(int64_t rows, const int64_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ cols,
                                                          unsigned long long* out0, unsigned long long* out1)
{
    const int64_t base = __ldg(rowptr);
    const int64_t nnz = __ldg(rowptr + rows) - base;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (int64_t i = tid; i <= rows; i += stride)
        acc += fp_term(fp_weight(nnz + 1 + i), static_cast<uint64_t>(__ldg(rowptr + i) - base));
    // columns: four per thread per iteration (int4 once 16-byte aligned)
    const int32_t* c = cols + base;
    const uintptr_t mis = reinterpret_cast<uintptr_t>(c) & 15;
    const int64_t head = mis ? static_cast<int64_t>((16 - mis) >> 2) : 0;
    const int64_t h = head < nnz ? head : nnz;
    for (int64_t q = tid; q < h; q += stride)
        acc += fp_term(fp_weight(q), static_cast<uint32_t>(__ldg(c + q)));
    const int64_t nvec = (nnz - h) >> 2;
    const int4* v = reinterpret_cast<const int4*>(c + h);
    uint64_t w = fp_weight(h + 4 * tid);
    const uint64_t wstep = 4ull * static_cast<uint64_t>(stride) * kFpK2;
    for (int64_t q = tid; q < nvec; q += stride, w += wstep) {
        // two adjacent columns per mixed term (the weight is the first one's):
        // still an injective (position, value) input, half the mixing work
        const int4 x = __ldg(v + q);
        acc += fp_term(w, static_cast<uint32_t>(x.x) | (static_cast<uint64_t>(static_cast<uint32_t>(x.y)) << 32))
            + fp_term(w + 2 * kFpK2,
                      static_cast<uint32_t>(x.z) | (static_cast<uint64_t>(static_cast<uint32_t>(x.w)) << 32));
    }
    for (int64_t q = h + 4 * nvec + tid; q < nnz; q += stride)
        acc += fp_term(fp_weight(q), static_cast<uint32_t>(__ldg(c + q)));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
        acc += __shfl_xor_sync(kFull, acc, off);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out0, static_cast<unsigned long long>(acc));
        if (out1)
            atomicAdd(out1, static_cast<unsigned long long>(acc));
    }
}

struct StepStageR {
    longlong2 row[32]; // x = B row offset, y = B row length
    double a[32];
};

// Record each product's slot: the C row's first-touch columns go into a
// per-warp hash (column -> position), then the row's products are walked in
// Thread-Sequential order and looked up.  Also fills the column cache.
template <typename PosT>
__global__ void __launch_bounds__(256) replay_build_kernel(const ReplayLaunch R)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    int32_t* keys = reinterpret_cast<int32_t*>(smem + (size_t)wib * R.warp_bytes);
    int32_t* posv = keys + R.T;
    const uint32_t tmask = static_cast<uint32_t>(R.T - 1);
    for (int t = lane; t < R.T; t += 32)
        keys[t] = kEmpty;
    __syncwarp();
    PosT* map = static_cast<PosT*>(R.map);
    const int64_t nwarps = (int64_t)gridDim.x * R.wpb;
    for (int64_t i = (int64_t)blockIdx.x * R.wpb + wib; i < R.m; i += nwarps) {
        const int64_t cbase = __ldg(R.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(R.c_rowptr + i + 1) - cbase);
        if (cap == 0)
            continue;
        for (int32_t q = lane; q < cap; q += 32) {
            const int32_t key = R.c_cols[cbase + q];
            R.ccache[cbase + q] = key;
            uint32_t s = hash_slot(key, R.shift);
            while (atomicCAS(&keys[s], kEmpty, key) != kEmpty)
                s = (s + 1) & tmask;
            posv[s] = q;
        }
        __syncwarp();
        int64_t poff = __ldg(R.prod_off + i);
        const int64_t abeg = __ldg(R.a_rowptr + i), aend = __ldg(R.a_rowptr + i + 1);
        for (int64_t p = abeg; p < aend; ++p) {
            const int32_t j = __ldg(R.a_cols + p);
            const int64_t b0 = __ldg(R.b_rowptr + j);
            const int64_t len = __ldg(R.b_rowptr + j + 1) - b0;
            for (int64_t t = lane; t < len; t += 32) {
                const int32_t key = __ldg(R.b_cols + b0 + t);
                uint32_t s = hash_slot(key, R.shift);
                int32_t k = keys[s];
                int probes = 0;
                while (k != key && k != kEmpty && probes++ < R.T) {
                    s = (s + 1) & tmask;
                    k = keys[s];
                }
                PosT pos = 0;
                if (k == key)
                    pos = static_cast<PosT>(posv[s]);
                else
                    raise_error(R.ctr, kDevReplay);
                map[poff + t] = pos;
            }
            poff += len;
        }
        __syncwarp();
        for (int32_t q = lane; q < cap; q += 32) {
            const int32_t key = R.c_cols[cbase + q];
            uint32_t s = hash_slot(key, R.shift);
            while (keys[s] != key)
                s = (s + 1) & tmask;
            keys[s] = kEmpty;
        }
        __syncwarp();
    }
}

// Replay: warp per C row, Thread-Sequential steps (one B row per step, lanes
// over its entries, so slots within a step are distinct), depth-2 register
// prefetch of (slot, B value) like numeric_lp_seq_kernel.
template <typename PosT>
__global__ void __launch_bounds__(256) replay_numeric_kernel(const ReplayLaunch R)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* region = smem + (size_t)wib * R.warp_bytes;
    StepStageR* stage = reinterpret_cast<StepStageR*>(region);
    double* acc = reinterpret_cast<double*>(region + sizeof(StepStageR));
    if (R.gate && !(R.gate[0] == R.gate[2] && R.gate[1] == R.gate[3]))
        return; // structure changed since the map was recorded: the hashing kernels run
    const PosT* __restrict__ map = static_cast<const PosT*>(R.map);
    const double* __restrict__ b_vals = R.b_vals;
    const uint64_t pol = l2_keep_policy(); // B values stay in L2; the map and C stream
    const int64_t nwarps = (int64_t)gridDim.x * R.wpb;
    for (int64_t i = R.row_lo + (int64_t)blockIdx.x * R.wpb + wib; i < R.row_hi; i += nwarps) {
        const int64_t cbase = __ldg(R.c_rowptr + i);
        const int32_t cap = static_cast<int32_t>(__ldg(R.c_rowptr + i + 1) - cbase);
        if (cap == 0)
            continue;
        for (int32_t q = lane; q < cap; q += 32)
            acc[q] = -0.0;
        int64_t poff = __ldg(R.prod_off + i);
        const int64_t abeg = __ldg(R.a_rowptr + i), aend = __ldg(R.a_rowptr + i + 1);
        bool bad = false;
        for (int64_t p0 = abeg; p0 < aend; p0 += 32) {
            const int na = static_cast<int>(aend - p0 < 32 ? aend - p0 : 32);
            int32_t bl = 0;
            if (lane < na) {
                const int32_t j = __ldg(R.a_cols + p0 + lane);
                const int64_t b0 = __ldg(R.b_rowptr + j);
                bl = static_cast<int32_t>(__ldg(R.b_rowptr + j + 1) - b0);
                stage->row[lane] = make_longlong2(b0, bl);
                stage->a[lane] = __ldg(R.a_vals + p0 + lane);
            } else {
                stage->row[lane] = make_longlong2(0, 0);
            }
            const bool long_rows = __any_sync(kFull, bl > 32);
            __syncwarp();
            if (long_rows) {
                for (int q = 0; q < na; ++q) {
                    const longlong2 rq = stage->row[q];
                    const double a = stage->a[q];
                    for (int64_t t = lane; t < rq.y; t += 32) {
                        const int32_t s = static_cast<int32_t>(__ldcs(map + poff + t));
                        const double v = __dmul_rn(a, ldg_keep(b_vals + rq.x + t, pol));
                        if (s < cap)
                            acc[s] = __dadd_rn(acc[s], v);
                        else
                            bad = true;
                    }
                    poff += rq.y;
                    __syncwarp();
                }
                continue;
            }
            // depth-2 pipeline; rows of the stage past na have length 0
            int32_t s0 = 0, s1 = 0, len0, len1;
            double v0 = 0.0, v1 = 0.0;
            int64_t o1, o2;
            {
                const longlong2 r0 = stage->row[0];
                const longlong2 r1 = stage->row[1];
                len0 = static_cast<int32_t>(r0.y);
                len1 = static_cast<int32_t>(r1.y);
                o1 = poff + len0;
                o2 = o1 + len1;
                if (lane < len0) {
                    s0 = __ldcs(map + poff + lane);
                    v0 = ldg_keep(b_vals + r0.x + lane, pol);
                }
                if (lane < len1) {
                    s1 = __ldcs(map + o1 + lane);
                    v1 = ldg_keep(b_vals + r1.x + lane, pol);
                }
            }
            for (int q = 0; q < na; ++q) {
                int32_t s2 = 0, len2 = 0;
                double v2 = 0.0;
                if (q + 2 < 32) {
                    const longlong2 r2 = stage->row[q + 2];
                    len2 = static_cast<int32_t>(r2.y);
                    if (lane < len2) {
                        s2 = __ldcs(map + o2 + lane);
                        v2 = ldg_keep(b_vals + r2.x + lane, pol);
                    }
                }
                if (lane < len0) {
                    const double v = __dmul_rn(stage->a[q], v0);
                    if (s0 < cap)
                        acc[s0] = __dadd_rn(acc[s0], v);
                    else
                        bad = true;
                }
                __syncwarp();
                s0 = s1;
                v0 = v1;
                len0 = len1;
                s1 = s2;
                v1 = v2;
                len1 = len2;
                o2 += len2;
            }
            {
                // products of this chunk: sum of the staged lengths
                int32_t tot = bl;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    tot += __shfl_xor_sync(kFull, tot, off);
                poff += tot;
            }
            __syncwarp();
        }
        if (__any_sync(kFull, bad) && lane == 0)
            raise_error(R.ctr, kDevReplay);
        for (int32_t q = lane; q < cap; q += 32) {
            st_stream(R.c_cols + cbase + q, __ldcs(R.ccache + cbase + q));
            st_stream(R.c_vals + cbase + q, acc[q]);
        }
        __syncwarp();
    }
}

template <typename K>
int blocks_per_sm(K kernel, int threads, size_t smem)
{
    const void* fn = reinterpret_cast<const void*>(kernel);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess)
        return 1;
    return b > 0 ? b : 1;
}

template <typename K>
cudaError_t launch_rows(K kernel, ReplayLaunch R, int64_t rows, cudaStream_t st)
{
    if (rows <= 0)
        return cudaSuccess;
    const size_t smem = (size_t)R.wpb * R.warp_bytes;
    const int per_sm = blocks_per_sm(kernel, R.wpb * 32, smem);
    const int64_t want = (rows + R.wpb - 1) / R.wpb;
    const int64_t fit = (int64_t)per_sm * sm_count();
    const int grid = static_cast<int>(want < fit ? want : fit);
    kernel<<<grid, R.wpb * 32, smem, st>>>(R);
    count_launch();
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_fingerprint(int64_t rows, const int64_t* rowptr, const int32_t* cols, unsigned long long* out0,
                               unsigned long long* out1, cudaStream_t st)
{
    const int grid = sm_count() * 4;
    fingerprint_kernel<<<grid, 256, 0, st>>>(rows, rowptr, cols, out0, out1);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_replay_build(ReplayLaunch R, int width, cudaStream_t st)
{
    R.warp_bytes = 8ull * R.T; // keys[T] + positions[T]
    R.wpb = static_cast<int>(R.warp_bytes >= 12288 ? 1 : 98304 / R.warp_bytes < 8 ? 98304 / R.warp_bytes : 8);
    return width == 1 ? launch_rows(replay_build_kernel<uint8_t>, R, R.m, st)
                      : launch_rows(replay_build_kernel<uint16_t>, R, R.m, st);
}

cudaError_t launch_replay_numeric(ReplayLaunch R, int width, int32_t max_row, cudaStream_t st)
{
    R.wpb = 8;
    R.warp_bytes = (sizeof(StepStageR) + 8ull * (max_row > 0 ? max_row : 1) + 15) & ~15ull;
    const int64_t rows = R.row_hi - R.row_lo;
    return width == 1 ? launch_rows(replay_numeric_kernel<uint8_t>, R, rows, st)
                      : launch_rows(replay_numeric_kernel<uint16_t>, R, rows, st);
}

} // namespace kk
