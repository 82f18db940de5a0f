// k_sort.cu — device-wide exclusive scan and a stable LSD radix sort of (uid, segment) pairs.
//
// The backward pass ("mirror image of the forward pass") needs, for every
// unique row, the list of its occurrences in ascending packed position — the transpose of
// the forward's inverse index.  A stable radix sort by uid over the packed stream gives it
// (ties keep ascending position), so per-row gradient sums follow the oracle's order.
//
// Per 8-bit pass (reduce-then-scan):
//   k_radix_hist    : per-tile digit histogram (warp-aggregated shared-memory counts),
//                     written digit-major so one exclusive scan gives every (digit, tile)
//                     its global output offset
//   scan            : three-phase device scan
//   k_radix_scatter : each warp ranks its contiguous 256 keys with __match_any_sync
//                     (stable: round, then lane), warps are prefixed per digit, then scatter
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.h"

namespace picasso {

constexpr int kRadix = 256;

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTileThreads) k_scan_reduce(const int32_t *in, int64_t n, int32_t *tile_sum) {
    using BlockReduce = cub::BlockReduce<int32_t, kTileThreads>;
    __shared__ typename BlockReduce::TempStorage tmp;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    int32_t s = 0;
    for (int i = threadIdx.x; i < kTile; i += kTileThreads) {
        const int64_t g = base + i;
        if (g < n) s += in[g];
    }
    s = BlockReduce(tmp).Sum(s);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k_scan_single(int32_t *x, int64_t n, int32_t *total) {
    __shared__ int32_t s_carry;
    using BlockScan = cub::BlockScan<int32_t, 1024>;
    __shared__ typename BlockScan::TempStorage tmp;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + threadIdx.x;
        int32_t v = i < n ? x[i] : 0, e, agg;
        BlockScan(tmp).ExclusiveSum(v, e, agg);
        if (i < n) x[i] = s_carry + e;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = s_carry;
}

__global__ void __launch_bounds__(kTileThreads) k_scan_down(const int32_t *in, int32_t *out, int64_t n,
                                                            const int32_t *tile_off) {
    using BlockScan = cub::BlockScan<int32_t, kTileThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    constexpr int IT = kTile / kTileThreads;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * IT;
    int32_t v[IT], s = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int32_t e;
    BlockScan(tmp).ExclusiveSum(s, e);
    e += tile_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        if (base + i < n) out[base + i] = e;
        e += v[i];
    }
}

size_t scan_scratch_ints(int64_t n) { return (size_t)((n + kTile - 1) / kTile) + 1; }

void launch_scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *scratch, int32_t *total,
                           cudaStream_t s) {
    const int64_t nt = (n + kTile - 1) / kTile;
    if (nt == 0) return;
    k_scan_reduce<<<(unsigned)nt, kTileThreads, 0, s>>>(in, n, scratch);
    k_scan_single<<<1, 1024, 0, s>>>(scratch, nt, total);
    k_scan_down<<<(unsigned)nt, kTileThreads, 0, s>>>(in, out, n, scratch);
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTileThreads) k_radix_hist(const int32_t *keys, int64_t n, int shift,
                                                             int32_t *hist, int64_t nblk) {
    __shared__ int32_t h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTile;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kTile; i += kTileThreads) {
        const int64_t g = base + i;
        const bool valid = g < n;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int d = (keys[g] >> shift) & (kRadix - 1);
            const unsigned peers = __match_any_sync(vm, d);
            if (lane == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kTileThreads) k_radix_scatter(const int32_t *kin, const int32_t *vin,
                                                                int32_t *kout, int32_t *vout, int64_t n,
                                                                int shift, const int32_t *hist_off,
                                                                int64_t nblk) {
    constexpr int kWarps = kTileThreads / 32;
    constexpr int kRounds = kTile / kTileThreads;  // 8 rounds of 32 keys per warp
    __shared__ int32_t wc[kWarps][kRadix];
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kTileThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * (32 * kRounds);
    int32_t key[kRounds], val[kRounds], rk[kRounds];
    int dg[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t g = base + r * 32 + lane;
        const bool valid = g < n;
        key[r] = valid ? kin[g] : 0;
        val[r] = valid ? vin[g] : 0;
        dg[r] = valid ? ((key[r] >> shift) & (kRadix - 1)) : (kRadix + lane);
        const unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
        int32_t before = 0;
        if (valid) before = wc[w][dg[r]];
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wc[w][dg[r]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // per digit: exclusive prefix across warps + global offset of (digit, tile)
        const int d = threadIdx.x;
        int32_t run = hist_off[(int64_t)d * nblk + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
            const int32_t t = wc[ww][d];
            wc[ww][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t g = base + r * 32 + lane;
        if (g < n) {
            const int32_t pos = wc[w][dg[r]] + rk[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
    }
}

size_t radix_hist_ints(int64_t n) { return (size_t)kRadix * (size_t)((n + kTile - 1) / kTile) + 1; }

void radix_sort_pairs(const int32_t *k_in, const int32_t *v_in, int32_t *k_a, int32_t *v_a, int32_t *k_b,
                      int32_t *v_b, int32_t **k_out, int32_t **v_out, int64_t n, int bits, int32_t *hist,
                      int32_t *scratch, cudaStream_t s, int64_t *launches) {
    const int64_t nblk = (n + kTile - 1) / kTile;
    const int32_t *ck = k_in, *cv = v_in;
    int32_t *bufk[2] = {k_a, k_b}, *bufv[2] = {v_a, v_b};
    int which = 0;
    if (bits < 1) bits = 1;
    for (int shift = 0; shift < bits; shift += 8) {
        if (nblk == 0) break;
        k_radix_hist<<<(unsigned)nblk, kTileThreads, 0, s>>>(ck, n, shift, hist, nblk);
        launch_scan_exclusive(hist, hist, (int64_t)kRadix * nblk, scratch, nullptr, s);
        k_radix_scatter<<<(unsigned)nblk, kTileThreads, 0, s>>>(ck, cv, bufk[which], bufv[which], n, shift, hist,
                                                                nblk);
        *launches += 5;
        ck = bufk[which];
        cv = bufv[which];
        which ^= 1;
    }
    *k_out = const_cast<int32_t *>(ck);
    *v_out = const_cast<int32_t *>(cv);
}

}  // namespace picasso
