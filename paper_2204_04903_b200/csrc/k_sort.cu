// k_sort.cu — device-wide exclusive scan (reduce-then-scan, three launches), used by the
// HybridHash refresh's tie ranking.  The backward's transpose (the stable radix sort of
// (uid, segment) pairs) lives in k_sort2.cu.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.h"

namespace picasso {

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

}  // namespace picasso
