// k_pool.cu — fused Gather + Stitch + SegmentReduction for one pack (PAPER.md L211-215,
// L380-382 "Shuffle&Stitch ... remove the explicit stitch kernel").
//
//   out[b, col(f) + d] = sum_{j in seg(f,b)} W[key_j][d]   (ascending j from +0.0f; mean: / len)
//
// One sub-warp of D/4 lanes (<= 32) per segment; each lane owns float4 columns, so a row is
// read with coalesced 128-bit loads (one 512-B request per warp at D = 128) and the pooled
// row is written with streaming 128-bit stores straight into the stitched output (the
// field's column block of the [B, out_width] matrix).  Row addresses of four consecutive
// IDs are computed first and their loads issued together (memory-level parallelism); the
// adds then run in ascending j, so the result is bit-identical to the sequential definition.
// Segments are walked sample-major (b, then the pack's fields) so adjacent sub-warps write
// adjacent column blocks.  Persistent grid-stride launch sized to the SM count.
#include "kernels.h"

namespace picasso {

template <int D>
__global__ void __launch_bounds__(256) k_pool(PoolArgs a) {
    constexpr int V4 = D / 4;
    constexpr int LANES = V4 < 32 ? V4 : 32;
    constexpr int VPL = V4 / LANES;
    constexpr int U = 4;
    const int li = threadIdx.x % LANES;
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    const int64_t S = (int64_t)a.Fp * a.B;
    for (int64_t s = grp; s < S; s += ngrp) {
        const int32_t b = (int32_t)(s / a.Fp);
        const int32_t k = (int32_t)(s - (int64_t)b * a.Fp);
        const int32_t f = __ldg(a.pack_fields + k);
        const FieldInfo fi = a.finfo[f];
        const int64_t sg = (int64_t)f * a.B + b;
        const int32_t j0 = __ldg(a.offsets + sg), j1 = __ldg(a.offsets + sg + 1);
        const float *wb = a.weight + (int64_t)li * 4;
        float4 acc[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        int32_t j = j0;
        for (; j + U <= j1; j += U) {
            int64_t r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = fi.base + row_of(a.id_mode, __ldg(a.ids + j + u), fi, a.err);
            float4 v[U][VPL];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < VPL; ++q) v[u][q] = ldg_f4(wb + r[u] * D + q * LANES * 4);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < VPL; ++q) acc[q] = add4(acc[q], v[u][q]);
        }
        for (; j < j1; ++j) {
            const int64_t r = fi.base + row_of(a.id_mode, __ldg(a.ids + j), fi, a.err);
#pragma unroll
            for (int q = 0; q < VPL; ++q) acc[q] = add4(acc[q], ldg_f4(wb + r * D + q * LANES * 4));
        }
        if (a.pool_mean && j1 > j0) {
            const float len = (float)(j1 - j0);
#pragma unroll
            for (int q = 0; q < VPL; ++q) acc[q] = div4(acc[q], len);
        }
        float *o = a.out + (int64_t)b * a.out_stride + fi.col + li * 4;
#pragma unroll
        for (int q = 0; q < VPL; ++q) stcs_f4(o + q * LANES * 4, acc[q]);
    }
}

void launch_pool(int D, const PoolArgs &a, int num_sms, cudaStream_t s) {
    const int64_t S = (int64_t)a.Fp * a.B;
    if (S == 0) return;
    const int lanes = D / 4 < 32 ? D / 4 : 32;
    int64_t blocks = (S * lanes + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    switch (D) {
#define PICASSO_POOL_CASE(DD) \
    case DD: k_pool<DD><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        PICASSO_POOL_CASE(4)
        PICASSO_POOL_CASE(8)
        PICASSO_POOL_CASE(16)
        PICASSO_POOL_CASE(32)
        PICASSO_POOL_CASE(64)
        PICASSO_POOL_CASE(128)
        PICASSO_POOL_CASE(256)
        PICASSO_POOL_CASE(384)
        PICASSO_POOL_CASE(512)
#undef PICASSO_POOL_CASE
        default: break;
    }
}

}  // namespace picasso
