// k_pool.cu — fused Gather + Stitch + SegmentReduction for one pack (PAPER.md L211-215,
// L380-382 "Shuffle&Stitch ... remove the explicit stitch kernel").
//
//   out[b, col(f) + d] = sum_{j in seg(f,b)} W[key_j][d]   (ascending j from +0.0f; mean: / len;
//                                                          empty segment: 0)
//
// Work decomposition (memory-level parallelism independent of the bag-length mix):
//  - a warp owns a tile of 32 consecutive segments of the pack in field-major order (k, b), so
//    the tile's offsets are one coalesced load and its IDs one contiguous range;
//  - the warp splits into R = 32 / LANES row groups (LANES = D/4 lanes, each lane owns float4
//    columns: a D = 128 row is one coalesced 512-B request);
//  - each group walks the flattened (segment, j) stream of its 32/R segments and issues U row
//    loads at a time (8 at D = 128: 4 KB in flight per warp) regardless of where segment
//    boundaries fall — one-hot and 50-hot bags keep the same number of loads in flight;
//  - rows are then added strictly in ascending j per segment (bit-identical to the
//    sequential definition); a finished segment is written straight into its column block of
//    the stitched [B, out_width] output with streaming 128-bit stores.
// The same walk records seg_of[g] (segment of every packed-stream position) for the backward.
#include "kernels.h"

namespace picasso {

template <int D>
struct PoolGeo {
    static constexpr int V4 = D / 4;
    static constexpr int LANES = V4 < 32 ? V4 : 32;
    static constexpr int VPL = V4 / LANES;
    static constexpr int R = 32 / LANES;    // row groups per warp
    static constexpr int SPG = 32 / R;      // segments per group per tile
    static constexpr int U = D >= 64 ? 8 : 4;  // rows in flight per group
};

template <int D>
__global__ void __launch_bounds__(256) k_pool(PoolArgs a) {
    using Gm = PoolGeo<D>;
    constexpr int LANES = Gm::LANES, VPL = Gm::VPL, SPG = Gm::SPG, U = Gm::U;
    __shared__ int32_t s_o0[8][32], s_o1[8][32], s_gb[8][32], s_sg[8][32], s_f[8][32];
    __shared__ int64_t s_out[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int li = lane % LANES, grp = lane / LANES;
    const int64_t S = (int64_t)a.Fp * a.B;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; t0 < S; t0 += nwarps * 32) {
        // ---- tile descriptors: lane i <- segment t0 + i
        {
            const int64_t s = t0 + lane;
            int32_t o0 = 0, o1 = 0, gb = 0, sg = 0, f = 0;
            int64_t ob = 0;
            if (s < S) {
                const int32_t k = (int32_t)(s / a.B);
                const int32_t b = (int32_t)(s - (int64_t)k * a.B);
                f = __ldg(a.pack_fields + k);
                sg = f * a.B + b;
                o0 = __ldg(a.offsets + sg);
                o1 = __ldg(a.offsets + sg + 1);
                gb = __ldg(a.field_gstart + f) - __ldg(a.id_start + f);  // g = j + gb
                ob = (int64_t)b * a.out_stride + a.finfo[f].col;
            }
            s_o0[wib][lane] = o0;
            s_o1[wib][lane] = o1;
            s_gb[wib][lane] = gb;
            s_sg[wib][lane] = sg;
            s_f[wib][lane] = f;
            s_out[wib][lane] = ob;
        }
        __syncwarp();
        const int nseg = (int)((S - t0) < 32 ? (S - t0) : 32);
        const int c_lo = grp * SPG, c_hi = min(nseg, c_lo + SPG);
        // field info of the group's first segment; refreshed when the field changes
        int cur = c_lo;
        int32_t j = cur < c_hi ? s_o0[wib][cur] : 0, e = cur < c_hi ? s_o1[wib][cur] : 0;
        float4 acc[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float *wb = a.weight + (int64_t)li * 4;
        while (cur < c_hi) {
            // ---- collect up to U (segment, j) pairs of the flattened stream
            int bseg[U];
            int32_t bj[U];
            int n = 0;
            {
                int c2 = cur;
                int32_t j2 = j, e2 = e;
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    while (j2 >= e2 && c2 < c_hi) {
                        ++c2;
                        if (c2 < c_hi) {
                            j2 = s_o0[wib][c2];
                            e2 = s_o1[wib][c2];
                        }
                    }
                    bseg[k] = c2;
                    bj[k] = j2;
                    if (c2 < c_hi) {
                        ++n;
                        ++j2;
                    }
                }
            }
            // ---- issue the row loads (keys recomputed from the raw IDs)
            float4 v[U][VPL];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (k < n) {
                    const FieldInfo fi = a.finfo[s_f[wib][bseg[k]]];
                    const int64_t r = fi.base + row_of(a.id_mode, __ldg(a.ids + bj[k]), fi, a.err);
#pragma unroll
                    for (int q = 0; q < VPL; ++q) v[k][q] = ldg_f4(wb + r * D + q * LANES * 4);
                    if (li == 0) a.seg_of[bj[k] + s_gb[wib][bseg[k]]] = s_sg[wib][bseg[k]];
                }
            }
            // ---- accumulate in ascending j; flush finished (and empty) segments
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (k < n) {
                    while (cur < bseg[k]) {
                        const int32_t len = s_o1[wib][cur] - s_o0[wib][cur];
                        float *o = a.out + s_out[wib][cur] + li * 4;
#pragma unroll
                        for (int q = 0; q < VPL; ++q) {
                            if (a.pool_mean && len > 0) acc[q] = div4(acc[q], (float)len);
                            stcs_f4(o + q * LANES * 4, acc[q]);
                            acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        ++cur;
                    }
#pragma unroll
                    for (int q = 0; q < VPL; ++q) acc[q] = add4(acc[q], v[k][q]);
                }
            }
            if (n < U) {  // stream exhausted: flush the rest
                while (cur < c_hi) {
                    const int32_t len = s_o1[wib][cur] - s_o0[wib][cur];
                    float *o = a.out + s_out[wib][cur] + li * 4;
#pragma unroll
                    for (int q = 0; q < VPL; ++q) {
                        if (a.pool_mean && len > 0) acc[q] = div4(acc[q], (float)len);
                        stcs_f4(o + q * LANES * 4, acc[q]);
                        acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    ++cur;
                }
            } else {
                cur = bseg[U - 1];
                j = bj[U - 1] + 1;
                e = s_o1[wib][cur];
            }
        }
        __syncwarp();
    }
}

void launch_pool(int D, const PoolArgs &a, int num_sms, cudaStream_t s) {
    const int64_t S = (int64_t)a.Fp * a.B;
    if (S == 0) return;
    int64_t blocks = (S + 255) / 256;  // 8 warps x 32 segments per block
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
