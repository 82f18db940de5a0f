// k_pool.cu — fused Gather + Stitch + SegmentReduction for one pack (PAPER.md L211-215,
// L380-382 "Shuffle&Stitch ... remove the explicit stitch kernel").
//
//   out[b, col(f) + d] = sum_{j in seg(f,b)} W[key_j][d]   (ascending j from +0.0f; mean: / len;
//                                                          empty segment: 0)
//
// Work decomposition (memory-level parallelism independent of the bag-length mix):
//  - a warp owns a tile of 32 consecutive segments of the pack in field-major order (k, b): the
//    tile's offsets are one coalesced load and its IDs one contiguous range;
//  - the warp splits into R = 32 / LANES row groups (LANES = D/4 lanes; each lane owns float4
//    columns, so a D = 128 row is one coalesced 512-B request); group g takes SPG = 32/R
//    consecutive segments of the tile;
//  - the group's (segment, j) pairs form one flattened stream; each lane resolves a different
//    pair (segment by a 5-step search over the tile's length prefix, raw ID, row hash, row
//    address), so the scalar work is spread over the lanes instead of repeated by all of them;
//  - addresses are broadcast with width-LANES shuffles and U rows are loaded at once (8 x 512 B
//    per warp at D = 128), then added strictly in ascending j per segment (bit-identical to the
//    sequential definition); a finished segment is written into its column block of the
//    stitched [B, out_width] output with streaming 128-bit stores.
// (seg_of, the segment of every packed-stream position, is written by k_seg_of beforehand.)
#include "kernels.h"

namespace picasso {

template <int D>
struct PoolGeo {
    static constexpr int V4 = D / 4;
    static constexpr int LANES = V4 < 32 ? V4 : 32;
    static constexpr int VPL = V4 / LANES;
    static constexpr int R = 32 / LANES;               // row groups per warp
    static constexpr int SPG = 32 / R;                 // segments per group per tile
    static constexpr int U = 8;                        // rows in flight per group
    static constexpr int PPL = U > LANES ? U / LANES : 1;  // pairs resolved per lane per round
    static constexpr int RND = LANES * PPL;            // pairs resolved per round (>= U)
};

struct SegTile {
    int32_t cum[8][64];   // per warp: per group, exclusive prefix of its SPG segment lengths
    int32_t o0[8][32];
    int32_t sg[8][32];
    int32_t gb[8][32];    // packed position = j + gb
    int64_t out[8][32];   // out offset of the segment's column block
    int64_t base[8][32];  // table base of the segment's field
    int64_t rows[8][32];
    uint64_t salt[8][32];
};

template <int D>
__device__ __forceinline__ void flush_seg(const PoolArgs &a, float4 *acc, int64_t out_off, int32_t len, int li) {
    constexpr int LANES = PoolGeo<D>::LANES, VPL = PoolGeo<D>::VPL;
    float *o = a.out + out_off + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        if (a.pool_mean && len > 0) acc[q] = div4(acc[q], (float)len);
        stcs_f4(o + q * LANES * 4, acc[q]);
        acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_pool(PoolArgs a) {
    using Gm = PoolGeo<D>;
    constexpr int LANES = Gm::LANES, VPL = Gm::VPL, SPG = Gm::SPG, U = Gm::U, PPL = Gm::PPL, RND = Gm::RND;
    __shared__ SegTile st;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int li = lane % LANES, grp = lane / LANES;
    const unsigned gmask = (LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << (grp * LANES));
    const int64_t S = (int64_t)a.Fp * a.B;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * 32; t0 < S; t0 += nwarps * 32) {
        // ---- tile descriptors: lane i <- segment t0 + i
        int32_t len = 0;
        {
            const int64_t s = t0 + lane;
            if (s < S) {
                const int32_t k = (int32_t)(s / a.B);
                const int32_t b = (int32_t)(s - (int64_t)k * a.B);
                const int32_t f = __ldg(a.pack_fields + k);
                const int32_t sg = f * a.B + b;
                const int32_t o0 = __ldg(a.offsets + sg);
                len = __ldg(a.offsets + sg + 1) - o0;
                const FieldInfo fi = a.finfo[f];
                st.o0[w][lane] = o0;
                st.sg[w][lane] = sg;
                st.gb[w][lane] = __ldg(a.field_gstart + f) - __ldg(a.id_start + f);
                st.out[w][lane] = (int64_t)b * a.out_stride + fi.col;
                st.base[w][lane] = fi.base;
                st.rows[w][lane] = fi.rows;
                st.salt[w][lane] = fi.salt;
            }
            // group-local inclusive scan of the lengths -> exclusive prefix in cum
            int32_t x = len;
#pragma unroll
            for (int o = 1; o < SPG; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, x, o, SPG);
                if ((lane % SPG) >= o) x += y;
            }
            st.cum[w][lane + (lane / SPG) + 1] = x;  // group g's prefix lives at [g*(SPG+1) ...]
            if (lane % SPG == 0) st.cum[w][lane + lane / SPG] = 0;
        }
        __syncwarp();
        const int nseg = (int)((S - t0) < 32 ? (S - t0) : 32);
        const int c_lo = grp * SPG, c_hi = min(nseg, c_lo + SPG);
        const int32_t *cum = &st.cum[w][grp * (SPG + 1)];  // cum[c - c_lo]
        const int32_t total = c_hi > c_lo ? cum[c_hi - c_lo] : 0;
        float4 acc[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        int cur = c_lo;
        const float *wb = a.weight + (int64_t)li * 4;
        for (int32_t q0 = 0; q0 < total; q0 += RND) {
            // ---- each lane resolves PPL pairs of the group's flattened stream
            int64_t myrow[PPL];
            int32_t myseg[PPL];
#pragma unroll
            for (int p = 0; p < PPL; ++p) {
                const int32_t q = q0 + p * LANES + li;
                myseg[p] = c_hi;
                myrow[p] = 0;
                if (q < total) {
                    int lo = 0, hi = c_hi - c_lo;  // last c with cum[c] <= q
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (cum[mid] <= q) lo = mid; else hi = mid;
                    }
                    const int c = c_lo + lo;
                    const int32_t j = st.o0[w][c] + (q - cum[lo]);
                    FieldInfo fi;
                    fi.base = st.base[w][c];
                    fi.rows = st.rows[w][c];
                    fi.salt = st.salt[w][c];
                    // float offset of the row: the local table (W = 1), or the row received for
                    // the position's unique key (W > 1: the stitched Shuffle output)
                    myrow[p] = a.row_off ? a.row_off[__ldg(a.inverse + j + st.gb[w][c])]
                                         : (fi.base + row_of(a.id_mode, __ldg(a.ids + j), fi, a.err)) * D;
                    myseg[p] = c;
                }
            }
            // ---- U rows at a time: broadcast addresses, load, add in ascending order
            const int32_t nround = min(RND, total - q0);
#pragma unroll 1
            for (int k0 = 0; k0 < nround; k0 += U) {
                float4 v[U][VPL];
                int sk[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    // PPL > 1 only when RND == U (k0 == 0): the slot index stays static
                    const int src = (k0 + k) % LANES, slot = PPL > 1 ? k / LANES : 0;
                    const int64_t r = __shfl_sync(gmask, myrow[slot], src, LANES);
                    sk[k] = __shfl_sync(gmask, myseg[slot], src, LANES);
                    if (k0 + k < nround) {
#pragma unroll
                        for (int qq = 0; qq < VPL; ++qq) v[k][qq] = ldg_f4(wb + r + qq * LANES * 4);
                    }
                }
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    if (k0 + k < nround) {
                        while (cur < sk[k]) {
                            flush_seg<D>(a, acc, st.out[w][cur], cum[cur - c_lo + 1] - cum[cur - c_lo], li);
                            ++cur;
                        }
#pragma unroll
                        for (int qq = 0; qq < VPL; ++qq) acc[qq] = add4(acc[qq], v[k][qq]);
                    }
                }
            }
        }
        while (cur < c_hi) {  // the last segment and trailing empty ones
            flush_seg<D>(a, acc, st.out[w][cur], cum[cur - c_lo + 1] - cum[cur - c_lo], li);
            ++cur;
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
