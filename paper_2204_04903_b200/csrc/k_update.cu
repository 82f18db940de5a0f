// k_update.cu — backward of the packed lookup fused with the sparse optimizer update.
//
// The backward is the mirror image of the forward: SegmentReduction^T
// scatters dY[b, col(f)] (mean: dY / len) to every occurrence, and Unique^T sums the
// occurrences of each unique row:  G_u = sum_{j: inverse[j] = u} dY[seg(j)] * s(j).
// The optimizer (north star; readings O9/O10) then updates each touched row once:
//   Adagrad   acc += G*G;  w -= lr * (G / (sqrt(acc) + eps))
//   lazy Adam m += (G-m)(1-b1); v += (G*G-v)(1-b2); w -= ss * (m / (sqrt(v) + eps))
// Fusing the two keeps G in registers: per touched row the kernel reads dY rows once and
// the weight/state rows once, writes weight/state once (no G round trip through HBM).
// Each contribution is formed in fp32 (dY, dY/len) and accumulated in fp64, then rounded
// once to fp32 (reading O6): the result is fp32(exact sum) whatever the summation order, so
// the chunked hot-row path and the oracle agree even when G nearly cancels.
//
//   k_csr_bounds     : row boundaries in the uid-sorted occurrence list (ustart)
//   k_segsum_update  : one sub-warp per unique row with <= kLongRow occurrences; sums in
//                      ascending position
//   k_long_update    : one block per hot row (Zipf heads reach 1e4-1e6 occurrences): the
//                      block's sub-warps sum fixed strided chunks, combined in sub-warp order
//                      (deterministic), then one update
// All arithmetic uses explicit _rn intrinsics: no FMA contraction, IEEE sqrt and division.
#include "kernels.h"

namespace picasso {

__global__ void k_csr_bounds(const int32_t *su, int64_t N, int32_t *ustart) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int32_t u = su[i];
    if (i == 0 || su[i - 1] != u) ustart[u] = (int32_t)i;
    if (i == N - 1) ustart[u + 1] = (int32_t)N;
}

void launch_csr_bounds(const int32_t *sorted_u, int64_t N, int32_t *ustart, int32_t *long_cnt, cudaStream_t s) {
    cudaMemsetAsync(long_cnt, 0, sizeof(int32_t), s);
    if (N > 0) k_csr_bounds<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(sorted_u, N, ustart);
}

template <int D>
struct Geo {
    static constexpr int V4 = D / 4;
    static constexpr int LANES = V4 < 32 ? V4 : 32;
    static constexpr int VPL = V4 / LANES;
};

struct dbl4 {
    double x, y, z, w;
};
__device__ __forceinline__ dbl4 zero4d() { return dbl4{0.0, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ dbl4 add4d(dbl4 a, float4 b) {
    return dbl4{__dadd_rn(a.x, (double)b.x), __dadd_rn(a.y, (double)b.y), __dadd_rn(a.z, (double)b.z),
                __dadd_rn(a.w, (double)b.w)};
}
__device__ __forceinline__ dbl4 add4d(dbl4 a, dbl4 b) {
    return dbl4{__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z), __dadd_rn(a.w, b.w)};
}
__device__ __forceinline__ float4 round4(dbl4 a) {
    return make_float4(__double2float_rn(a.x), __double2float_rn(a.y), __double2float_rn(a.z),
                       __double2float_rn(a.w));
}

template <int VPL>
__device__ __forceinline__ void accumulate_one(const UpdateArgs &a, int32_t seg, const float *dyl, int LANES,
                                               dbl4 *g) {
    const int32_t f = seg / a.B;
    const int32_t b = seg - f * a.B;
    const float *p = dyl + (int64_t)b * a.dy_stride + a.finfo[f].col;
    float4 c[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) c[q] = ldg_f4(p + q * LANES * 4);
    if (a.pool_mean) {
        const float len = (float)(__ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg));
#pragma unroll
        for (int q = 0; q < VPL; ++q) c[q] = div4(c[q], len);
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], c[q]);
}

template <int D>
__device__ __forceinline__ void accumulate_range(const UpdateArgs &a, int32_t i0, int32_t i1, int32_t step,
                                                 int li, dbl4 *g) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const float *dyl = a.dy + li * 4;
    int32_t i = i0;
    // issue four independent dY row loads, then add in ascending order
    for (; i + 3 * step < i1; i += 4 * step) {
        int32_t sg[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sg[u] = __ldg(a.sorted_seg + i + u * step);
        float4 c[4][VPL];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t f = sg[u] / a.B;
            const int32_t b = sg[u] - f * a.B;
            const float *p = dyl + (int64_t)b * a.dy_stride + a.finfo[f].col;
#pragma unroll
            for (int q = 0; q < VPL; ++q) c[u][q] = ldg_f4(p + q * LANES * 4);
            if (a.pool_mean) {
                const float len = (float)(__ldg(a.offsets + sg[u] + 1) - __ldg(a.offsets + sg[u]));
#pragma unroll
                for (int q = 0; q < VPL; ++q) c[u][q] = div4(c[u][q], len);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], c[u][q]);
    }
    for (; i < i1; i += step) accumulate_one<VPL>(a, __ldg(a.sorted_seg + i), dyl, LANES, g);
}

template <int D>
__device__ __forceinline__ void apply_update(const UpdateArgs &a, int64_t row, int li, const float4 *g) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    float *w = a.weight + row * D + li * 4;
    float *s1 = a.state1 + row * D + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        float4 wv = *reinterpret_cast<float4 *>(w + q * LANES * 4);
        float4 sv = *reinterpret_cast<float4 *>(s1 + q * LANES * 4);
        const float gg[4] = {g[q].x, g[q].y, g[q].z, g[q].w};
        float ww[4] = {wv.x, wv.y, wv.z, wv.w};
        float ss[4] = {sv.x, sv.y, sv.z, sv.w};
        if (a.opt == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float acc = __fadd_rn(ss[e], __fmul_rn(gg[e], gg[e]));
                ss[e] = acc;
                const float qq = __fdiv_rn(gg[e], __fadd_rn(__fsqrt_rn(acc), a.eps));
                ww[e] = __fsub_rn(ww[e], __fmul_rn(a.lr, qq));
            }
        } else {
            float *s2 = a.state2 + row * D + li * 4;
            float4 vv = *reinterpret_cast<float4 *>(s2 + q * LANES * 4);
            float v2[4] = {vv.x, vv.y, vv.z, vv.w};
            const float omb1 = __fsub_rn(1.0f, a.beta1), omb2 = __fsub_rn(1.0f, a.beta2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float mo = ss[e], vo = v2[e];
                const float mu = __fmul_rn(__fsub_rn(gg[e], mo), omb1);
                const float vu = __fmul_rn(__fsub_rn(__fmul_rn(gg[e], gg[e]), vo), omb2);
                const float mn = __fadd_rn(mu, mo), vn = __fadd_rn(vu, vo);
                ss[e] = mn;
                v2[e] = vn;
                const float qq = __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), a.eps));
                ww[e] = __fsub_rn(ww[e], __fmul_rn(a.adam_ss, qq));
            }
            *reinterpret_cast<float4 *>(s2 + q * LANES * 4) = make_float4(v2[0], v2[1], v2[2], v2[3]);
        }
        *reinterpret_cast<float4 *>(w + q * LANES * 4) = make_float4(ww[0], ww[1], ww[2], ww[3]);
        *reinterpret_cast<float4 *>(s1 + q * LANES * 4) = make_float4(ss[0], ss[1], ss[2], ss[3]);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_segsum_update(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int li = threadIdx.x % LANES;
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    for (int64_t u = u0 + grp; u < u1; u += ngrp) {
        const int32_t i0 = __ldg(a.ustart + u), i1 = __ldg(a.ustart + u + 1);
        if (i1 - i0 > kLongRow) {
            if (li == 0) a.long_list[atomicAdd(a.long_cnt, 1)] = (int32_t)u;
            continue;
        }
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        accumulate_range<D>(a, i0, i1, 1, li, g);
        float4 g32[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g32[q] = round4(g[q]);
        const int64_t row = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off);
        apply_update<D>(a, row, li, g32);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_long_update(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    constexpr int G = 256 / LANES;
    __shared__ dbl4 part[G][LANES * VPL];
    const int li = threadIdx.x % LANES;
    const int gi = threadIdx.x / LANES;
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    const int32_t n = *a.long_cnt;
    for (int32_t e = blockIdx.x; e < n; e += gridDim.x) {
        const int32_t u = a.long_list[e];
        if (u < u0 || u >= u1) continue;  // block-uniform
        const int32_t i0 = __ldg(a.ustart + u), i1 = __ldg(a.ustart + u + 1);
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        accumulate_range<D>(a, i0 + gi, i1, G, li, g);
#pragma unroll
        for (int q = 0; q < VPL; ++q) part[gi][q * LANES + li] = g[q];
        __syncthreads();
        if (gi == 0) {
            dbl4 t[VPL];
#pragma unroll
            for (int q = 0; q < VPL; ++q) t[q] = part[0][q * LANES + li];
            for (int x = 1; x < G; ++x)
#pragma unroll
                for (int q = 0; q < VPL; ++q) t[q] = add4d(t[q], part[x][q * LANES + li]);
            float4 g32[VPL];
#pragma unroll
            for (int q = 0; q < VPL; ++q) g32[q] = round4(t[q]);
            const int64_t row = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off);
            apply_update<D>(a, row, li, g32);
        }
        __syncthreads();
    }
}

#define PICASSO_DISPATCH_D(D, CALL)                       \
    switch (D) {                                          \
        case 4: CALL(4); break;                           \
        case 8: CALL(8); break;                           \
        case 16: CALL(16); break;                         \
        case 32: CALL(32); break;                         \
        case 64: CALL(64); break;                         \
        case 128: CALL(128); break;                       \
        case 256: CALL(256); break;                       \
        case 384: CALL(384); break;                       \
        case 512: CALL(512); break;                       \
        default: break;                                   \
    }

void launch_segsum_update(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    const unsigned blocks = (unsigned)num_sms * 8;
#define CALL(DD) k_segsum_update<DD><<<blocks, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

void launch_long_update(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    const unsigned blocks = (unsigned)num_sms * 2;
#define CALL(DD) k_long_update<DD><<<blocks, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

}  // namespace picasso
