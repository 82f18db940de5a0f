// k_update.cu — backward of the packed lookup fused with the sparse optimizer update.
//
// The backward is the mirror image of the forward: SegmentReduction^T
// scatters dY[b, col(f)] (mean: dY / len) to every occurrence, and Unique^T sums the
// occurrences of each unique row:  G_u = sum_{j: inverse[j] = u} dY[seg(j)] * s(j).
// The optimizer (north star; readings O9/O10) then updates each touched row once:
//   Adagrad   acc += G*G;  w -= lr * (G / (sqrt(acc) + eps))
//   lazy Adam m += (G-m)(1-b1); v += (G*G-v)(1-b2); w -= ss * (m / (sqrt(v) + eps))
// Fusing the two keeps G in registers: per touched row the kernel reads its dY rows once and
// the weight/state rows once, and writes weight/state once (no G round trip through HBM).
// Each contribution is formed in fp32 (dY, dY/len), accumulated in fp64 and rounded once
// (reading O6): G = fp32(exact sum) whatever the summation order, so the chunked hot-row
// path and the oracle agree even when G nearly cancels.
//
//   k_csr_bounds     : row boundaries in the uid-sorted occurrence list (ustart)
//   k_segsum_update  : a warp owns 32 consecutive unique rows, split into LANES-wide row
//                      groups; each group walks the flattened occurrence stream of its rows
//                      with U dY-row loads in flight, prefetches the weight/state row of the
//                      row it is summing, and updates it when the row's occurrences end.
//                      Rows with > kLongRow occurrences are deferred to the chunked path.
//   k_long_plan      : chunk counts (kChunk occurrences per chunk) of the deferred rows + scan
//   k_long_partial   : one row group per chunk -> fp64 partial sums (all chunks in parallel:
//                      a Zipf head with 1e5 occurrences is spread over the whole GPU)
//   k_long_finish    : per deferred row, partials summed in chunk order, rounded, updated
// All fp32 arithmetic uses explicit _rn intrinsics: no FMA contraction, IEEE sqrt/division.
#include <cub/block/block_scan.cuh>

#include "kernels.h"

namespace picasso {

constexpr int kChunk = 128;

__global__ void k_csr_bounds(const int32_t *su, int64_t N, int32_t *ustart) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int32_t u = su[i];
    if (i == 0 || su[i - 1] != u) ustart[u] = (int32_t)i;
    if (i == N - 1) ustart[u + 1] = (int32_t)N;
}

void launch_csr_bounds(const int32_t *sorted_u, int64_t N, int32_t *ustart, int32_t *long_cnt, int32_t n_cnt,
                       cudaStream_t s) {
    cudaMemsetAsync(long_cnt, 0, sizeof(int32_t) * n_cnt, s);
    if (N > 0) k_csr_bounds<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(sorted_u, N, ustart);
}

template <int D>
struct Geo {
    static constexpr int V4 = D / 4;
    static constexpr int LANES = V4 < 32 ? V4 : 32;
    static constexpr int VPL = V4 / LANES;
    static constexpr int R = 32 / LANES;
    static constexpr int SPG = 32 / R;
    static constexpr int U = D >= 64 ? 8 : 4;
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

// One dY contribution (fp32, mean: dY / len) of the occurrence in segment `seg`.
template <int D>
__device__ __forceinline__ void load_contrib(const UpdateArgs &a, int32_t seg, int li, float4 *c) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int32_t f = seg / a.B;
    const int32_t b = seg - f * a.B;
    const float *p = a.dy + (int64_t)b * a.dy_stride + a.finfo[f].col + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) c[q] = ldg_f4(p + q * LANES * 4);
    if (a.pool_mean) {
        const float len = (float)(__ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg));
#pragma unroll
        for (int q = 0; q < VPL; ++q) c[q] = div4(c[q], len);
    }
}

// Weight / state row registers of one update.
template <int VPL>
struct RowRegs {
    float4 w[VPL], s1[VPL], s2[VPL];
};

template <int D>
__device__ __forceinline__ void load_row(const UpdateArgs &a, int64_t row, int li, RowRegs<Geo<D>::VPL> &r) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int64_t o = row * D + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        r.w[q] = *reinterpret_cast<const float4 *>(a.weight + o + q * LANES * 4);
        r.s1[q] = *reinterpret_cast<const float4 *>(a.state1 + o + q * LANES * 4);
        if (a.opt == 1) r.s2[q] = *reinterpret_cast<const float4 *>(a.state2 + o + q * LANES * 4);
    }
}

template <int D>
__device__ __forceinline__ void update_row(const UpdateArgs &a, int64_t row, int li, RowRegs<Geo<D>::VPL> &r,
                                           const dbl4 *g64) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int64_t o = row * D + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        const float4 g4 = round4(g64[q]);
        const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
        float ww[4] = {r.w[q].x, r.w[q].y, r.w[q].z, r.w[q].w};
        float ss[4] = {r.s1[q].x, r.s1[q].y, r.s1[q].z, r.s1[q].w};
        if (a.opt == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float acc = __fadd_rn(ss[e], __fmul_rn(gg[e], gg[e]));
                ss[e] = acc;
                const float qq = __fdiv_rn(gg[e], __fadd_rn(__fsqrt_rn(acc), a.eps));
                ww[e] = __fsub_rn(ww[e], __fmul_rn(a.lr, qq));
            }
        } else {
            float v2[4] = {r.s2[q].x, r.s2[q].y, r.s2[q].z, r.s2[q].w};
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
            *reinterpret_cast<float4 *>(a.state2 + o + q * LANES * 4) = make_float4(v2[0], v2[1], v2[2], v2[3]);
        }
        *reinterpret_cast<float4 *>(a.weight + o + q * LANES * 4) = make_float4(ww[0], ww[1], ww[2], ww[3]);
        *reinterpret_cast<float4 *>(a.state1 + o + q * LANES * 4) = make_float4(ss[0], ss[1], ss[2], ss[3]);
    }
}

// ------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_segsum_update(UpdateArgs a) {
    using Gm = Geo<D>;
    constexpr int LANES = Gm::LANES, VPL = Gm::VPL, SPG = Gm::SPG, U = Gm::U;
    __shared__ int32_t s_i0[8][32], s_i1[8][32];
    __shared__ int64_t s_row[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int li = lane % LANES, grp = lane / LANES;
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    const int64_t nU = (int64_t)u1 - u0;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; t0 < nU; t0 += nwarps * 32) {
        {
            const int64_t u = u0 + t0 + lane;
            int32_t i0 = 0, i1 = 0;
            int64_t row = -1;
            if (u < u1) {
                i0 = __ldg(a.ustart + u);
                i1 = __ldg(a.ustart + u + 1);
                if (i1 - i0 > kLongRow) {  // Zipf head: chunked path
                    a.long_list[atomicAdd(a.long_cnt, 1)] = (int32_t)u;
                    i1 = i0;
                } else {
                    row = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off);
                }
            }
            s_i0[wib][lane] = i0;
            s_i1[wib][lane] = i1;
            s_row[wib][lane] = row;
        }
        __syncwarp();
        const int nrow = (int)((nU - t0) < 32 ? (nU - t0) : 32);
        const int c_lo = grp * SPG, c_hi = min(nrow, c_lo + SPG);
        int cur = c_lo;
        int32_t i = cur < c_hi ? s_i0[wib][cur] : 0, e = cur < c_hi ? s_i1[wib][cur] : 0;
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        RowRegs<VPL> rr;
        if (cur < c_hi && s_row[wib][cur] >= 0) load_row<D>(a, s_row[wib][cur], li, rr);
        while (cur < c_hi) {
            int bcur[U];
            int32_t bpos[U];
            int n = 0;
            {
                int c2 = cur;
                int32_t i2 = i, e2 = e;
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    while (i2 >= e2 && c2 < c_hi) {
                        ++c2;
                        if (c2 < c_hi) {
                            i2 = s_i0[wib][c2];
                            e2 = s_i1[wib][c2];
                        }
                    }
                    bcur[k] = c2;
                    bpos[k] = i2;
                    if (c2 < c_hi) {
                        ++n;
                        ++i2;
                    }
                }
            }
            float4 c[U][VPL];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (k < n) load_contrib<D>(a, __ldg(a.sorted_seg + bpos[k]), li, c[k]);
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (k < n) {
                    while (cur < bcur[k]) {  // row `cur` complete: update, prefetch the next
                        if (s_row[wib][cur] >= 0) update_row<D>(a, s_row[wib][cur], li, rr, g);
#pragma unroll
                        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
                        ++cur;
                        if (s_row[wib][cur] >= 0) load_row<D>(a, s_row[wib][cur], li, rr);
                    }
#pragma unroll
                    for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], c[k][q]);
                }
            }
            if (n < U) {
                while (cur < c_hi) {
                    if (s_row[wib][cur] >= 0) update_row<D>(a, s_row[wib][cur], li, rr, g);
#pragma unroll
                    for (int q = 0; q < VPL; ++q) g[q] = zero4d();
                    ++cur;
                    if (cur < c_hi && s_row[wib][cur] >= 0) load_row<D>(a, s_row[wib][cur], li, rr);
                }
            } else {
                cur = bcur[U - 1];
                i = bpos[U - 1] + 1;
                e = s_i1[wib][cur];
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_long_plan(UpdateArgs a) {
    using BlockScan = cub::BlockScan<int32_t, 1024>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ int32_t carry;
    const int32_t K = *a.long_cnt;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int32_t base = 0; base < K; base += 1024) {
        const int32_t e = base + threadIdx.x;
        int32_t n = 0;
        if (e < K) {
            const int32_t u = a.long_list[e];
            n = (__ldg(a.ustart + u + 1) - __ldg(a.ustart + u) + kChunk - 1) / kChunk;
        }
        int32_t ex, agg;
        BlockScan(tmp).ExclusiveSum(n, ex, agg);
        if (e < K) a.chunk_off[e] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.chunk_off[K] = carry;
}

template <int D>
__global__ void __launch_bounds__(256) k_long_partial(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL, U = Geo<D>::U;
    const int li = threadIdx.x % LANES;
    const int32_t K = *a.long_cnt;
    if (K == 0) return;
    const int32_t total = a.chunk_off[K];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t c = grp; c < total; c += ngrp) {
        const int64_t e = upper_bound_dev(a.chunk_off, 0, K + 1, (int32_t)c) - 1;
        const int32_t u = a.long_list[e];
        const int32_t ci = (int32_t)(c - a.chunk_off[e]);
        const int32_t p0 = __ldg(a.ustart + u) + ci * kChunk;
        const int32_t p1 = min(p0 + kChunk, __ldg(a.ustart + u + 1));
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        for (int32_t p = p0; p < p1; p += U) {
            float4 cc[U][VPL];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (p + k < p1) load_contrib<D>(a, __ldg(a.sorted_seg + p + k), li, cc[k]);
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (p + k < p1)
#pragma unroll
                    for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], cc[k][q]);
        }
        dbl4 *out = a.partial + c * (D / 4) + li;
#pragma unroll
        for (int q = 0; q < VPL; ++q) out[q * LANES] = g[q];
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_long_finish(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int li = threadIdx.x % LANES;
    const int32_t K = *a.long_cnt;
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t e = grp; e < K; e += ngrp) {
        const int32_t u = a.long_list[e];
        const int64_t row = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off);
        RowRegs<VPL> rr;
        load_row<D>(a, row, li, rr);
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        for (int32_t c = a.chunk_off[e]; c < a.chunk_off[e + 1]; ++c) {  // chunk order
            const dbl4 *pp = a.partial + (int64_t)c * (D / 4) + li;
#pragma unroll
            for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], pp[q * LANES]);
        }
        update_row<D>(a, row, li, rr, g);
    }
}

#define PICASSO_DISPATCH_D(D, CALL) \
    switch (D) {                    \
        case 4: CALL(4); break;     \
        case 8: CALL(8); break;     \
        case 16: CALL(16); break;   \
        case 32: CALL(32); break;   \
        case 64: CALL(64); break;   \
        case 128: CALL(128); break; \
        case 256: CALL(256); break; \
        case 384: CALL(384); break; \
        case 512: CALL(512); break; \
        default: break;             \
    }

void launch_segsum_update(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    const unsigned blocks = (unsigned)num_sms * 8;
#define CALL(DD) k_segsum_update<DD><<<blocks, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

int launch_long_update(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    k_long_plan<<<1, 1024, 0, s>>>(a);
    const unsigned blocks = (unsigned)num_sms * 4;
#define CALL(DD) k_long_partial<DD><<<blocks, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
#define CALL(DD) k_long_finish<DD><<<(unsigned)num_sms, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
    return 3;
}

size_t long_partial_doubles(int64_t N, int maxD) {
    return (size_t)(N / kChunk + N / (kLongRow + 1) + 2) * (size_t)maxD;
}

}  // namespace picasso
