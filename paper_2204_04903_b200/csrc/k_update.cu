// k_update.cu — backward of the packed lookup fused with the sparse optimizer update.
//
// The backward is the mirror image of the forward: SegmentReduction^T
// scatters dY[b, col(f)] (mean: dY / len) to every occurrence, and Unique^T sums the
// occurrences of each unique row:  G_u = sum_{j: inverse[j] = u} dY[seg(j)] * s(j).
// The optimizer (north star; readings O9/O10) then updates each touched row once:
//   Adagrad   acc += G*G;  w -= lr * (G / (sqrt(acc) + eps))
//   lazy Adam m += (G-m)(1-b1); v += (G*G-v)(1-b2); w -= ss * (m / (sqrt(v) + eps))
// Each contribution is formed in fp32 (dY, dY/len), accumulated in fp64 and rounded once
// (reading O6): G = fp32(exact sum) whatever the summation order, so the chunked hot-row
// path and the oracle agree even when G nearly cancels.
//
//   k_csr_bounds     : row boundaries in the uid-sorted occurrence list (ustart)
//   k_segsum         : (narrow packs, D < 64) a warp walks the rows that start in its tile of
//                      occurrence positions and writes their rounded G (the fused / pipelined
//                      backward of D >= 64 lives in k_segsum_bulk.cu); rows with > kLongRow
//                      occurrences are deferred to the chunked path.
//   k_long_plan      : chunk counts (kChunk occurrences per chunk) of the deferred rows + scan
//   k_long_partial   : one row group per chunk -> fp64 partial sums (all chunks in parallel:
//                      a Zipf head with 1e5 occurrences is spread over the whole GPU)
//   k_long_finish    : per deferred row, partials summed in chunk order, rounded, updated
// All fp32 arithmetic uses explicit _rn intrinsics: no FMA contraction, IEEE sqrt/division.
#include <cub/block/block_scan.cuh>

#include <cstdlib>

#include "kernels.h"

namespace picasso {

constexpr int kChunk = 64;      // occurrences per hot-row chunk (latency per chunk vs partials to combine)
constexpr int kMaxChunks = 64;  // chunks per hot row at most (bounds the final combine)

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

// Where the G row of unique u goes: the hot-gradient buffer for a HybridHash hot row (and its
// occurrence count into hot_touch), else the rows/G buffer (send layout at W > 1, pack layout
// at W = 1).
template <int D>
__device__ __forceinline__ float *g_row_ptr(const UpdateArgs &a, int64_t u, int32_t u0, float *gp, int li,
                                            float nocc) {
    if (a.hslot) {
        const int32_t hs = a.hslot[u];
        if (hs >= 0) {
            if (li == 0) a.hot_touch[hs] = nocc;
            return a.hot_g + a.hot_g_off[a.pack] + (int64_t)(hs - a.hot_pslot[a.pack]) * D;
        }
    }
    if (a.dst_off) return a.dst_buf[a.dst_rank[u]] + a.dst_off[u];
    return a.row_off ? a.gbuf + a.row_off[u] : gp + (u - u0) * D;
}

// One dY contribution (fp32, mean: dY / len) of the occurrence in segment `seg`.
template <int D>
__device__ __forceinline__ void load_contrib(const UpdateArgs &a, int32_t seg, int li, float4 *c) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int32_t f = seg / a.B;
    const int32_t b = seg - f * a.B;
    const float *p = a.dy + (int64_t)b * a.dy_stride + dy_col(a, f) + li * 4;
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
__device__ __forceinline__ void update_row32(const UpdateArgs &a, int64_t row, int li, RowRegs<Geo<D>::VPL> &r,
                                             const float4 *g32) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    const int64_t o = row * D + li * 4;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
        const float4 g4 = g32[q];
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

template <int D>
__device__ __forceinline__ void update_row(const UpdateArgs &a, int64_t row, int li, RowRegs<Geo<D>::VPL> &r,
                                           const dbl4 *g64) {
    float4 g32[Geo<D>::VPL];
#pragma unroll
    for (int q = 0; q < Geo<D>::VPL; ++q) g32[q] = round4(g64[q]);
    update_row32<D>(a, row, li, r, g32);
}

// ------------------------------------------------------------------------------------------
// first row that starts at or after position p (p in [P0, P1); rows partition the positions)
__device__ __forceinline__ int32_t row_at_or_after(const int32_t *su, int32_t p, int32_t P0) {
    const int32_t u = __ldg(su + p);
    return (p == P0 || __ldg(su + p - 1) != u) ? u : u + 1;
}

// ------------------------------------------------------------------------------------------
// Split backward: k_segsum writes the rounded G of every
// unique row of the pack into a G buffer (rows in uid order: coalesced), k_update_rows then
// applies the optimizer row by row with two rows' weight/state loads in flight per group.
// Costs one extra G write + read (4·D bytes per unique row each way); used for the packs the fused
// k_segsum_upd (k_segsum_bulk.cu) does not take.
template <int D>
__global__ void __launch_bounds__(256) k_segsum(UpdateArgs a) {
    using Gm = Geo<D>;
    constexpr int LANES = Gm::LANES, VPL = Gm::VPL, R = Gm::R, SPG = Gm::SPG, U = Gm::U;
    constexpr int PPL = U > LANES ? U / LANES : 1, RND = LANES * PPL;
    __shared__ int32_t s_i0[8][32], s_cum[8][R][SPG + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int li = lane % LANES, grp = lane / LANES;
    const unsigned gmask = (LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << (grp * LANES));
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    if (u1 <= u0) return;
    float *gp = a.gbuf + a.pack_gbase[a.pack];
    const int32_t P0 = __ldg(a.ustart + u0), P1 = __ldg(a.ustart + u1);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t tile = ((int64_t)(P1 - P0) + nwarps - 1) / nwarps;
    tile = tile < 64 ? 64 : tile;
    for (int64_t pa = P0 + ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * tile; pa < P1; pa += nwarps * tile) {
        const int64_t pb = pa + tile < P1 ? pa + tile : P1;
        const int32_t ua = row_at_or_after(a.sorted_u, (int32_t)pa, P0);
        const int32_t ub = pb == P1 ? u1 : row_at_or_after(a.sorted_u, (int32_t)pb, P0);
#pragma unroll 1
        for (int32_t t0 = ua; t0 < ub; t0 += 32) {
            {
                const int32_t u = t0 + lane;
                int32_t i0 = 0, n = 0;
                if (u < ub) {
                    i0 = __ldg(a.ustart + u);
                    n = __ldg(a.ustart + u + 1) - i0;
                    if (n > kLongRow) {  // Zipf head: chunked path
                        a.long_list[atomicAdd(a.long_cnt, 1)] = u;
                        n = 0;
                    }
                }
                s_i0[w][lane] = i0;
                int32_t x = n;
#pragma unroll
                for (int o = 1; o < SPG; o <<= 1) {
                    const int32_t y = __shfl_up_sync(0xffffffffu, x, o, SPG);
                    if ((lane % SPG) >= o) x += y;
                }
                s_cum[w][lane / SPG][lane % SPG + 1] = x;
                if (lane % SPG == 0) s_cum[w][lane / SPG][0] = 0;
            }
            __syncwarp();
            const int nrow = (ub - t0) < 32 ? (ub - t0) : 32;
            const int c_lo = grp * SPG, c_hi = min(nrow, c_lo + SPG);
            const int32_t *cum = s_cum[w][grp];
            const int32_t total = c_hi > c_lo ? cum[c_hi - c_lo] : 0;
            dbl4 g[VPL];
#pragma unroll
            for (int q = 0; q < VPL; ++q) g[q] = zero4d();
            int cur = c_lo;
            auto finish = [&](int c) {  // rows deferred to the chunked path write nothing here
                const int32_t nocc = cum[c - c_lo + 1] - cum[c - c_lo];
                if (nocc > 0) {
                    float *o = g_row_ptr<D>(a, t0 + c, u0, gp, li, (float)nocc) + li * 4;
#pragma unroll
                    for (int q = 0; q < VPL; ++q) *reinterpret_cast<float4 *>(o + q * LANES * 4) = round4(g[q]);
                }
#pragma unroll
                for (int q = 0; q < VPL; ++q) g[q] = zero4d();
            };
#pragma unroll 1
            for (int32_t q0 = 0; q0 < total; q0 += RND) {
                int64_t myoff[PPL];
                int32_t myc[PPL], mylen[PPL];
#pragma unroll
                for (int p = 0; p < PPL; ++p) {
                    const int32_t q = q0 + p * LANES + li;
                    myc[p] = c_hi;
                    myoff[p] = 0;
                    mylen[p] = 0;
                    if (q < total) {
                        int lo = 0, hi = c_hi - c_lo;
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (cum[mid] <= q) lo = mid; else hi = mid;
                        }
                        const int32_t seg = __ldg(a.sorted_seg + s_i0[w][c_lo + lo] + (q - cum[lo]));
                        const int32_t f = seg / a.B;
                        myoff[p] = (int64_t)(seg - f * a.B) * a.dy_stride + dy_col(a, f);
                        if (a.pool_mean) mylen[p] = __ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg);
                        myc[p] = c_lo + lo;
                    }
                }
                const int32_t nround = min(RND, total - q0);
#pragma unroll 1
                for (int k0 = 0; k0 < nround; k0 += U) {
                    float4 c4[U][VPL];
                    int ck[U];
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        const int src = (k0 + k) % LANES, slot = PPL > 1 ? k / LANES : 0;
                        const int64_t off = __shfl_sync(gmask, myoff[slot], src, LANES);
                        const int32_t len = __shfl_sync(gmask, mylen[slot], src, LANES);
                        ck[k] = __shfl_sync(gmask, myc[slot], src, LANES);
                        if (k0 + k < nround) {
                            const float *p = a.dy + off + li * 4;
#pragma unroll
                            for (int qq = 0; qq < VPL; ++qq) c4[k][qq] = ldg_f4(p + qq * LANES * 4);
                            if (a.pool_mean) {
#pragma unroll
                                for (int qq = 0; qq < VPL; ++qq) c4[k][qq] = div4(c4[k][qq], (float)len);
                            }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        if (k0 + k < nround) {
                            while (cur < ck[k]) finish(cur++);
#pragma unroll
                            for (int qq = 0; qq < VPL; ++qq) g[qq] = add4d(g[qq], c4[k][qq]);
                        }
                    }
                }
            }
            while (cur < c_hi) finish(cur++);
            __syncwarp();
        }
    }
}

// Narrow rows (D <= 32: one float4 chunk per thread, D/4 threads per row): a thread group per
// unique row, rows dealt round robin over the whole grid, each thread walking the row's
// occurrences with two dY chunks in flight.  At these widths a pack's dY block (B x F_p x D)
// mostly stays in L2, so the warp-cooperative kernel above is bound by its per-occurrence
// instruction count, not by bytes; this one spends ~10 instructions per occurrence and chunk.
// It wins at D <= 8 only: wider rows (more threads per row walking the same dependent
// seg -> dY chain) lose to the warp kernel's broadcast addresses.
// Rows with > kLongRow occurrences go to the chunked path as above.
template <int D>
__global__ void __launch_bounds__(256) k_segsum_flat(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES;
    static_assert(Geo<D>::VPL == 1, "one float4 chunk per thread");
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    float *gp = a.gbuf + a.pack_gbase[a.pack];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int li = (int)(t % LANES);
    const int64_t ng = (int64_t)gridDim.x * blockDim.x / LANES;
#pragma unroll 1
    for (int64_t u = u0 + t / LANES; u < u1; u += ng) {
        const int32_t i0 = __ldg(a.ustart + u), i1 = __ldg(a.ustart + u + 1);
        if (i1 - i0 > kLongRow) {
            if (li == 0) a.long_list[atomicAdd(a.long_cnt, 1)] = (int32_t)u;
            continue;
        }
        dbl4 g = zero4d();
        int32_t i = i0;
#pragma unroll 1
        for (; i + 2 <= i1; i += 2) {
            const int32_t s0 = __ldg(a.sorted_seg + i), s1 = __ldg(a.sorted_seg + i + 1);
            float4 c0, c1;
            load_contrib<D>(a, s0, li, &c0);
            load_contrib<D>(a, s1, li, &c1);
            g = add4d(add4d(g, c0), c1);
        }
        if (i < i1) {
            float4 c0;
            load_contrib<D>(a, __ldg(a.sorted_seg + i), li, &c0);
            g = add4d(g, c0);
        }
        float *o = g_row_ptr<D>(a, u, u0, gp, li, (float)(i1 - i0)) + li * 4;
        *reinterpret_cast<float4 *>(o) = round4(g);
    }
}

__global__ void __launch_bounds__(256) k_dy_pack(const float4 *dy, int32_t B, int64_t ow4, const int32_t *col4_field,
                                                 const FieldInfo *finfo, const int64_t *dst_base,
                                                 const int32_t *fstride, float *dyp) {
    const int64_t n = (int64_t)B * ow4;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = q / ow4, c4 = q - b * ow4;
        const int32_t f = __ldg(col4_field + c4);
        if (f < 0) continue;  // a column no field owns
        const int64_t within = 4 * c4 - finfo[f].col;
        const float4 v = __ldcs(dy + q);  // read once
        *reinterpret_cast<float4 *>(dyp + __ldg(dst_base + f) + b * __ldg(fstride + f) + within) = v;
    }
}

void launch_dy_pack(const float *dy, int32_t B, int64_t out_width, const int32_t *col4_field, const FieldInfo *finfo,
                    const int64_t *dst_base, const int32_t *fstride, float *dyp, cudaStream_t s) {
    if (B <= 0 || out_width <= 0) return;
    k_dy_pack<<<2048, 256, 0, s>>>(reinterpret_cast<const float4 *>(dy), B, out_width / 4, col4_field, finfo, dst_base,
                                   fstride, dyp);
}

template <int D>
__global__ void __launch_bounds__(256) k_update_rows(UpdateArgs a) {
    constexpr int LANES = Geo<D>::LANES, VPL = Geo<D>::VPL;
    constexpr int RB = 2;  // rows per group iteration (their loads are issued together)
    const int li = threadIdx.x % LANES;
    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    const float *gp = a.gbuf + a.pack_gbase[a.pack];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
#pragma unroll 1
    for (int64_t ub = u0 + grp * RB; ub < u1; ub += ngrp * RB) {
        RowRegs<VPL> rr[RB];
        float4 g32[RB][VPL];
        int64_t row[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const int64_t u = ub + r;
            row[r] = -1;
            if (u < u1) {
                row[r] = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off);
                const float *gr = gp + (u - u0) * D + li * 4;
#pragma unroll
                for (int q = 0; q < VPL; ++q) g32[r][q] = ldg_f4(gr + q * LANES * 4);
                load_row<D>(a, row[r], li, rr[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (row[r] >= 0) update_row32<D>(a, row[r], li, rr[r], g32[r]);
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
            n = min((__ldg(a.ustart + u + 1) - __ldg(a.ustart + u) + kChunk - 1) / kChunk, kMaxChunks);
        }
        int32_t ex, agg;
        BlockScan(tmp).ExclusiveSum(n, ex, agg);
        if (e < K) {
            a.chunk_off[e] = carry + ex;
            for (int32_t i = 0; i < n; ++i) a.chunk_row[carry + ex + i] = e;  // chunk -> row
        }
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
    constexpr int PPL = U > LANES ? U / LANES : 1, RND = LANES * PPL;
    const int grp_in_warp = (threadIdx.x & 31) / LANES;
    const unsigned gmask = (LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << (grp_in_warp * LANES));
    const int32_t total = a.chunk_off[K];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
#pragma unroll 1
    for (int64_t c = grp; c < total; c += ngrp) {
        const int32_t e = a.chunk_row[c];
        const int32_t u = a.long_list[e];
        const int32_t ci = (int32_t)(c - a.chunk_off[e]);
        // a row of len occurrences is cut into nc = min(ceil(len/kChunk), kMaxChunks) equal chunks
        const int32_t r0 = __ldg(a.ustart + u), len = __ldg(a.ustart + u + 1) - r0;
        const int32_t nc = a.chunk_off[e + 1] - a.chunk_off[e], clen = (len + nc - 1) / nc;
        const int32_t p0 = r0 + ci * clen;
        const int32_t n = min(clen, r0 + len - p0);
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
#pragma unroll 1
        for (int32_t q0 = 0; q0 < n; q0 += RND) {
            // each lane resolves PPL occurrences; addresses broadcast, U dY rows in flight
            int64_t myoff[PPL];
            int32_t mylen[PPL];
#pragma unroll
            for (int p = 0; p < PPL; ++p) {
                const int32_t q = q0 + p * LANES + li;
                myoff[p] = 0;
                mylen[p] = 0;
                if (q < n) {
                    const int32_t seg = __ldg(a.sorted_seg + p0 + q);
                    const int32_t f = seg / a.B;
                    myoff[p] = (int64_t)(seg - f * a.B) * a.dy_stride + dy_col(a, f);
                    if (a.pool_mean) mylen[p] = __ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg);
                }
            }
            const int32_t nround = min(RND, n - q0);
#pragma unroll 1
            for (int k0 = 0; k0 < nround; k0 += U) {
                float4 c4[U][VPL];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int src = (k0 + k) % LANES, slot = PPL > 1 ? k / LANES : 0;
                    const int64_t off = __shfl_sync(gmask, myoff[slot], src, LANES);
                    const int32_t len = __shfl_sync(gmask, mylen[slot], src, LANES);
                    if (k0 + k < nround) {
                        const float *p = a.dy + off + li * 4;
#pragma unroll
                        for (int qq = 0; qq < VPL; ++qq) c4[k][qq] = ldg_f4(p + qq * LANES * 4);
                        if (a.pool_mean) {
#pragma unroll
                            for (int qq = 0; qq < VPL; ++qq) c4[k][qq] = div4(c4[k][qq], (float)len);
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < U; ++k)
                    if (k0 + k < nround)
#pragma unroll
                        for (int qq = 0; qq < VPL; ++qq) g[qq] = add4d(g[qq], c4[k][qq]);
            }
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
        if (!a.gbuf) load_row<D>(a, row, li, rr);
        dbl4 g[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q] = zero4d();
        const int32_t c0 = a.chunk_off[e], c1 = a.chunk_off[e + 1];
#pragma unroll 1
        for (int32_t c = c0; c < c1; c += 16) {  // chunk order; 16 partial loads in flight
            dbl4 pv[16][VPL];
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (c + k < c1) {
                    const dbl4 *pp = a.partial + (int64_t)(c + k) * (D / 4) + li;
#pragma unroll
                    for (int q = 0; q < VPL; ++q) pv[k][q] = pp[q * LANES];
                }
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (c + k < c1)
#pragma unroll
                    for (int q = 0; q < VPL; ++q) g[q] = add4d(g[q], pv[k][q]);
        }
        if (a.gbuf) {  // split backward: the update kernel applies the optimizer
            const int32_t u0 = a.pack_ustart[a.pack];
            float *o = g_row_ptr<D>(a, u, u0, a.gbuf + a.pack_gbase[a.pack], li,
                                    (float)(__ldg(a.ustart + u + 1) - __ldg(a.ustart + u))) + li * 4;
#pragma unroll
            for (int q = 0; q < VPL; ++q) *reinterpret_cast<float4 *>(o + q * LANES * 4) = round4(g[q]);
        } else {
            update_row<D>(a, row, li, rr, g);
        }
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

void launch_segsum(int D, const UpdateArgs &a, int num_sms, cudaStream_t s, bool flat_small) {
    if (flat_small && D <= 8) {  // measured at C3: D = 8 0.96 -> 0.75 ms; D = 16 / 32 slower (0.99 -> 1.10, 1.18 -> 1.87)
        const unsigned blocks = (unsigned)num_sms * 8;
        switch (D) {
            case 4: k_segsum_flat<4><<<blocks, 256, 0, s>>>(a); return;
            case 8: k_segsum_flat<8><<<blocks, 256, 0, s>>>(a); return;
            case 16: k_segsum_flat<16><<<blocks, 256, 0, s>>>(a); return;
            case 32: k_segsum_flat<32><<<blocks, 256, 0, s>>>(a); return;
            default: break;
        }
    }
    const unsigned blocks = (unsigned)num_sms * 4;
#define CALL(DD) k_segsum<DD><<<blocks, 256, 0, s>>>(a)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

void launch_update_rows(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    const unsigned blocks = (unsigned)num_sms * 8;
#define CALL(DD) k_update_rows<DD><<<blocks, 256, 0, s>>>(a)
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
