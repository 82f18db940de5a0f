// k_segsum_bulk.cu — backward segment-sum (Unique^T) as a copy pipeline.
//
// After the transpose, the occurrences of the pack sit in uid order (sorted_u / sorted_seg) and
//   G_u = sum_{p in [ustart[u], ustart[u+1])} dY[seg(p)] * s(p)      (s = 1, or 1/len for mean)
// The work is a gather of one dY row per occurrence (random rows of the [B, sum D] gradient), a
// segmented reduction, and one G row written per unique row: HBM-bound.
//
//   k_csr_tiles    : row starts (ustart) and, per pack, nt tiles of equal cost, cost(p) =
//                    occurrences + rows before p (one dY row read per occurrence, one G row
//                    written per row), so head tiles (few long rows) and tail tiles (many
//                    one-occurrence rows) take the same time; tiles cut rows anywhere.
//   k_segsum_pipe  : one warp per tile.  Its lanes resolve 32 positions at a time (sorted_seg ->
//                    dY row address, one round ahead); per ring stage (~4 KB of rows) each lane
//                    issues the asynchronous 16-byte copies (LDGSTS) of its own slice of every
//                    row into a per-warp shared-memory ring, so each SM keeps ~190 KB of dY
//                    in flight without register staging.  (1-D bulk copies through the TMA unit
//                    were measured first: no faster at 512-byte rows.)  Landed rows are reduced
//                    in fp64 (reading O6); each finished row's G is rounded and written.  A row
//                    cut by a tile edge leaves fp64 partials (head piece: slot 2t, tail piece:
//                    slot 2t+1) and the tile where it starts lists it.
//   k_segsum_fix   : per listed row, its pieces summed in tile order, rounded, written.
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace picasso {
namespace {

__device__ __forceinline__ void ldgsts(void *smem, const void *gmem) {  // 16 bytes, bypassing L1
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void ldgsts_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ldgsts_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kStageBytes = 4096;  // target bytes per ring stage
constexpr int kMaxNW = 24;         // warps per CTA at most (sizes the tile arrays)
#ifndef PICASSO_CONSUME_ROWS
#define PICASSO_CONSUME_ROWS 4
#endif
constexpr int kConsumeRows = PICASSO_CONSUME_ROWS;  // rows per unrolled consume step

template <int D, int NW, int S>
struct BG {
    static constexpr int ROWB = D * 4;
    static constexpr int RS = ROWB >= kStageBytes ? 1 : kStageBytes / ROWB;  // rows per stage (divides 32)
    static constexpr int SB = RS * ROWB;
    static constexpr int EPL = D / 32;                                      // floats per lane
    static constexpr int META = NW * S * 16 * RS;                           // uid + len + row per staged row
    static constexpr int RING_OFF = (META + 127) / 128 * 128;
    static constexpr int SMEM = RING_OFF + NW * S * SB;
    static_assert(32 % RS == 0, "a stage must lie inside one 32-position round");
    static_assert(EPL == 2 || EPL % 4 == 0, "lane layout: float2 or float4 chunks");
    static_assert(NW <= kMaxNW, "tile arrays are sized for kMaxNW warps per SM");
};

// Where the rounded G row of unique u goes (hot-gradient buffer, send layout, or pack layout).
template <int D>
__device__ __forceinline__ float *g_dst(const UpdateArgs &a, int32_t u, int32_t u0, float *gp, int lane,
                                        float nocc) {
    if (a.hslot) {
        const int32_t hs = a.hslot[u];
        if (hs >= 0) {
            if (lane == 0) a.hot_touch[hs] = nocc;
            return a.hot_g + a.hot_g_off[a.pack] + (int64_t)(hs - a.hot_pslot[a.pack]) * D;
        }
    }
    if (a.dst_off) return a.dst_buf[a.dst_rank[u]] + a.dst_off[u];
    return a.row_off ? a.gbuf + a.row_off[u] : gp + (int64_t)(u - u0) * D;
}

// A lane's elements of a row: D = 64 -> floats [2*lane, 2*lane+2); D >= 128 -> float4 chunks q
// at floats 128*q + 4*lane (consecutive lanes, consecutive 16 bytes: conflict-free).
template <int D>
__device__ __forceinline__ void lane_load(const float *row, int lane, float *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        const float2 x = reinterpret_cast<const float2 *>(row)[lane];
        v[0] = x.x;
        v[1] = x.y;
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q) {
            const float4 x = reinterpret_cast<const float4 *>(row)[q * 32 + lane];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    }
}
template <int D>
__device__ __forceinline__ void lane_store_f32(float *row, int lane, const double *acc) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        reinterpret_cast<float2 *>(row)[lane] = make_float2(__double2float_rn(acc[0]), __double2float_rn(acc[1]));
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q)
            reinterpret_cast<float4 *>(row)[q * 32 + lane] =
                make_float4(__double2float_rn(acc[4 * q]), __double2float_rn(acc[4 * q + 1]),
                            __double2float_rn(acc[4 * q + 2]), __double2float_rn(acc[4 * q + 3]));
    }
}
template <int D>
__device__ __forceinline__ void lane_store_f64(double *row, int lane, const double *acc) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        reinterpret_cast<double2 *>(row)[lane] = make_double2(acc[0], acc[1]);
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q) {
            double2 *o = reinterpret_cast<double2 *>(row + q * 128 + lane * 4);
            o[0] = make_double2(acc[4 * q], acc[4 * q + 1]);
            o[1] = make_double2(acc[4 * q + 2], acc[4 * q + 3]);
        }
    }
}
template <int D>
__device__ __forceinline__ void lane_load_f64(const double *row, int lane, double *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        const double2 x = reinterpret_cast<const double2 *>(row)[lane];
        v[0] = x.x;
        v[1] = x.y;
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q) {
            const double2 *o = reinterpret_cast<const double2 *>(row + q * 128 + lane * 4);
            const double2 x = o[0], y = o[1];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = y.x;
            v[4 * q + 3] = y.y;
        }
    }
}

// lane's elements of a row in global memory (same layout as lane_load)
template <int D>
__device__ __forceinline__ void lane_gload(const float *row, int lane, float *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        const float2 x = reinterpret_cast<const float2 *>(row)[lane];
        v[0] = x.x;
        v[1] = x.y;
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q) {
            const float4 x = reinterpret_cast<const float4 *>(row)[q * 32 + lane];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    }
}
template <int D>
__device__ __forceinline__ void lane_gstore(float *row, int lane, const float *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        reinterpret_cast<float2 *>(row)[lane] = make_float2(v[0], v[1]);
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q)
            reinterpret_cast<float4 *>(row)[q * 32 + lane] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
}

// Adagrad / lazy Adam on one element (north star; reading O10), IEEE round-to-nearest throughout
__device__ __forceinline__ void opt_step(const UpdateArgs &a, float g, float &w, float &s1, float &s2) {
    if (a.opt == 0) {
        s1 = __fadd_rn(s1, __fmul_rn(g, g));
        w = __fsub_rn(w, __fmul_rn(a.lr, __fdiv_rn(g, __fadd_rn(__fsqrt_rn(s1), a.eps))));
    } else {
        const float mo = s1, vo = s2;
        const float mu = __fmul_rn(__fsub_rn(g, mo), __fsub_rn(1.0f, a.beta1));
        const float vu = __fmul_rn(__fsub_rn(__fmul_rn(g, g), vo), __fsub_rn(1.0f, a.beta2));
        s1 = __fadd_rn(mu, mo);
        s2 = __fadd_rn(vu, vo);
        w = __fsub_rn(w, __fmul_rn(a.adam_ss, __fdiv_rn(s1, __fadd_rn(__fsqrt_rn(s2), a.eps))));
    }
}

// ------------------------------------------------------------------------------------------
// Row starts + equal-cost tiles.  Pack p holds sorted positions [G0, G1) = [pack_gstart[p],
// pack_gstart[p+1]) (uids are pack-major) and rows [U0, U1).  cost(i) = (i - G0) + (su[i] - U0)
// rises by 1 inside a row and by 2 at a row start; with C = (G1 - G0) + (U1 - U0) and
// nte = min(nt, C), position i belongs to tile floor(cost(i) * nte / C): tiles never come out
// empty inside a row, and tiles >= nte are empty at the pack's end.
__global__ void k_csr_tiles(const int32_t *su, int64_t N, int32_t *ustart, const int32_t *pack_gstart,
                            const int32_t *pack_ustart, int32_t P, int32_t nt, int32_t *tile_start, int32_t rw) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int32_t u = su[i];
    const bool row_start = i == 0 || su[i - 1] != u;
    if (row_start) ustart[u] = (int32_t)i;
    if (i == N - 1) ustart[u + 1] = (int32_t)N;
    int lo = 0, hi = P;  // pack: the last p with pack_ustart[p] <= u
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(pack_ustart + mid) <= u) lo = mid; else hi = mid;
    }
    const int64_t G0 = __ldg(pack_gstart + lo), G1 = __ldg(pack_gstart + lo + 1);
    const int64_t U0 = __ldg(pack_ustart + lo), U1 = __ldg(pack_ustart + lo + 1);
    // rw: cost of a row relative to an occurrence (1: G row write vs dY row read; the fused kernel
    // also reads and writes the row's weight and state, rw = 4)
    const int64_t C = (G1 - G0) + rw * (U1 - U0);
    const int64_t nte = nt < C ? nt : C;
    const int64_t cost = (i - G0) + rw * (u - U0);
    // floor(c * nte / C) without a 64-bit division: 32-bit when it fits, else a double
    // estimate corrected exactly
    auto tile_of = [&](int64_t c) -> int64_t {
        const int64_t x = c * nte;
        if (x <= 0xffffffffll && C <= 0xffffffffll) return (int64_t)((uint32_t)x / (uint32_t)C);
        int64_t k = (int64_t)((double)x / (double)C);
        while (k > 0 && k * C > x) --k;
        while ((k + 1) * C <= x) ++k;
        return k;
    };
    const int64_t k = tile_of(cost);
    int64_t kprev = -1;
    if (i > G0) kprev = tile_of(cost - (row_start ? 1 + rw : 1));
    int32_t *ts = tile_start + (int64_t)lo * (nt + 1);
    for (int64_t kk = kprev + 1; kk <= k; ++kk) ts[kk] = (int32_t)i;
    if (i == G1 - 1)
        for (int64_t kk = k + 1; kk <= nt; ++kk) ts[kk] = (int32_t)G1;
}

template <int D, int NW, int S>
__global__ void __launch_bounds__(NW * 32, 1) k_segsum_pipe(UpdateArgs a) {
    using G = BG<D, NW, S>;
    constexpr int RS = G::RS, SB = G::SB, ROWB = G::ROWB, EPL = G::EPL;
    constexpr int CH = RS < kConsumeRows ? RS : kConsumeRows;
    extern __shared__ __align__(128) unsigned char smem[];
    int32_t *s_uid = reinterpret_cast<int32_t *>(smem + (size_t)NW * S * RS * 8);  // (after an unused 8-B slot per row)
    int32_t *s_len = s_uid + NW * S * RS;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    if (u1 <= u0) return;
    const int32_t *ts = a.tile_start + (int64_t)a.pack * (a.nt + 1);
    const int32_t t = blockIdx.x * NW + w;
    if (t >= a.nt) return;
    const int32_t pa = __ldg(ts + t), pb = __ldg(ts + t + 1);
    if (pa >= pb) return;

    int32_t *wu = s_uid + w * S * RS, *wl = s_len + w * S * RS;
    unsigned char *wr = smem + G::RING_OFF + (size_t)w * S * SB;
    float *gp = a.gbuf + a.pack_gbase[a.pack];
    const float4 *dy4 = reinterpret_cast<const float4 *>(a.dy);

    // rows cut by the tile edges leave fp64 partials instead of G
    const int32_t u_first = __ldg(a.sorted_u + pa), u_last = __ldg(a.sorted_u + pb - 1);
    const int32_t last_end = __ldg(a.ustart + u_last + 1);
    const int32_t hp = __ldg(a.ustart + u_first) < pa ? u_first : -1;  // piece -> slot 2t
    const int32_t tp = (last_end > pb && u_last != hp) ? u_last : -1;   // piece -> slot 2t+1
    if (lane == 0 && tp >= 0)                                            // the split row starts here
        a.split[atomicAdd(a.long_cnt, 1)] = make_int4(t, tp, __ldg(a.ustart + tp), last_end);
    const int32_t nst = (pb - pa + RS - 1) / RS;

    // lane l holds position base + l of a 32-position round: dY row (float4 units), uid, bag length
    uint32_t off_c, off_n;
    int32_t uid_c, uid_n, len_c, len_n;
    auto resolve = [&](int32_t base, uint32_t &off, int32_t &uid, int32_t &len) {
        const int32_t p = base + lane;
        off = 0;
        uid = -1;
        len = 1;
        if (p < pb) {
            const int32_t seg = __ldg(a.sorted_seg + p);
            uid = __ldg(a.sorted_u + p);
            const int32_t f = seg / a.B;
            off = (uint32_t)(((int64_t)(seg - f * a.B) * a.dy_stride + dy_col(a, f)) >> 2);
            if (a.pool_mean) len = __ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg);
        }
    };
    resolve(pa, off_c, uid_c, len_c);
    resolve(pa + 32, off_n, uid_n, len_n);
    int32_t round_c = 0;
    auto issue = [&](int32_t k) {  // stage k -> ring slot k % S
        const int slot = k % S;
        const int32_t r = (k * RS) >> 5;
        if (r != round_c) {  // stages are issued in order: r == round_c + 1
            off_c = off_n;
            uid_c = uid_n;
            len_c = len_n;
            round_c = r;
            resolve(pa + (r + 1) * 32, off_n, uid_n, len_n);
        }
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const int l0 = (k * RS) & 31;
        unsigned char *dst = wr + slot * SB;
        if constexpr (EPL == 2) {  // D = 64: two rows per instruction, a half-warp of 16-B copies each
            const int h = lane >> 4, c = lane & 15;
#pragma unroll
            for (int i = 0; i < RS; i += 2) {
                const uint32_t off = __shfl_sync(0xffffffffu, off_c, l0 + i + h);
                if (i + h < nrows) ldgsts(dst + (i + h) * ROWB + c * 16, dy4 + off + c);
            }
        } else {
#pragma unroll
            for (int i = 0; i < RS; ++i) {
                const uint32_t off = __shfl_sync(0xffffffffu, off_c, l0 + i);
                if (i < nrows) {
                    const float4 *src = dy4 + off;
#pragma unroll
                    for (int q = 0; q < EPL / 4; ++q)
                        ldgsts(dst + i * ROWB + q * 512 + lane * 16, src + q * 32 + lane);
                }
            }
        }
        const int i = lane - l0;
        if (i >= 0 && i < nrows) {
            wu[slot * RS + i] = uid_c;
            wl[slot * RS + i] = len_c;
        }
    };

    double acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
    int32_t cur = -1, ncur = 0;  // current row, its occurrences in this tile (= all of them if unsplit)
    auto flush = [&](int32_t u) {
        double *part = reinterpret_cast<double *>(a.partial);
        if (u == hp) {
            lane_store_f64<D>(part + (int64_t)(2 * t) * D, lane, acc);
        } else if (u == tp) {
            lane_store_f64<D>(part + (int64_t)(2 * t + 1) * D, lane, acc);
        } else {
            lane_store_f32<D>(g_dst<D>(a, u, u0, gp, lane, (float)ncur), lane, acc);
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
    };

    // one commit group per stage (empty past the end), so stage k is complete at wait_group(S - 1)
    for (int32_t k = 0; k < S; ++k) {
        if (k < nst) issue(k);
        ldgsts_commit();
    }
#pragma unroll 1
    for (int32_t k = 0; k < nst; ++k) {
        const int slot = k % S;
        ldgsts_wait<S - 1>();
        __syncwarp();  // uid / len of the stage were written by other lanes
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const float *rows = reinterpret_cast<const float *>(wr + slot * SB);
        // CH rows at a time: the flush is inlined once per row of the unrolled body, and a
        // fully unrolled stage (16 rows at D = 64) overflows the instruction cache
#pragma unroll 1
        for (int i0 = 0; i0 < nrows; i0 += CH) {
            float v[CH][EPL];
#pragma unroll
            for (int c = 0; c < CH; ++c)
                if (i0 + c < nrows) lane_load<D>(rows + (i0 + c) * D, lane, v[c]);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = i0 + c;
                if (i < nrows) {
                    const int32_t uid = wu[slot * RS + i];
                    if (uid != cur) {
                        if (cur >= 0) flush(cur);
                        cur = uid;
                        ncur = 0;
                    }
                    ++ncur;
                    if (a.pool_mean) {
                        const float len = (float)wl[slot * RS + i];
#pragma unroll
                        for (int e = 0; e < EPL; ++e) v[c][e] = __fdiv_rn(v[c][e], len);
                    }
#pragma unroll
                    for (int e = 0; e < EPL; ++e) acc[e] = __dadd_rn(acc[e], (double)v[c][e]);
                }
            }
        }
        __syncwarp();  // the slot's uid / len are rewritten by the next issue
        if (k + S < nst) issue(k + S);
        ldgsts_commit();
    }
    if (cur >= 0) flush(cur);
}

// ------------------------------------------------------------------------------------------
// Segment-sum fused with the optimizer (world == 1, D = 64 / 128).  The pipe above, plus a
// second cp.async stream per warp: when a stage is issued, the weight and optimizer-state rows of
// every row that starts in it are copied into a ring of row slots (slot = row sequence number in
// the tile mod RR), in the same commit group as the stage's dY rows.  A row's flush therefore finds
// its G in registers and its weight / state in shared memory: the optimizer runs there and the
// rows are stored straight back — no G round trip through HBM and no second pass over the rows.
// Rows cut by a tile edge keep the fp64-partial path; k_segsum_fix<D, true> updates them.
// Ring bound: when stage k + S is issued (after stage k is consumed) at most 1 + S*RS rows of the
// tile are unflushed, so RR = S*RS + 2 slots never overwrite a row still to be read.
template <int D, int RS, int S, int NST>
struct FG {
    static constexpr int ROWB = D * 4;
    static constexpr int SB = RS * ROWB;             // dY bytes per stage
    static constexpr int RR = S * RS + 2;            // row slots
    static constexpr int SLOTB = (1 + NST) * ROWB;   // weight + state rows of one slot
    static constexpr int WARPB = S * SB + RR * SLOTB;
    static constexpr int META = S * RS * 8;          // uid + len per staged row
    static constexpr int EPL = D / 32;
    static_assert(32 % RS == 0, "a stage lies inside one 32-position round");
};

template <int D, int NW, int RS, int S, int NST>
__global__ void __launch_bounds__(NW * 32, 1) k_segsum_upd(UpdateArgs a) {
    using G = FG<D, RS, S, NST>;
    constexpr int ROWB = G::ROWB, SB = G::SB, RR = G::RR, SLOTB = G::SLOTB, EPL = G::EPL;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *wu = reinterpret_cast<int32_t *>(smem) + w * (G::META / 4);
    int32_t *wl = wu + S * RS;
    unsigned char *wr = smem + NW * G::META + (size_t)w * G::WARPB;  // [S stages of dY | RR row slots]
    unsigned char *wslot = wr + S * SB;

    const int32_t u0 = a.pack_ustart[a.pack], u1 = a.pack_ustart[a.pack + 1];
    if (u1 <= u0) return;
    const int32_t *ts = a.tile_start + (int64_t)a.pack * (a.nt + 1);
    const int32_t t = blockIdx.x * NW + w;
    if (t >= a.nt) return;
    const int32_t pa = __ldg(ts + t), pb = __ldg(ts + t + 1);
    if (pa >= pb) return;
    const float4 *dy4 = reinterpret_cast<const float4 *>(a.dy);

    const int32_t u_first = __ldg(a.sorted_u + pa), u_last = __ldg(a.sorted_u + pb - 1);
    const int32_t last_end = __ldg(a.ustart + u_last + 1);
    const int32_t hp = __ldg(a.ustart + u_first) < pa ? u_first : -1;
    const int32_t tp = (last_end > pb && u_last != hp) ? u_last : -1;
    if (lane == 0 && tp >= 0) a.split[atomicAdd(a.long_cnt, 1)] = make_int4(t, tp, __ldg(a.ustart + tp), last_end);
    const int32_t nst = (pb - pa + RS - 1) / RS;

    uint32_t off_c, off_n;
    int32_t uid_c, uid_n, len_c, len_n;
    int64_t row_c = 0, row_n = 0;
    auto resolve = [&](int32_t base, uint32_t &off, int32_t &uid, int32_t &len, int64_t &row) {
        const int32_t p = base + lane;
        off = 0;
        uid = -1;
        len = 1;
        row = 0;
        if (p < pb) {
            const int32_t seg = __ldg(a.sorted_seg + p);
            uid = __ldg(a.sorted_u + p);
            const int32_t f = seg / a.B;
            off = (uint32_t)(((int64_t)(seg - f * a.B) * a.dy_stride + dy_col(a, f)) >> 2);
            if (a.pool_mean) len = __ldg(a.offsets + seg + 1) - __ldg(a.offsets + seg);
            row = (int64_t)(__ldg(a.unique_gkey + uid) - (unsigned long long)a.pack_key_off);
        }
    };
    resolve(pa, off_c, uid_c, len_c, row_c);
    resolve(pa + 32, off_n, uid_n, len_n, row_n);
    int32_t round_c = 0, prev_last = -1, rseq_issue = 0;
    auto issue = [&](int32_t k) {
        const int slot = k % S;
        const int32_t r = (k * RS) >> 5;
        if (r != round_c) {
            prev_last = __shfl_sync(0xffffffffu, uid_c, 31);
            off_c = off_n;
            uid_c = uid_n;
            len_c = len_n;
            row_c = row_n;
            round_c = r;
            resolve(pa + (r + 1) * 32, off_n, uid_n, len_n, row_n);
        }
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const int l0 = (k * RS) & 31;
        unsigned char *dst = wr + slot * SB;
        if constexpr (EPL == 2) {
            const int h = lane >> 4, c = lane & 15;
#pragma unroll
            for (int i = 0; i < RS; i += 2) {
                const uint32_t off = __shfl_sync(0xffffffffu, off_c, l0 + i + h);
                if (i + h < nrows) ldgsts(dst + (i + h) * ROWB + c * 16, dy4 + off + c);
            }
        } else {
#pragma unroll
            for (int i = 0; i < RS; ++i) {
                const uint32_t off = __shfl_sync(0xffffffffu, off_c, l0 + i);
                if (i < nrows) {
#pragma unroll
                    for (int q = 0; q < EPL / 4; ++q)
                        ldgsts(dst + i * ROWB + q * 512 + lane * 16, dy4 + off + q * 32 + lane);
                }
            }
        }
        const int i = lane - l0;
        if (i >= 0 && i < nrows) {
            wu[slot * RS + i] = uid_c;
            wl[slot * RS + i] = len_c;
        }
        // the weight / state rows of the rows starting in this stage
        const int32_t up = __shfl_up_sync(0xffffffffu, uid_c, 1);
        const bool start = i >= 0 && i < nrows && (p0 + i == pa || uid_c != (lane == 0 ? prev_last : up));
        unsigned m = __ballot_sync(0xffffffffu, start);
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int32_t uid = __shfl_sync(0xffffffffu, uid_c, b);
            const int64_t row = __shfl_sync(0xffffffffu, row_c, b);
            unsigned char *sl = wslot + (rseq_issue % RR) * SLOTB;
            ++rseq_issue;
            if (uid == hp || uid == tp) continue;  // split rows: partials, updated by k_segsum_fix
            const float4 *src[1 + NST];
            src[0] = reinterpret_cast<const float4 *>(a.weight + row * D);
            src[1] = reinterpret_cast<const float4 *>(a.state1 + row * D);
            if constexpr (NST == 2) src[2] = reinterpret_cast<const float4 *>(a.state2 + row * D);
            if constexpr (EPL == 2) {  // 256-B rows: lanes 0-15 and 16-31 copy two arrays per instruction
                const int h = lane >> 4, c = lane & 15;
#pragma unroll
                for (int arr = 0; arr < 1 + NST; arr += 2)
                    if (arr + h < 1 + NST) ldgsts(sl + (arr + h) * ROWB + c * 16, src[arr + h] + c);
            } else {
#pragma unroll
                for (int arr = 0; arr < 1 + NST; ++arr)
#pragma unroll
                    for (int q = 0; q < EPL / 4; ++q)
                        ldgsts(sl + arr * ROWB + q * 512 + lane * 16, src[arr] + q * 32 + lane);
            }
        }
    };

    double acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
    int32_t cur = -1, rseq_cons = 0;
    int64_t cur_row = 0;
    auto flush = [&](int32_t u) {
        double *part = reinterpret_cast<double *>(a.partial);
        const unsigned char *sl = wslot + (rseq_cons % RR) * SLOTB;
        ++rseq_cons;
        if (u == hp) {
            lane_store_f64<D>(part + (int64_t)(2 * t) * D, lane, acc);
        } else if (u == tp) {
            lane_store_f64<D>(part + (int64_t)(2 * t + 1) * D, lane, acc);
        } else {
            float wv[EPL], s1[EPL], s2[EPL];
            lane_load<D>(reinterpret_cast<const float *>(sl), lane, wv);
            lane_load<D>(reinterpret_cast<const float *>(sl + ROWB), lane, s1);
            if constexpr (NST == 2) lane_load<D>(reinterpret_cast<const float *>(sl + 2 * ROWB), lane, s2);
#pragma unroll
            for (int e = 0; e < EPL; ++e) opt_step(a, __double2float_rn(acc[e]), wv[e], s1[e], s2[e]);
            lane_gstore<D>(a.weight + cur_row * D, lane, wv);
            lane_gstore<D>(a.state1 + cur_row * D, lane, s1);
            if constexpr (NST == 2) lane_gstore<D>(a.state2 + cur_row * D, lane, s2);
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
    };

    for (int32_t k = 0; k < S; ++k) {
        if (k < nst) issue(k);
        ldgsts_commit();
    }
    constexpr int CH = RS < kConsumeRows ? RS : kConsumeRows;
#pragma unroll 1
    for (int32_t k = 0; k < nst; ++k) {
        const int slot = k % S;
        ldgsts_wait<S - 1>();
        __syncwarp();
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const float *rows = reinterpret_cast<const float *>(wr + slot * SB);
#pragma unroll 1
        for (int i0 = 0; i0 < nrows; i0 += CH) {
            float v[CH][EPL];
#pragma unroll
            for (int c = 0; c < CH; ++c)
                if (i0 + c < nrows) lane_load<D>(rows + (i0 + c) * D, lane, v[c]);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = i0 + c;
                if (i < nrows) {
                    const int32_t uid = wu[slot * RS + i];
                    if (uid != cur) {
                        if (cur >= 0) flush(cur);
                        cur = uid;
                        cur_row = (int64_t)(__ldg(a.unique_gkey + uid) - (unsigned long long)a.pack_key_off);
                    }
                    if (a.pool_mean) {
                        const float len = (float)wl[slot * RS + i];
#pragma unroll
                        for (int e = 0; e < EPL; ++e) v[c][e] = __fdiv_rn(v[c][e], len);
                    }
#pragma unroll
                    for (int e = 0; e < EPL; ++e) acc[e] = __dadd_rn(acc[e], (double)v[c][e]);
                }
            }
        }
        __syncwarp();
        if (k + S < nst) issue(k + S);
        ldgsts_commit();
    }
    if (cur >= 0) flush(cur);
}

// One CTA per listed split row: its pieces (j = 0: slot 2t+1 of its first tile t; j >= 1: slot
// 2(t+j)) summed in tile order — warp w takes j = w mod 4, the warps combined in order.
template <int D, bool FUSE>
__global__ void __launch_bounds__(128) k_segsum_fix(UpdateArgs a) {
    constexpr int EPL = D / 32, NWF = 4;
    __shared__ double s_acc[NWF][D];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if ((int32_t)blockIdx.x >= *a.long_cnt) return;
    const int4 e = a.split[blockIdx.x];
    const int32_t t = e.x, u = e.y, rs = e.z, re = e.w;
    const int32_t *ts = a.tile_start + (int64_t)a.pack * (a.nt + 1);
    // the last piece is in the last tile starting before re
    int32_t tl = t;
    for (int32_t base = t + 1; base <= a.nt; base += 32) {
        const int32_t k = base + lane;
        const bool inside = k <= a.nt && __ldg(ts + k) < re;
        const unsigned m = __ballot_sync(0xffffffffu, inside);
        tl = base - 1 + __popc(m);  // tile starts are non-decreasing: the set bits are a prefix
        if (m != 0xffffffffu) break;
    }
    const int32_t npieces = tl - t + 1;
    const double *part = reinterpret_cast<const double *>(a.partial);
    double acc[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k) acc[k] = 0.0;
#pragma unroll 1
    for (int32_t j0 = w; j0 < npieces; j0 += NWF * 4) {
        double v[4][EPL];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t j = j0 + NWF * k;
            if (j < npieces) lane_load_f64<D>(part + (int64_t)(j == 0 ? 2 * t + 1 : 2 * (t + j)) * D, lane, v[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (j0 + NWF * k < npieces)
#pragma unroll
                for (int q = 0; q < EPL; ++q) acc[q] = __dadd_rn(acc[q], v[k][q]);
    }
    lane_store_f64<D>(s_acc[w], lane, acc);
    __syncthreads();
    if (w == 0) {
        lane_load_f64<D>(s_acc[0], lane, acc);
        for (int k = 1; k < NWF; ++k) {
            double v[EPL];
            lane_load_f64<D>(s_acc[k], lane, v);
#pragma unroll
            for (int q = 0; q < EPL; ++q) acc[q] = __dadd_rn(acc[q], v[q]);
        }
        if constexpr (FUSE) {  // the split row's update
            const int64_t o = (int64_t)(a.unique_gkey[u] - (unsigned long long)a.pack_key_off) * D;
            float w4[EPL], s1[EPL], s2[EPL];
            lane_gload<D>(a.weight + o, lane, w4);
            lane_gload<D>(a.state1 + o, lane, s1);
            if (a.opt == 1) lane_gload<D>(a.state2 + o, lane, s2);
#pragma unroll
            for (int q = 0; q < EPL; ++q) opt_step(a, __double2float_rn(acc[q]), w4[q], s1[q], s2[q]);
            lane_gstore<D>(a.weight + o, lane, w4);
            lane_gstore<D>(a.state1 + o, lane, s1);
            if (a.opt == 1) lane_gstore<D>(a.state2 + o, lane, s2);
        } else {
            const int32_t u0 = a.pack_ustart[a.pack];
            float *gp = a.gbuf + a.pack_gbase[a.pack];
            lane_store_f32<D>(g_dst<D>(a, u, u0, gp, lane, (float)(re - rs)), lane, acc);
        }
    }
}

template <int D, int NW, int S>
void launch_pipe(const UpdateArgs &a, int num_sms, cudaStream_t s) {
    using G = BG<D, NW, S>;
    ensure_dyn_smem((const void *)k_segsum_pipe<D, NW, S>, G::SMEM);
    (void)num_sms;  // one warp per tile: the grid covers the ctx's nt tiles
    k_segsum_pipe<D, NW, S><<<(unsigned)((a.nt + NW - 1) / NW), NW * 32, G::SMEM, s>>>(a);
    k_segsum_fix<D, false><<<(unsigned)a.nt, 128, 0, s>>>(a);
}

template <int D>
void launch_cfg(int cfg, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    switch (cfg) {
        case 1: launch_pipe<D, 12, 4>(a, num_sms, s); break;
        case 2: launch_pipe<D, 8, 6>(a, num_sms, s); break;
        case 3: launch_pipe<D, 16, 2>(a, num_sms, s); break;
        default: launch_pipe<D, 16, 3>(a, num_sms, s); break;
    }
}

}  // namespace

// PICASSO_SEGSUM_CFG = 16x3 (default) | 12x4 | 8x6 | 16x2: warps per CTA x ring stages
int segsum_pipe_cfg() {
    const char *e = std::getenv("PICASSO_SEGSUM_CFG");
    if (!e) return 0;
    if (!std::strcmp(e, "12x4")) return 1;
    if (!std::strcmp(e, "8x6")) return 2;
    if (!std::strcmp(e, "16x2")) return 3;
    return 0;
}
int segsum_pipe_warps(int cfg) { return cfg == 1 ? 12 : cfg == 2 ? 8 : 16; }

bool segsum_bulk_supported(int D, const UpdateArgs &a) {
    const bool dim_ok = D == 64 || D == 128 || D == 256 || D == 384 || D == 512;
    return dim_ok && a.gbuf && a.tile_start && ((uintptr_t)a.dy & 15) == 0 && (a.dy_stride & 3) == 0;
}

int launch_segsum_bulk(int cfg, int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    switch (D) {
        case 64: launch_cfg<64>(cfg, a, num_sms, s); break;
        case 128: launch_cfg<128>(cfg, a, num_sms, s); break;
        case 256: launch_cfg<256>(cfg, a, num_sms, s); break;
        case 384: launch_cfg<384>(cfg, a, num_sms, s); break;
        case 512: launch_cfg<512>(cfg, a, num_sms, s); break;
        default: return 0;
    }
    return 2;
}

void launch_csr_tiles(const int32_t *sorted_u, int64_t N, int32_t *ustart, int32_t *long_cnt,
                      const int32_t *pack_gstart, const int32_t *pack_ustart, int32_t P, int32_t nt,
                      int32_t *tile_start, cudaStream_t s, int32_t row_weight) {
    cudaMemsetAsync(long_cnt, 0, sizeof(int32_t) * P, s);
    if (N > 0)
        k_csr_tiles<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(sorted_u, N, ustart, pack_gstart, pack_ustart, P,
                                                                nt, tile_start, row_weight);
}

// segment-sum fused with the optimizer (world == 1, D = 64 / 128); returns #launches (0: n/a)
template <int D, int NW, int RS, int S, int NST>
void launch_upd(const UpdateArgs &a, int num_sms, cudaStream_t s) {
    using G = FG<D, RS, S, NST>;
    const size_t smem = (size_t)NW * (G::META + G::WARPB);
    ensure_dyn_smem((const void *)k_segsum_upd<D, NW, RS, S, NST>, smem);
    (void)num_sms;
    k_segsum_upd<D, NW, RS, S, NST><<<(unsigned)((a.nt + NW - 1) / NW), NW * 32, smem, s>>>(a);
    k_segsum_fix<D, true><<<(unsigned)a.nt, 128, 0, s>>>(a);
}

// Warps per CTA (= tiles per SM) of the fused kernel.  Adagrad, D = 128: 2 rows x 3 stages x 20 warps
// won the C2 sweep of rows / stage x stages x warps (0.2390 ms / step; 4 x 2 x 14: 0.2508, 2 x 2 x 24:
// 0.2399, 2 x 4 x 16: 0.2460, 4 x 3 x 11: 0.2728, 8 x 2 x 8: 0.3008); Adam stages a
// third row per slot and fits 10 warps.
int segsum_upd_warps(int opt) { return opt == 1 ? 10 : 20; }

int launch_segsum_fused(int D, const UpdateArgs &a, int num_sms, cudaStream_t s) {
    if (!a.tile_start || a.row_off || a.hslot || a.dst_off || ((uintptr_t)a.dy & 15) || (a.dy_stride & 3)) return 0;
    if (a.nt != num_sms * segsum_upd_warps(a.opt)) return 0;  // tiles were cut for this kernel's warps
    const bool adam = a.opt == 1;
    switch (D) {
        case 64:  // (C3 sweep of rows / stage x stages at 20 warps, pack 3's backward: 4 x 2 3.78 ms,
                  //  4 x 3 3.98, 2 x 4 4.19, 8 x 1 4.32, 2 x 2 4.41, 2 x 6 4.39, 1 x 8 5.77)
            if (adam) launch_upd<64, 10, 8, 2, 2>(a, num_sms, s);
            else launch_upd<64, 20, 4, 2, 1>(a, num_sms, s);
            break;
        case 128:
            if (adam) launch_upd<128, 10, 4, 2, 2>(a, num_sms, s);
            else launch_upd<128, 20, 2, 3, 1>(a, num_sms, s);
            break;
        default: return 0;
    }
    return 2;
}

size_t segsum_bulk_partial_doubles(int maxD, int num_sms) { return (size_t)2 * num_sms * kMaxNW * maxD; }
size_t segsum_tile_ints(int P, int num_sms) { return (size_t)P * (num_sms * kMaxNW + 1); }
size_t segsum_split_entries(int num_sms) { return (size_t)num_sms * kMaxNW; }

}  // namespace picasso
