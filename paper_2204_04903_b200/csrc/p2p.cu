// p2p.cu — the row-sharded exchange over NVLink peer memory (world W > 1, one GPU per rank).
//
// Every rank exposes one IPC-shared window: barrier flags, its bucket counts, its send list
// (requested local rows, owner-major), and its rows/G buffer in the send layout.  The owner
// side then needs no staged all-to-all (SURVEY §8(f) "kernel-initiated Shuffle&Stitch"):
//   k_p2p_tables : owner block table and G-slot bases from every rank's bucket counts (device-
//                  side sizes: no host synchronisation, so a step can be captured in a CUDA graph)
//   k_p2p_dst_insert : requester side, each unique row's G slot at its owner; owner side, each
//                  requested key read straight from the requester's send list (NVLink loads)
//                  into a direct (row, source) table
//   k_p2p_gather : gathers the owner's rows and stores them straight into each requester's rows
//                  buffer at the slot its send layout reserved (NVLink stores): Gather + Shuffle
//                  + Stitch in one kernel, the transfer overlapping the gather row by row
//   (segment-sum) : stores each G row at its slot in the owner's memory (NVLink stores:
//                  segment-sum + gradient Shuffle in one kernel)
//   k_p2p_update : per owner position whose source is the row's lowest requesting source (each
//                  row once), the <= W pushed G rows summed in source-rank order (fp64,
//                  reading O6') and the optimizer applied
//   k_p2p_signal / k_p2p_wait : epoch flags in the peers' windows (system-scope release /
//                  acquire), with a timeout that latches an error instead of hanging
#include "kernels.h"
#include "multi.h"
#include "p2p.h"

namespace picasso {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------------------------------
__global__ void k_p2p_signal(P2PArgs a, int slot) {
    if (threadIdx.x != 0) return;
    const uint32_t e = ++a.epoch[slot];
    __threadfence_system();
    for (int q = 0; q < a.W; ++q) st_release_sys(a.peer.flags[q] + slot * kP2PMaxW + a.rank, e);
}

// The waiter counts its own waits per slot (epoch[kP2PFlags + slot]): its target never depends
// on whether this rank's own signal of the slot (possibly on another stream) has run yet.
__global__ void k_p2p_wait(P2PArgs a, int slot) {
    __shared__ uint32_t s_e;
    if (threadIdx.x == 0) s_e = ++a.epoch[kP2PFlags + slot];
    __syncthreads();
    const int q = threadIdx.x;
    if (q < a.W) {
        const uint32_t e = s_e;
        const uint32_t *f = a.peer.flags[a.rank] + slot * kP2PMaxW + q;
        const uint64_t t0 = globaltimer();
        while ((int32_t)(ld_acquire_sys(f) - e) < 0) {
            if (globaltimer() - t0 > kP2PTimeoutNs) {  // a peer never arrived: latch, do not hang
                atomicOr(a.err, ERR_PEER_TIMEOUT);
                break;
            }
            __nanosleep(200);
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Both sides' tables from every rank's bucket counts, staged once in shared memory (one NVLink
// round trip for the whole W x (W*P) count matrix).  One block of 1024 threads.
//  owner side, pack-major blocks (pack p, source s): ostart (owner-stream position), rstart =
//    index of the block's first key in s's send list, rroff = float offset of its first row in
//    s's rows buffer; pack starts, received count R, float layout of the received G rows;
//  requester side: dbase[(r, p)] = float offset of my requests' G block in owner r's receive
//    buffer (owner r holds pack p's requests pack-major, then by source rank).
__global__ void __launch_bounds__(1024) k_p2p_tables(P2PArgs a) {
    __shared__ int32_t cm[kP2PMaxW][kMaxOwnerBlocks];  // cm[s][b]: source s's count of bucket b
    __shared__ int32_t wsum[32];
    __shared__ int64_t s_total;
    const int t = threadIdx.x, nb = a.W * a.P;
    for (int e = t; e < a.W * nb; e += blockDim.x) cm[e / nb][e % nb] = __ldcv(a.peer.bcount[e / nb] + e % nb);
    __syncthreads();
    // requester side
    if (t < nb) {
        const int r = t / a.P, p = t - (t / a.P) * a.P;
        int64_t f = 0;
        for (int q = 0; q < p; ++q) {  // packs before p at owner r, all sources
            int64_t n = 0;
            for (int s = 0; s < a.W; ++s) n += cm[s][r * a.P + q];
            f += n * __ldg(a.pack_dim + q);
        }
        int64_t before = 0;  // sources before me, same pack
        for (int s = 0; s < a.rank; ++s) before += cm[s][t];
        a.dbase[t] = f + before * __ldg(a.pack_dim + p);
    }
    // owner side
    const int p = t / a.W, s = t - (t / a.W) * a.W;
    int32_t c = 0;
    int64_t ks = 0, gs = 0;
    if (t < nb) {
        const int me = a.rank * a.P + p;
        for (int b = 0; b < me; ++b) {  // s's buckets before (rank, p): owner-major, then pack
            ks += cm[s][b];
            gs += (int64_t)cm[s][b] * __ldg(a.pack_dim + (b % a.P));
        }
        c = cm[s][me];
        a.cnt_recv[s * a.P + p] = c;
    }
    const int lane = t & 31, w = t >> 5;  // block exclusive scan of c in t order
    int32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int32_t y = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        wsum[lane] = y;
        if (lane == 31) s_total = y;
    }
    __syncthreads();
    const int64_t total = s_total;
    const bool over = total > a.max_recv;  // capacity: latch, process nothing
    const int64_t ostart = over ? 0 : (int64_t)(w ? wsum[w - 1] : 0) + x - c;
    if (t < nb) {
        OwnerBlock b;
        b.ostart = ostart;
        b.rstart = ks;
        b.rroff = gs;
        b.pack = p;
        b.src = s;
        a.oblk[t] = b;
        if (s == 0) {
            a.pack_ostart[p] = ostart;
            a.opack_gstart[p] = (int32_t)ostart;
        }
    }
    if (t == 0) {
        a.pack_ostart[a.P] = over ? 0 : total;
        a.opack_gstart[a.P] = (int32_t)(over ? 0 : total);
        *a.R = (int32_t)(over ? 0 : total);
        if (over) atomicOr(a.err, ERR_CAPACITY);
    }
    __syncthreads();
    if (t < a.P) a.ocount[t] = 0;
    if (t == 0) {  // float layout of the received G rows: pack-major, D_p floats per position
        int64_t f = 0;
        for (int q = 0; q < a.P; ++q) {
            a.pack_fbase[q] = f;
            f += (a.pack_ostart[q + 1] - a.pack_ostart[q]) * __ldg(a.pack_dim + q);
        }
        a.pack_fbase[a.P] = f;
    }
}

__device__ __forceinline__ int owner_block_p(const OwnerBlock *blk, int nb, int64_t opos) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (blk[mid].ostart <= opos) lo = mid; else hi = mid;
    }
    return lo;
}

// One launch, two index ranges.  e < U (requester side): the owner receive-buffer slot of my
// unique row e's G (k_segsum_pipe stores it there).  e >= U (owner side, opos = e - U): the
// requested key read from the requester's send list (NVLink load); per owner position: local
// row, source, float offset of the requester's row slot; dtab[(row_base[p] + row) * W + src] =
// opos (each requester asks for a key at most once, so (row, src) is unique: a direct table
// replaces the owner hash).
__global__ void __launch_bounds__(256) k_p2p_dst_insert(P2PArgs a) {
    __shared__ OwnerBlock sb[kMaxOwnerBlocks];
    const int nb = a.W * a.P;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = a.oblk[i];
    __syncthreads();
    const int64_t U = *a.d_total, R = *a.R;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < U + R; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < U) {
            const int32_t b = a.bkey[e];  // bucket (owner, pack) from the Partition pass
            if (b >= nb) continue;        // hot: G goes to the replicated hot buffer
            a.dst_rank[e] = b / a.P;
            a.dst_off[e] = a.dbase[b] + (a.send_pos[e] - a.bstart[b]) * __ldg(a.pack_dim + (b % a.P));
            continue;
        }
        const int64_t opos = e - U;
        const int k = owner_block_p(sb, nb, opos);
        const int64_t j = opos - sb[k].ostart;
        const int p = sb[k].pack, src = sb[k].src;
        const int32_t lr = __ldcv(a.peer.send_keys[src] + sb[k].rstart + j);
        a.lrow[opos] = lr;
        a.osrc[opos] = src;
        a.roff[opos] = sb[k].rroff + j * __ldg(a.pack_dim + p);
        a.dtab[(a.row_base[p] + lr) * a.W + src] = (int32_t)opos;
        if (a.fcnt) atomicAdd(a.fcnt + a.fcnt_off[p] + lr, 1u);  // FCounter (Alg. 1)
    }
}

// W > 2: rows requested this step, listed once each (by the lowest requesting source), per pack:
// olist[pack_ostart[p] + i], i < ocount[p] (order irrelevant: each row's update is independent).
// With more sources per row the update then walks rows, not positions (at W = 2 the update's own
// leader test is cheaper than this pass: see k_p2p_update)
__global__ void k_p2p_leaders(P2PArgs a) {
    const int64_t R = *a.R;
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count; one atomic per (warp, pack) instead of one per row
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < R;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t opos = base + lane;
        int p = 0;
        int32_t row = 0;
        bool leader = false;
        if (opos < R) {
            while (p + 1 < a.P && a.pack_ostart[p + 1] <= opos) ++p;
            row = a.lrow[opos];
            const int32_t src = a.osrc[opos];
            const int32_t *dt = a.dtab + (a.row_base[p] + row) * a.W;
            int32_t op[kP2PMaxW];
#pragma unroll
            for (int s = 0; s < kP2PMaxW; ++s) op[s] = s < src ? __ldcg(dt + s) : -1;  // independent loads
            leader = true;
#pragma unroll
            for (int s = 0; s < kP2PMaxW; ++s) leader = leader & (op[s] < 0);
        }
        const unsigned lm = __ballot_sync(0xffffffffu, leader);
        if (leader) {
            const unsigned peers = __match_any_sync(lm, p);
            const int first = __ffs(peers) - 1;
            int32_t b = 0;
            if (lane == first) b = atomicAdd(a.ocount + p, __popc(peers));
            b = __shfl_sync(peers, b, first);
            a.olist[a.pack_ostart[p] + b + __popc(peers & ((1u << lane) - 1u))] = row;
        }
    }
}

// clears the previous step's direct-table entries (positions of the last forward)
__global__ void k_p2p_reset(P2PArgs a) {
    const int64_t R = *a.R;
    for (int64_t opos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; opos < R;
         opos += (int64_t)gridDim.x * blockDim.x) {
        int p = 0;
        while (p + 1 < a.P && a.pack_ostart[p + 1] <= opos) ++p;
        a.dtab[(a.row_base[p] + a.lrow[opos]) * a.W + a.osrc[opos]] = -1;
    }
}

// owner rows -> the requesters' rows buffers (peer stores).  One thread per 16-B chunk of a row
// (grid-stride): the most independent requests in flight per SM for this random-row pattern
// (tools/gather_bench.cu).
template <int D>
__global__ void __launch_bounds__(256) k_p2p_gather(P2PArgs a, const float *weight, int pack) {
    constexpr int V4 = D / 4;
    const int64_t o0 = a.pack_ostart[pack], o1 = a.pack_ostart[pack + 1];
    const int64_t n = (o1 - o0) * V4;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t opos = o0 + e / V4;
        const int c = (int)(e % V4);
        const float4 v = ldg_f4(weight + (int64_t)__ldg(a.lrow + opos) * D + c * 4);
        __stcg(reinterpret_cast<float4 *>(a.peer.gbuf[__ldg(a.osrc + opos)] + __ldg(a.roff + opos) + c * 4), v);
    }
}

// k_p2p_gather with one thread per 32-B chunk (D >= 16, D % 8 == 0, 32-B aligned rows and
// buffers): 256-bit loads of the owner's row, 256-bit peer stores
template <int D>
__global__ void __launch_bounds__(256) k_p2p_gather8(P2PArgs a, const float *weight, int pack) {
    constexpr int V8 = D / 8;
    const int64_t o0 = a.pack_ostart[pack], o1 = a.pack_ostart[pack + 1];
    const int64_t n = (o1 - o0) * V8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t opos = o0 + e / V8;
        const int c = (int)(e % V8);
        const f8 v = ldg_f8(weight + (int64_t)__ldg(a.lrow + opos) * D + c * 8);
        float *dst = a.peer.gbuf[__ldg(a.osrc + opos)] + __ldg(a.roff + opos) + c * 8;
        asm volatile("st.global.cg.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "f"(v.v[0]), "f"(v.v[1]),
                     "f"(v.v[2]), "f"(v.v[3]), "f"(v.v[4]), "f"(v.v[5]), "f"(v.v[6]), "f"(v.v[7])
                     : "memory");
    }
}

// Per owner position of the pack (one G row pushed by one source), the row's update is done by
// the position of its lowest requesting source ("leader"; the others return after reading the
// row's W table entries): the <= W pushed G rows (in this owner's receive buffer) summed in
// source-rank order in fp64 (reading O6'), rounded once, Adagrad / lazy Adam.  Walking the
// positions directly replaces a separate leader-listing pass (one random table read per
// position fewer, no row list).  One thread per 16-B chunk of a row; the <= NFW table entries
// and contributions of a chunk are loaded together.
template <int D, int NFW, bool LIST>
__global__ void __launch_bounds__(256) k_p2p_update(P2PArgs a, int pack, float *weight, float *state1,
                                                    float *state2, int opt, float lr, float eps, float beta1,
                                                    float beta2, float adam_ss) {
    constexpr int V4 = D / 4;
    // a barrier of this or an earlier step timed out (sticky until the context is destroyed): the
    // pushed G rows may be stale or partial, so the tables and optimizer state are left untouched
    if (__ldcg(a.err) & ERR_PEER_TIMEOUT) return;
    const int64_t o0 = a.pack_ostart[pack];
    const int64_t n = (LIST ? (int64_t)a.ocount[pack] : a.pack_ostart[pack + 1] - o0) * V4;
    const int64_t rb = a.row_base[pack];
    const float *gin = a.peer.ogbuf[a.rank] + a.pack_fbase[pack];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t opos = o0 + e / V4;
        const int32_t row = LIST ? __ldg(a.olist + opos) : __ldg(a.lrow + opos);
        const int32_t src = LIST ? 0 : __ldg(a.osrc + opos);  // (LIST: every listed row is updated)
        const int c = (int)(e % V4);
        const int32_t *dt = a.dtab + (rb + row) * a.W;
        int32_t op[NFW];
#pragma unroll
        for (int s = 0; s < NFW; ++s) op[s] = s < a.W ? __ldcg(dt + s) : -1;
        bool leader = true;
#pragma unroll
        for (int s = 0; s < NFW; ++s) leader = leader && !(s < src && op[s] >= 0);
        if (!leader) continue;
        const int64_t o = (int64_t)row * D + c * 4;
        float4 x[NFW];
#pragma unroll
        for (int s = 0; s < NFW; ++s)
            if (op[s] >= 0) x[s] = __ldcg(reinterpret_cast<const float4 *>(gin + (op[s] - o0) * D + c * 4));
        const float4 w4 = *reinterpret_cast<const float4 *>(weight + o);
        const float4 a4 = *reinterpret_cast<const float4 *>(state1 + o);
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (opt == 1) v4 = *reinterpret_cast<const float4 *>(state2 + o);
        double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int s = 0; s < NFW; ++s)  // source rank ascending
            if (op[s] >= 0) {
                g[0] = __dadd_rn(g[0], (double)x[s].x);
                g[1] = __dadd_rn(g[1], (double)x[s].y);
                g[2] = __dadd_rn(g[2], (double)x[s].z);
                g[3] = __dadd_rn(g[3], (double)x[s].w);
            }
        float ww[4] = {w4.x, w4.y, w4.z, w4.w};
        float ss[4] = {a4.x, a4.y, a4.z, a4.w};
        float v2[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float gg = __double2float_rn(g[k]);
            if (opt == 0) {
                const float acc = __fadd_rn(ss[k], __fmul_rn(gg, gg));
                ss[k] = acc;
                ww[k] = __fsub_rn(ww[k], __fmul_rn(lr, __fdiv_rn(gg, __fadd_rn(__fsqrt_rn(acc), eps))));
            } else {
                const float mo = ss[k], vo = v2[k];
                const float mu = __fmul_rn(__fsub_rn(gg, mo), __fsub_rn(1.0f, beta1));
                const float vu = __fmul_rn(__fsub_rn(__fmul_rn(gg, gg), vo), __fsub_rn(1.0f, beta2));
                const float mn = __fadd_rn(mu, mo), vn = __fadd_rn(vu, vo);
                ss[k] = mn;
                v2[k] = vn;
                ww[k] = __fsub_rn(ww[k], __fmul_rn(adam_ss, __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), eps))));
            }
        }
        *reinterpret_cast<float4 *>(weight + o) = make_float4(ww[0], ww[1], ww[2], ww[3]);
        *reinterpret_cast<float4 *>(state1 + o) = make_float4(ss[0], ss[1], ss[2], ss[3]);
        if (opt == 1) *reinterpret_cast<float4 *>(state2 + o) = make_float4(v2[0], v2[1], v2[2], v2[3]);
    }
}

// G rows written by the peers before the barrier: L2 only (the .cg path of __ldcg), 32 B at once
__device__ __forceinline__ f8 ldcg_f8(const float *p) {
    f8 r;
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
    return r;
}

// k_p2p_update with one thread per 32-B chunk (D % 8 == 0, every pack's rows and the receive
// buffer 32-B aligned): 256-bit loads and stores, half the memory instructions of the 16-B form
// for the same bytes in flight.  Same arithmetic, same order.
template <int D, int NFW, bool LIST>
__global__ void __launch_bounds__(256) k_p2p_update8(P2PArgs a, int pack, float *weight, float *state1,
                                                     float *state2, int opt, float lr, float eps, float beta1,
                                                     float beta2, float adam_ss) {
    constexpr int V8 = D / 8;
    if (__ldcg(a.err) & ERR_PEER_TIMEOUT) return;
    const int64_t o0 = a.pack_ostart[pack];
    const int64_t n = (LIST ? (int64_t)a.ocount[pack] : a.pack_ostart[pack + 1] - o0) * V8;
    const int64_t rb = a.row_base[pack];
    const float *gin = a.peer.ogbuf[a.rank] + a.pack_fbase[pack];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t opos = o0 + e / V8;
        const int32_t row = LIST ? __ldg(a.olist + opos) : __ldg(a.lrow + opos);
        const int32_t src = LIST ? 0 : __ldg(a.osrc + opos);  // (LIST: every listed row is updated)
        const int c = (int)(e % V8);
        const int32_t *dt = a.dtab + (rb + row) * a.W;
        int32_t op[NFW];
#pragma unroll
        for (int s = 0; s < NFW; ++s) op[s] = s < a.W ? __ldcg(dt + s) : -1;
        bool leader = true;
#pragma unroll
        for (int s = 0; s < NFW; ++s) leader = leader && !(s < src && op[s] >= 0);
        if (!leader) continue;
        const int64_t o = (int64_t)row * D + c * 8;
        f8 x[NFW];
#pragma unroll
        for (int s = 0; s < NFW; ++s)
            if (op[s] >= 0) x[s] = ldcg_f8(gin + (op[s] - o0) * D + c * 8);
        f8 w8 = ld_f8(weight + o), a8 = ld_f8(state1 + o), v8;
        if (opt == 1) v8 = ld_f8(state2 + o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double g = 0.0;
#pragma unroll
            for (int s = 0; s < NFW; ++s)  // source rank ascending
                if (op[s] >= 0) g = __dadd_rn(g, (double)x[s].v[k]);
            const float gg = __double2float_rn(g);
            if (opt == 0) {
                const float acc = __fadd_rn(a8.v[k], __fmul_rn(gg, gg));
                a8.v[k] = acc;
                w8.v[k] = __fsub_rn(w8.v[k], __fmul_rn(lr, __fdiv_rn(gg, __fadd_rn(__fsqrt_rn(acc), eps))));
            } else {
                const float mo = a8.v[k], vo = v8.v[k];
                const float mu = __fmul_rn(__fsub_rn(gg, mo), __fsub_rn(1.0f, beta1));
                const float vu = __fmul_rn(__fsub_rn(__fmul_rn(gg, gg), vo), __fsub_rn(1.0f, beta2));
                const float mn = __fadd_rn(mu, mo), vn = __fadd_rn(vu, vo);
                a8.v[k] = mn;
                v8.v[k] = vn;
                w8.v[k] = __fsub_rn(w8.v[k], __fmul_rn(adam_ss, __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), eps))));
            }
        }
        st_f8(weight + o, w8);
        st_f8(state1 + o, a8);
        if (opt == 1) st_f8(state2 + o, v8);
    }
}

// ------------------------------------------------------------------------------------------
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

void launch_p2p_signal(const P2PArgs &a, int slot, cudaStream_t s) { k_p2p_signal<<<1, 32, 0, s>>>(a, slot); }
void launch_p2p_wait(const P2PArgs &a, int slot, cudaStream_t s) { k_p2p_wait<<<1, 32, 0, s>>>(a, slot); }
void launch_p2p_tables(const P2PArgs &a, cudaStream_t s) { k_p2p_tables<<<1, 1024, 0, s>>>(a); }
void launch_p2p_dst_insert(const P2PArgs &a, int num_sms, cudaStream_t s) {
    k_p2p_dst_insert<<<(unsigned)num_sms * 4, 256, 0, s>>>(a);
}
void launch_p2p_leaders(const P2PArgs &a, int num_sms, cudaStream_t s) {
    k_p2p_leaders<<<(unsigned)num_sms * 4, 256, 0, s>>>(a);
}
void launch_p2p_reset(const P2PArgs &a, int num_sms, cudaStream_t s) {
    k_p2p_reset<<<(unsigned)num_sms * 4, 256, 0, s>>>(a);
}
void launch_p2p_gather(int D, const P2PArgs &a, const float *weight, int pack, int num_sms, cudaStream_t s,
                       bool vec8) {
    if (vec8 && D % 8 == 0 && D >= 16) {
        switch (D) {
            case 16: k_p2p_gather8<16><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 32: k_p2p_gather8<32><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 64: k_p2p_gather8<64><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 128: k_p2p_gather8<128><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 256: k_p2p_gather8<256><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 384: k_p2p_gather8<384><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            case 512: k_p2p_gather8<512><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack); return;
            default: break;
        }
    }
#define CALL(DD) k_p2p_gather<DD><<<(unsigned)num_sms * 16, 256, 0, s>>>(a, weight, pack)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
template <bool L>
static void update_dispatch(int D, const P2PArgs &a, int pack, float *w, float *s1, float *s2, int opt, float lr,
                            float eps, float b1, float b2, float ss, int num_sms, cudaStream_t s, bool vec8) {
    const unsigned grid = (unsigned)num_sms * 16;
    if (vec8 && D % 8 == 0 && D >= 16) {  // (D = 8: one thread per row measured slower than two)
#define DISPATCH8(D, CALL)          \
    switch (D) {                    \
        case 16: CALL(16); break;   \
        case 32: CALL(32); break;   \
        case 64: CALL(64); break;   \
        case 128: CALL(128); break; \
        case 256: CALL(256); break; \
        case 384: CALL(384); break; \
        case 512: CALL(512); break; \
        default: break;             \
    }
        if (a.W <= 2) {
#define CALL(DD) k_p2p_update8<DD, 2, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
            DISPATCH8(D, CALL)
#undef CALL
        } else if (a.W <= 4) {
#define CALL(DD) k_p2p_update8<DD, 4, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
            DISPATCH8(D, CALL)
#undef CALL
        } else {
#define CALL(DD) k_p2p_update8<DD, 8, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
            DISPATCH8(D, CALL)
#undef CALL
        }
#undef DISPATCH8
        return;
    }
    if (a.W <= 2) {
#define CALL(DD) k_p2p_update<DD, 2, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
        PICASSO_DISPATCH_D(D, CALL)
#undef CALL
    } else if (a.W <= 4) {
#define CALL(DD) k_p2p_update<DD, 4, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
        PICASSO_DISPATCH_D(D, CALL)
#undef CALL
    } else {
#define CALL(DD) k_p2p_update<DD, 8, L><<<grid, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
        PICASSO_DISPATCH_D(D, CALL)
#undef CALL
    }
}

void launch_p2p_update(int D, const P2PArgs &a, int pack, float *w, float *s1, float *s2, int opt, float lr, float eps,
                       float b1, float b2, float ss, int num_sms, cudaStream_t s, bool vec8, bool list) {
    if (list) update_dispatch<true>(D, a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss, num_sms, s, vec8);
    else update_dispatch<false>(D, a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss, num_sms, s, vec8);
}

}  // namespace picasso
