// p2p.cu — the row-sharded exchange over NVLink peer memory (world W > 1, one GPU per rank).
//
// Every rank exposes one IPC-shared window: barrier flags, its bucket counts, its send list
// (requested local rows, owner-major), and its rows/G buffer in the send layout.  The owner
// side then needs no staged all-to-all (SURVEY §8(f) "kernel-initiated Shuffle&Stitch"):
//   k_p2p_blocks : owner block table from the peers' bucket counts (device-side sizes: no host
//                  synchronisation, so the whole step can be captured in a CUDA graph)
//   k_p2p_insert : reads each requested key straight from the requester's send list (NVLink
//                  loads) and inserts it in the owner hash (first occurrence, as k_owner_insert)
//   k_p2p_gather : gathers the owner's rows and stores them straight into each requester's rows
//                  buffer at the slot its send layout reserved (NVLink stores): Gather + Shuffle
//                  + Stitch in one kernel, the transfer overlapping the gather row by row
//   k_p2p_update : pulls each owner-unique row's <= W gradient rows from the requesters' G
//                  buffers (source rank ascending, fp64, reading O6') and applies the optimizer
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
__global__ void k_p2p_signal(P2PArgs a, int phase) {
    if (threadIdx.x != 0) return;
    const uint32_t e = ++a.epoch[phase];
    __threadfence_system();
    for (int q = 0; q < a.W; ++q) st_release_sys(a.peer.flags[q] + phase * kP2PMaxW + a.rank, e);
}

__global__ void k_p2p_wait(P2PArgs a, int phase) {
    const int q = threadIdx.x;
    if (q < a.W) {
        const uint32_t e = a.epoch[phase];
        const uint32_t *f = a.peer.flags[a.rank] + phase * kP2PMaxW + q;
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
// Owner block table, pack-major (pack p, source s): ostart (owner-stream position), rstart =
// index of the block's first key in s's send list, rroff = float offset of its first row in s's
// rows buffer.  One block of W*P <= 1024 threads.
__global__ void __launch_bounds__(1024) k_p2p_blocks(P2PArgs a) {
    __shared__ int32_t wsum[32];
    __shared__ int64_t s_total;
    const int t = threadIdx.x, nb = a.W * a.P;
    const int p = t / a.W, s = t - (t / a.W) * a.W;
    int32_t c = 0;
    int64_t ks = 0, gs = 0;
    if (t < nb) {
        const int32_t *bc = a.peer.bcount[s];
        const int me = a.rank * a.P + p;
        for (int b = 0; b < me; ++b) {  // s's buckets before (rank, p): owner-major, then pack
            const int32_t x = __ldcv(bc + b);
            ks += x;
            gs += (int64_t)x * __ldg(a.pack_dim + (b % a.P));
        }
        c = __ldcv(bc + me);
        a.cnt_recv[s * a.P + p] = c;
    }
    // block exclusive scan of c in t order
    const int lane = t & 31, w = t >> 5;
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
}

__device__ __forceinline__ int owner_block_p(const OwnerBlock *blk, int nb, int64_t opos) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (blk[mid].ostart <= opos) lo = mid; else hi = mid;
    }
    return lo;
}

// requested key -> owner hash; per owner position: local row, source, float offset of the
// requester's row slot
__global__ void __launch_bounds__(256) k_p2p_insert(P2PArgs a, Slot *table, uint32_t cap_mask) {
    __shared__ OwnerBlock sb[kMaxOwnerBlocks];
    const int nb = a.W * a.P;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = a.oblk[i];
    __syncthreads();
    const int64_t R = *a.R;
    const int64_t opos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = opos < R;
    unsigned long long key = 0;
    if (valid) {
        const int k = owner_block_p(sb, nb, opos);
        const int64_t j = opos - sb[k].ostart;
        const int32_t lr = __ldcv(a.peer.send_keys[sb[k].src] + sb[k].rstart + j);
        a.lrow[opos] = lr;
        a.osrc[opos] = sb[k].src;
        a.roff[opos] = sb[k].rroff + j * __ldg(a.pack_dim + sb[k].pack);
        key = (unsigned long long)(a.pack_key_off[sb[k].pack] + (int64_t)lr);
        if (a.fcnt) atomicAdd(a.fcnt + a.fcnt_off[sb[k].pack] + lr, 1u);  // FCounter (Alg. 1)
    }
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(vmask, key);
    const int leader = __ffs(peers) - 1;
    uint32_t slot = 0;
    if (lane == leader) {
        slot = slot_hash(key) & cap_mask;
        for (uint32_t probe = 0;; ++probe) {
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(&table[slot].key);
            if (cur == kEmptyKey) cur = atomicCAS(&table[slot].key, kEmptyKey, key);
            if (cur == kEmptyKey || cur == key) break;
            slot = (slot + 1) & cap_mask;
            if (probe > cap_mask) {
                atomicOr(a.err, ERR_CAPACITY);
                break;
            }
        }
        atomicMin(&table[slot].minpos, (unsigned int)opos);
    }
    slot = __shfl_sync(vmask, slot, leader);
    a.oslot[opos] = (int32_t)slot;
}

// contrib[ou * W + src] = owner position of source src's request for owner-unique row ou
__global__ void k_p2p_contrib(P2PArgs a) {
    const int64_t R = *a.R;
    for (int64_t opos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; opos < R;
         opos += (int64_t)gridDim.x * blockDim.x)
        a.contrib[(int64_t)a.oinv[opos] * a.W + a.osrc[opos]] = (int32_t)opos;
}

// owner rows -> the requesters' rows buffers (peer stores)
template <int D>
__global__ void __launch_bounds__(256) k_p2p_gather(P2PArgs a, const float *weight, int pack) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES, RB = 4;
    const int li = threadIdx.x % LANES;
    const int64_t o0 = a.pack_ostart[pack], o1 = a.pack_ostart[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t ob = o0 + grp * RB; ob < o1; ob += ngrp * RB) {
        float4 v[RB][VPL];
        float *dst[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const int64_t opos = ob + r;
            dst[r] = nullptr;
            if (opos < o1) {
                dst[r] = a.peer.gbuf[a.osrc[opos]] + a.roff[opos] + li * 4;
                const float *src = weight + (int64_t)a.lrow[opos] * D + li * 4;
#pragma unroll
                for (int q = 0; q < VPL; ++q) v[r][q] = ldg_f4(src + q * LANES * 4);
            }
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (dst[r])
#pragma unroll
                for (int q = 0; q < VPL; ++q) __stcg(reinterpret_cast<float4 *>(dst[r] + q * LANES * 4), v[r][q]);
    }
}

// per owner-unique row: its <= W gradient rows pulled from the requesters (source ascending),
// summed in fp64, rounded once, Adagrad / lazy Adam
template <int D>
__global__ void __launch_bounds__(256) k_p2p_update(P2PArgs a, int pack, float *weight, float *state1, float *state2,
                                                    int opt, float lr, float eps, float beta1, float beta2,
                                                    float adam_ss) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t u0 = a.opack_ustart[pack], u1 = a.opack_ustart[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t ou = u0 + grp; ou < u1; ou += ngrp) {
        const int64_t row = (int64_t)(a.ouid_key[ou] - (unsigned long long)a.pack_key_off[pack]);
        const int64_t o = row * D + li * 4;
        float4 w[VPL], s1[VPL], s2[VPL];
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
            w[q] = *reinterpret_cast<const float4 *>(weight + o + q * LANES * 4);
            s1[q] = *reinterpret_cast<const float4 *>(state1 + o + q * LANES * 4);
            if (opt == 1) s2[q] = *reinterpret_cast<const float4 *>(state2 + o + q * LANES * 4);
        }
        double g[VPL][4];
#pragma unroll
        for (int q = 0; q < VPL; ++q) g[q][0] = g[q][1] = g[q][2] = g[q][3] = 0.0;
        constexpr int NF = VPL == 1 ? kP2PMaxW : 2;  // contributions in flight at once
        for (int s0 = 0; s0 < a.W; s0 += NF) {
            float4 c[NF][VPL];
            int32_t ci[NF];
#pragma unroll
            for (int k = 0; k < NF; ++k) {
                ci[k] = s0 + k < a.W ? a.contrib[ou * a.W + s0 + k] : -1;
                if (ci[k] >= 0) {
                    const float *gr = a.peer.gbuf[s0 + k] + a.roff[ci[k]] + li * 4;
#pragma unroll
                    for (int q = 0; q < VPL; ++q) c[k][q] = __ldcv(reinterpret_cast<const float4 *>(gr + q * LANES * 4));
                }
            }
#pragma unroll
            for (int k = 0; k < NF; ++k)  // source rank ascending
                if (ci[k] >= 0)
#pragma unroll
                    for (int q = 0; q < VPL; ++q) {
                        g[q][0] = __dadd_rn(g[q][0], (double)c[k][q].x);
                        g[q][1] = __dadd_rn(g[q][1], (double)c[k][q].y);
                        g[q][2] = __dadd_rn(g[q][2], (double)c[k][q].z);
                        g[q][3] = __dadd_rn(g[q][3], (double)c[k][q].w);
                    }
        }
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
            float ww[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
            float ss[4] = {s1[q].x, s1[q].y, s1[q].z, s1[q].w};
            float v2[4] = {s2[q].x, s2[q].y, s2[q].z, s2[q].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float gg = __double2float_rn(g[q][e]);
                if (opt == 0) {
                    const float acc = __fadd_rn(ss[e], __fmul_rn(gg, gg));
                    ss[e] = acc;
                    ww[e] = __fsub_rn(ww[e], __fmul_rn(lr, __fdiv_rn(gg, __fadd_rn(__fsqrt_rn(acc), eps))));
                } else {
                    const float mo = ss[e], vo = v2[e];
                    const float mu = __fmul_rn(__fsub_rn(gg, mo), __fsub_rn(1.0f, beta1));
                    const float vu = __fmul_rn(__fsub_rn(__fmul_rn(gg, gg), vo), __fsub_rn(1.0f, beta2));
                    const float mn = __fadd_rn(mu, mo), vn = __fadd_rn(vu, vo);
                    ss[e] = mn;
                    v2[e] = vn;
                    ww[e] = __fsub_rn(ww[e], __fmul_rn(adam_ss, __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), eps))));
                }
            }
            *reinterpret_cast<float4 *>(weight + o + q * LANES * 4) = make_float4(ww[0], ww[1], ww[2], ww[3]);
            *reinterpret_cast<float4 *>(state1 + o + q * LANES * 4) = make_float4(ss[0], ss[1], ss[2], ss[3]);
            if (opt == 1)
                *reinterpret_cast<float4 *>(state2 + o + q * LANES * 4) = make_float4(v2[0], v2[1], v2[2], v2[3]);
        }
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

void launch_p2p_signal(const P2PArgs &a, int phase, cudaStream_t s) { k_p2p_signal<<<1, 32, 0, s>>>(a, phase); }
void launch_p2p_wait(const P2PArgs &a, int phase, cudaStream_t s) { k_p2p_wait<<<1, 32, 0, s>>>(a, phase); }
void launch_p2p_blocks(const P2PArgs &a, cudaStream_t s) { k_p2p_blocks<<<1, 1024, 0, s>>>(a); }
void launch_p2p_insert(const P2PArgs &a, Slot *table, uint32_t cap_mask, cudaStream_t s) {
    if (a.max_recv > 0) k_p2p_insert<<<(unsigned)((a.max_recv + 255) / 256), 256, 0, s>>>(a, table, cap_mask);
}
void launch_p2p_contrib(const P2PArgs &a, int num_sms, cudaStream_t s) {
    k_p2p_contrib<<<(unsigned)num_sms * 4, 256, 0, s>>>(a);
}
void launch_p2p_gather(int D, const P2PArgs &a, const float *weight, int pack, int num_sms, cudaStream_t s) {
#define CALL(DD) k_p2p_gather<DD><<<(unsigned)num_sms * 8, 256, 0, s>>>(a, weight, pack)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_p2p_update(int D, const P2PArgs &a, int pack, float *w, float *s1, float *s2, int opt, float lr, float eps,
                       float b1, float b2, float ss, int num_sms, cudaStream_t s) {
#define CALL(DD) k_p2p_update<DD><<<(unsigned)num_sms * 8, 256, 0, s>>>(a, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

}  // namespace picasso
