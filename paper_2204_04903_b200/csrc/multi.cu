// multi.cu — kernels of the row-sharded multi-GPU path (world W > 1): Partition, the owner
// side of the Shuffle, and the owner's reduce + optimizer update.
//
// Row-wise model parallelism: pack key k lives on rank k mod W
// at local row k div W (reading O3).  Per rank and step:
//   Partition (L211, fused with Unique per L375-379): every unique key of the rank gets a
//     send slot, owner-major, then pack, then first-occurrence order (k_bucket + one stable
//     radix pass + k_send_prep); the same layout, with D_p floats per slot, receives the rows
//     back and later holds the rank's gradient rows — so a unique row's address is row_off[u]
//     in every phase and Stitch needs no separate kernel (L380-382).
//   Owner side: the received keys are viewed pack-major (pack, then source rank, then the
//     requester's order) — the "received lists concatenated by source rank" of reading O2 —
//     and deduplicated with the same hash machinery (first occurrence) (k_owner_insert);
//     rows are gathered into the send buffer (k_gather); contributions of each owner-unique
//     row are indexed by source (k_contrib) so the backward sums them in source-rank order.
//   Backward: the owner sums the <= W received gradient rows of each owner-unique row in fp64,
//     source rank ascending, rounds once and applies Adagrad / lazy Adam (k_owner_update).
#include "kernels.h"
#include "multi.h"

namespace picasso {

// owner = key mod W, local row = key div W (reading O3); shifts when W is a power of two
__device__ __forceinline__ uint64_t key_owner(uint64_t key, int W) {
    return (W & (W - 1)) == 0 ? (key & (uint64_t)(W - 1)) : key % (uint64_t)W;
}
__device__ __forceinline__ uint64_t key_local(uint64_t key, int W) {
    return (W & (W - 1)) == 0 ? (key >> (__ffs(W) - 1)) : key / (uint64_t)W;
}

// ------------------------------------------------------------------------------------------
// bucket of uid u = owner * P + pack; keys/values for one stable radix pass + its histogram
__global__ void __launch_bounds__(kTileThreads) k_bucket(MultiArgs m) {
    __shared__ int32_t h[kMaxRadix];
    const int radix = 1 << m.bucket_bits;
    for (int d = threadIdx.x; d < radix; d += kTileThreads) h[d] = 0;
    __syncthreads();
    const int32_t U = *m.d_total;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kTile; i += kTileThreads) {
        const int64_t u = (int64_t)blockIdx.x * kTile + i;
        const bool valid = u < U;
        int32_t b = 0;
        if (valid) {
            const int64_t p = upper_bound_dev(m.pack_ustart, 0, m.P + 1, (int32_t)u) - 1;
            const uint64_t key = m.unique_gkey[u] - (unsigned long long)m.pack_key_off[p];
            b = (int32_t)key_owner(key, m.W) * m.P + (int32_t)p;
            if (m.hot_k > 0 && m.hslot[u] >= 0) b = m.W * m.P;  // hot: served by the replica, not sent
            m.bkey[u] = b;
            m.bval[u] = (int32_t)u;
        }
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(vm, b);
            if (lane == __ffs(peers) - 1) atomicAdd(&h[b], __popc(peers));
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kTileThreads) m.bhist[(int64_t)d * m.nblk + blockIdx.x] = h[d];
}

// bucket starts (elements) and send-row offsets (floats) from the bucket counts (1 block)
__global__ void k_bucket_prefix(MultiArgs m) {
    if (threadIdx.x != 0) return;
    int64_t e = 0, f = 0;
    for (int b = 0; b < m.W * m.P; ++b) {
        m.bstart[b] = e;
        m.sroff[b] = f;
        const int32_t c = m.bcount[b];
        e += c;
        f += (int64_t)c * m.pack_dim[b % m.P];
    }
    m.bstart[m.W * m.P] = e;
    m.sroff[m.W * m.P] = f;
}

// send slot i <-> uid u; requested local row; float offset of u's row in the rows buffer
__global__ void k_send_prep(MultiArgs m) {
    const int32_t U = *m.d_total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < U; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = m.send_uid[i];
        const int64_t p = upper_bound_dev(m.pack_ustart, 0, m.P + 1, u) - 1;
        const uint64_t key = m.unique_gkey[u] - (unsigned long long)m.pack_key_off[p];
        m.send_pos[u] = (int32_t)i;
        const int32_t hs = m.hot_k > 0 ? m.hslot[u] : -1;
        if (hs >= 0) {  // row of the local replica (offset relative to the rows buffer)
            m.row_off[u] = (int64_t)((m.hot_arena + m.hot_w_off[p] + (int64_t)(hs - m.hot_pslot[p]) * m.pack_dim[p]) -
                                     m.gbuf_base);
            continue;
        }
        const int32_t b = (int32_t)key_owner(key, m.W) * m.P + (int32_t)p;
        m.send_keys[i] = (int32_t)key_local(key, m.W);
        m.row_off[u] = m.sroff[b] + (i - m.bstart[b]) * m.pack_dim[p];
    }
}

// ------------------------------------------------------------------------------------------
// Partition for the peer-memory exchange: the same stable layout as the NCCL driver's sort
// (owner-major, pack, then first-occurrence = uid order inside a bucket, so each bucket is
// exactly oracle_partition's per-owner list of the pack), placed without the sort's second
// buffer: k_bucket counts every 2048-uid tile per bucket, k_scan_rows turns the digit-major
// counts into per-tile bucket offsets, and k_part_place ranks each uid stably inside its tile
// (warp by warp, __match_any_sync) and writes its send slot, requested local row and row offset.
__global__ void __launch_bounds__(kTileThreads) k_part_place(MultiArgs m) {
    constexpr int kWarps = kTileThreads / 32;
    constexpr int kRounds = kTile / kTileThreads;  // 8 rounds of 32 uids per warp
    const int nb = m.W * m.P;  // bucket nb = hot (not sent)
    extern __shared__ int64_t smp[];
    int64_t *s_start = smp, *s_foff = smp + nb + 1;              // [nb+1] each
    int32_t *wcf = reinterpret_cast<int32_t *>(smp + 2 * (nb + 1));  // [kWarps][nb+1]
    auto wc = [&](int ww, int b) -> int32_t & { return wcf[ww * (nb + 1) + b]; };
    for (int i = threadIdx.x; i < kWarps * (nb + 1); i += kTileThreads) wcf[i] = 0;
    if (threadIdx.x == 0) {  // bucket starts (slots) and float offsets (rows buffer)
        int64_t e = 0, f = 0;
        for (int b = 0; b < nb; ++b) {
            s_start[b] = e;
            s_foff[b] = f;
            const int32_t c = m.bcount[b];
            e += c;
            f += (int64_t)c * m.pack_dim[b % m.P];
        }
        s_start[nb] = e;
        s_foff[nb] = f;
    }
    __syncthreads();
    if (blockIdx.x == 0)
        for (int b = threadIdx.x; b <= nb; b += kTileThreads) {
            m.bstart[b] = s_start[b];
            m.sroff[b] = s_foff[b];
        }
    const int32_t U = *m.d_total;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * (32 * kRounds);
    int32_t bk[kRounds], rk[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t u = base + r * 32 + lane;
        bk[r] = u < U ? __ldg(m.bkey + u) : nb + 1 + lane;  // invalid lanes never match a bucket
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // stable rank inside the warp's 256 uids
        const bool valid = base + r * 32 + lane < U;
        const unsigned peers = __match_any_sync(0xffffffffu, bk[r]);
        int32_t before = 0;
        if (valid) before = wc(w, bk[r]);
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wc(w, bk[r]) = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kTileThreads) {  // warp prefixes + this tile's bucket offset
        int32_t run = m.bhist[(int64_t)b * m.nblk + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
            const int32_t t = wc(ww, b);
            wc(ww, b) = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t u = base + r * 32 + lane;
        if (u >= U) continue;
        const int32_t b = bk[r];
        const int64_t p = upper_bound_dev(m.pack_ustart, 0, m.P + 1, (int32_t)u) - 1;
        if (b >= nb) {  // hot: row of the local replica (offset relative to the rows buffer)
            const int32_t hs = m.hslot[u];
            m.send_pos[u] = -1;
            m.row_off[u] = (int64_t)((m.hot_arena + m.hot_w_off[p] + (int64_t)(hs - m.hot_pslot[p]) * m.pack_dim[p]) -
                                     m.gbuf_base);
            continue;
        }
        const uint64_t key = m.unique_gkey[u] - (unsigned long long)m.pack_key_off[p];
        const int32_t j = wc(w, b) + rk[r];  // rank of u inside its bucket (uid order)
        const int64_t i = s_start[b] + j;
        m.send_pos[u] = (int32_t)i;
        m.send_keys[i] = (int32_t)key_local(key, m.W);
        m.row_off[u] = s_foff[b] + (int64_t)j * m.pack_dim[p];
    }
}

// ------------------------------------------------------------------------------------------
// owner stream position -> block (pack-major (p, src)) by a search over the block table
__device__ __forceinline__ int owner_block(const OwnerBlock *blk, int nb, int64_t opos) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (blk[mid].ostart <= opos) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_owner_insert(MultiArgs m, Slot *table, uint32_t cap_mask, int *err) {
    __shared__ OwnerBlock sb[kMaxOwnerBlocks];
    const int nb = m.W * m.P;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = m.oblk[i];
    __syncthreads();
    const int64_t opos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = opos < m.R;
    unsigned long long key = 0;
    if (valid) {
        const int k = owner_block(sb, nb, opos);
        const int64_t i = sb[k].rstart + (opos - sb[k].ostart);
        m.opos_map[opos] = (int32_t)i;
        key = (unsigned long long)(m.pack_key_off[sb[k].pack] + (int64_t)m.recv_keys[i]);
        // FCounter (Alg. 1 L501/L511): one count per requesting rank (its keys are unique)
        if (m.fcnt) atomicAdd(m.fcnt + m.fcnt_off[sb[k].pack] + m.recv_keys[i], 1u);
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
                atomicOr(err, ERR_CAPACITY);
                break;
            }
        }
        atomicMin(&table[slot].minpos, (unsigned int)opos);
    }
    slot = __shfl_sync(vmask, slot, leader);
    m.oslot[opos] = (int32_t)slot;
}

// contrib[ou * W + src] = receive index of source src's request for owner-unique row ou
__global__ void __launch_bounds__(256) k_contrib(MultiArgs m) {
    __shared__ OwnerBlock sb[kMaxOwnerBlocks];
    const int nb = m.W * m.P;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = m.oblk[i];
    __syncthreads();
    const int64_t opos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (opos >= m.R) return;
    const int k = owner_block(sb, nb, opos);
    m.contrib[(int64_t)m.oinv[opos] * m.W + sb[k].src] = m.opos_map[opos];
}

// rows of the owner's shard -> send buffer (requester order); remembers each row's offset
template <int D>
__global__ void __launch_bounds__(256) k_gather(MultiArgs m, const float *weight, int pack) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES, RB = 4;
    __shared__ OwnerBlock sb[kMaxOwnerBlocks];
    const int nb = m.W * m.P;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = m.oblk[i];
    __syncthreads();
    const int li = threadIdx.x % LANES;
    const int64_t o0 = m.pack_ostart[pack], o1 = m.pack_ostart[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t ob = o0 + grp * RB; ob < o1; ob += ngrp * RB) {
        float4 v[RB][VPL];
        int64_t dst[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const int64_t opos = ob + r;
            dst[r] = -1;
            if (opos < o1) {
                const int k = owner_block(sb, nb, opos);
                const int64_t i = sb[k].rstart + (opos - sb[k].ostart);
                dst[r] = sb[k].rroff + (opos - sb[k].ostart) * D;
                const int64_t lr = m.recv_keys[i];
                const float *src = weight + lr * D + li * 4;
#pragma unroll
                for (int q = 0; q < VPL; ++q) v[r][q] = ldg_f4(src + q * LANES * 4);
                if (li == 0) m.rsend_off[i] = dst[r];
            }
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (dst[r] >= 0)
#pragma unroll
                for (int q = 0; q < VPL; ++q)
                    *reinterpret_cast<float4 *>(m.rows_send + dst[r] + li * 4 + q * LANES * 4) = v[r][q];
    }
}

// ------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_owner_update(MultiArgs m, int pack, float *weight, float *state1,
                                                      float *state2, int opt, float lr, float eps, float beta1,
                                                      float beta2, float adam_ss) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t u0 = m.opack_ustart[pack], u1 = m.opack_ustart[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t ou = u0 + grp; ou < u1; ou += ngrp) {
        // owner keys are local rows (requesters send key div W)
        const int64_t row = (int64_t)(m.ouid_key[ou] - (unsigned long long)m.pack_key_off[pack]);
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
        for (int src = 0; src < m.W; ++src) {  // source rank ascending (reading O6)
            const int32_t i = m.contrib[ou * m.W + src];
            if (i < 0) continue;
            const float *gr = m.rows_send + m.rsend_off[i] + li * 4;
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
                const float4 c = ldg_f4(gr + q * LANES * 4);
                g[q][0] = __dadd_rn(g[q][0], (double)c.x);
                g[q][1] = __dadd_rn(g[q][1], (double)c.y);
                g[q][2] = __dadd_rn(g[q][2], (double)c.z);
                g[q][3] = __dadd_rn(g[q][3], (double)c.w);
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

void launch_bucket(const MultiArgs &m, cudaStream_t s) {
    k_bucket<<<(unsigned)m.nblk, kTileThreads, 0, s>>>(m);
}
void launch_bucket_prefix(const MultiArgs &m, cudaStream_t s) { k_bucket_prefix<<<1, 32, 0, s>>>(m); }
void launch_send_prep(const MultiArgs &m, int num_sms, cudaStream_t s) {
    k_send_prep<<<(unsigned)num_sms * 4, 256, 0, s>>>(m);
}
void launch_partition_p2p(const MultiArgs &m, int num_sms, cudaStream_t s) {
    (void)num_sms;
    k_bucket<<<(unsigned)m.nblk, kTileThreads, 0, s>>>(m);
    bucket_scan(m.bhist, m.nblk, m.bcount, 1 << m.bucket_bits, s);
    const int nb = m.W * m.P;
    const size_t sm = sizeof(int64_t) * 2 * (nb + 1) + sizeof(int32_t) * (kTileThreads / 32) * (nb + 1);
    ensure_dyn_smem((const void *)k_part_place, sm);
    k_part_place<<<(unsigned)m.nblk, kTileThreads, sm, s>>>(m);
}
void launch_owner_insert(const MultiArgs &m, Slot *table, uint32_t cap_mask, int *err, cudaStream_t s) {
    if (m.R > 0) k_owner_insert<<<(unsigned)((m.R + 255) / 256), 256, 0, s>>>(m, table, cap_mask, err);
}
void launch_contrib(const MultiArgs &m, cudaStream_t s) {
    if (m.R > 0) k_contrib<<<(unsigned)((m.R + 255) / 256), 256, 0, s>>>(m);
}
void launch_gather(int D, const MultiArgs &m, const float *weight, int pack, int num_sms, cudaStream_t s) {
#define CALL(DD) k_gather<DD><<<(unsigned)num_sms * 4, 256, 0, s>>>(m, weight, pack)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_owner_update(int D, const MultiArgs &m, int pack, float *w, float *s1, float *s2, int opt, float lr,
                         float eps, float b1, float b2, float ss, int num_sms, cudaStream_t s) {
#define CALL(DD) k_owner_update<DD><<<(unsigned)num_sms * 4, 256, 0, s>>>(m, pack, w, s1, s2, opt, lr, eps, b1, b2, ss)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}

}  // namespace picasso
