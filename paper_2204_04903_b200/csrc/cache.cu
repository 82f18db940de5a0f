// cache.cu — HybridHash on B200 (Alg. 1), row-sharded setting.
//
// Hot storage = the top-k rows by FCounter, replicated in every rank's HBM (weights and
// optimizer state); cold storage = the row-sharded tables reached over NVLink.  A unique key
// found in the hot index is served from the local replica and leaves the AllToAllv; its
// gradient rows are summed over the ranks (AllReduce) and every rank applies the same
// optimizer step to its replica, so the replicas stay bitwise identical and the result is
// the one the uncached step computes ("tier transparency").  FCounter counts every
// key once per rank-step in which it is in the rank's unique set (reading O11): owners count
// the keys they receive, ranks count their hot hits per slot.  The refresh (Alg. 1)
// writes replicas back to the owners, merges the counts, selects the global top-k by
// (count desc, pack asc, key asc) within the capacity, and fetches the new rows.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "kernels.h"
#include "multi.h"

namespace picasso {

__global__ void k_hot_probe(MultiArgs m) {
    const int32_t U = *m.d_total;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = m.unique_gkey[u];
        uint32_t s = slot_hash(key) & m.hot_mask;
        int32_t hs = -1;
        for (uint32_t probe = 0; probe <= m.hot_mask; ++probe) {
            const unsigned long long k = m.hot_index[s].key;
            if (k == key) {
                hs = (int32_t)m.hot_index[s].minpos;
                break;
            }
            if (k == kEmptyKey) break;
            s = (s + 1) & m.hot_mask;
        }
        m.hslot[u] = hs;
        if (hs >= 0) atomicAdd(m.hot_cnt + hs, 1u);  // FCounter, post-unique, this rank
    }
}

// replica rows of the hot slots after the summed gradient (same arithmetic on every rank)
template <int D>
__global__ void __launch_bounds__(256) k_hot_update(MultiArgs m, int pack, int opt, float lr, float eps, float beta1,
                                                    float beta2, float adam_ss) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t s0 = m.hot_pslot[pack], s1e = m.hot_pslot[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t s = s0 + grp; s < s1e; s += ngrp) {
        if (m.hot_touch[s] == 0.0f) continue;  // untouched rows stay bitwise unchanged (O9)
        const int64_t i = s - s0;
        float *w = m.hot_arena + m.hot_w_off[pack] + i * D + li * 4;
        float *a1 = m.hot_arena + m.hot_s1_off[pack] + i * D + li * 4;
        float *a2 = m.hot_arena + m.hot_s2_off[pack] + i * D + li * 4;
        const float *g = m.hot_g + m.hot_g_off[pack] + i * D + li * 4;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
            const float4 g4 = *reinterpret_cast<const float4 *>(g + q * LANES * 4);
            float4 w4 = *reinterpret_cast<float4 *>(w + q * LANES * 4);
            float4 s4 = *reinterpret_cast<float4 *>(a1 + q * LANES * 4);
            float4 v4 = opt == 1 ? *reinterpret_cast<float4 *>(a2 + q * LANES * 4) : make_float4(0, 0, 0, 0);
            float gg[4] = {g4.x, g4.y, g4.z, g4.w}, ww[4] = {w4.x, w4.y, w4.z, w4.w};
            float ss[4] = {s4.x, s4.y, s4.z, s4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (opt == 0) {
                    const float acc = __fadd_rn(ss[e], __fmul_rn(gg[e], gg[e]));
                    ss[e] = acc;
                    ww[e] = __fsub_rn(ww[e], __fmul_rn(lr, __fdiv_rn(gg[e], __fadd_rn(__fsqrt_rn(acc), eps))));
                } else {
                    const float mo = ss[e], vo = vv[e];
                    const float mu = __fmul_rn(__fsub_rn(gg[e], mo), __fsub_rn(1.0f, beta1));
                    const float vu = __fmul_rn(__fsub_rn(__fmul_rn(gg[e], gg[e]), vo), __fsub_rn(1.0f, beta2));
                    const float mn = __fadd_rn(mu, mo), vn = __fadd_rn(vu, vo);
                    ss[e] = mn;
                    vv[e] = vn;
                    ww[e] = __fsub_rn(ww[e], __fmul_rn(adam_ss, __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), eps))));
                }
            }
            *reinterpret_cast<float4 *>(w + q * LANES * 4) = make_float4(ww[0], ww[1], ww[2], ww[3]);
            *reinterpret_cast<float4 *>(a1 + q * LANES * 4) = make_float4(ss[0], ss[1], ss[2], ss[3]);
            if (opt == 1) *reinterpret_cast<float4 *>(a2 + q * LANES * 4) = make_float4(vv[0], vv[1], vv[2], vv[3]);
        }
    }
}

// loopback AllReduce: sum the W ranks' buffers in rank order into dst (n floats)
__global__ void k_sum_ranks(RankPtrs src, int W, float *dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float s = static_cast<const float *>(src.p[0])[i];
        for (int r = 1; r < W; ++r) s = __fadd_rn(s, static_cast<const float *>(src.p[r])[i]);
        dst[i] = s;
    }
}
__global__ void k_sum_ranks_u32(RankPtrs src, int W, uint32_t *dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int r = 0; r < W; ++r) s += static_cast<const uint32_t *>(src.p[r])[i];
        dst[i] = s;
    }
}

// ---- refresh ------------------------------------------------------------------------------
// replicas -> owners' shards (owned hot keys), and the summed hot counts into FCounter
template <int D>
__global__ void __launch_bounds__(256) k_writeback(MultiArgs m, int pack, const unsigned long long *hot_keys,
                                                   float *weight, float *state1, float *state2, int nst,
                                                   const uint32_t *cnt_sum, int rank) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t s0 = m.hot_pslot[pack], s1e = m.hot_pslot[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t s = s0 + grp; s < s1e; s += ngrp) {
        const int64_t key = (int64_t)(hot_keys[s] - (unsigned long long)m.pack_key_off[pack]);
        if (key % m.W != rank) continue;
        const int64_t lr = key / m.W, i = s - s0;
        if (li == 0) m.fcnt[m.fcnt_off[pack] + lr] += cnt_sum[s];
        float *dst[3] = {weight, state1, state2};
        const int64_t off[3] = {m.hot_w_off[pack], m.hot_s1_off[pack], m.hot_s2_off[pack]};
        for (int a = 0; a < nst; ++a)
#pragma unroll
            for (int q = 0; q < VPL; ++q)
                *reinterpret_cast<float4 *>(dst[a] + lr * D + li * 4 + q * LANES * 4) =
                    *reinterpret_cast<const float4 *>(m.hot_arena + off[a] + i * D + li * 4 + q * LANES * 4);
    }
}

// FCounter histogram of the owned rows (counts clamped to kCntBins - 1)
constexpr int kCntBins = 1 << 16;
// Most rows have small counts (Zipf tail): those bins are counted per block in shared memory
// with warp-aggregated adds, and merged once per block; large counts go straight to global.
constexpr int kSmallBins = 1024;
__global__ void __launch_bounds__(256) k_count_hist(const uint32_t *fcnt, int64_t n, uint32_t *hist) {
    __shared__ uint32_t sh[kSmallBins];
    for (int i = threadIdx.x; i < kSmallBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < n;
         b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b0 + lane;
        const uint32_t c = i < n ? __ldg(fcnt + i) : 0u;
        const uint32_t bin = c < kCntBins ? c : kCntBins - 1;
        const unsigned active = __ballot_sync(0xffffffffu, c != 0);
        if (c) {
            const unsigned peers = __match_any_sync(active, bin);
            if (lane == __ffs(peers) - 1) {
                if (bin < kSmallBins) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
                else atomicAdd(hist + bin, (uint32_t)__popc(peers));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSmallBins; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// ---- the selection (Alg. 1 L515 top-k): every rank finds the same global threshold from
// AllReduced histograms, so no candidate list ever leaves its owner.  Rows are taken by (count
// desc, key asc) while their bytes fit: all rows above the threshold count c*, then the rows at
// c* in ascending key up to the key cut.
__device__ __forceinline__ uint32_t cnt_bin(uint32_t c) { return c < kCntBins ? c : kCntBins - 1; }

// byte units (16 B) of pack p's owned rows at count c*, by global-key bin.  Each thread walks
// kRun consecutive rows (consecutive keys, stride W) and adds once per bin it leaves: one bin
// holds thousands of consecutive rows, so per-row atomics would all hit the same address.
constexpr int kRun = 64;
__global__ void k_tie_keyhist(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                              uint32_t unit, uint32_t *hist) {
    for (int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun; r0 < n;
         r0 += (int64_t)gridDim.x * blockDim.x * kRun) {
        int64_t bin = -1;
        uint32_t acc = 0;
        for (int64_t r = r0; r < r0 + kRun && r < n; ++r) {
            if (cnt_bin(__ldg(fcnt + r)) != cstar) continue;
            const int64_t b = (key0 + r * W) >> kshift;
            if (b != bin) {
                if (acc) atomicAdd(hist + bin, acc);
                bin = b;
                acc = 0;
            }
            acc += unit;
        }
        if (acc) atomicAdd(hist + bin, acc);
    }
}

// this owner's rows at count c* inside key bin b* (the key cut falls inside it)
__global__ void k_tie_bin_collect(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                                  int64_t bstar, unsigned long long *out, int32_t *out_n, int32_t cap) {
    const int64_t lo = ((bstar << kshift) - key0 + W - 1) / W, hi = (((bstar + 1) << kshift) - key0 + W - 1) / W;
    for (int64_t r = max(lo, (int64_t)0) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < min(hi, n);
         r += (int64_t)gridDim.x * blockDim.x)
        if (cnt_bin(__ldg(fcnt + r)) == cstar) {
            const int32_t o = atomicAdd(out_n, 1);
            if (o < cap) out[o] = (unsigned long long)(key0 + r * W);
        }
}

// selected owned rows -> bits of the global selection bitmap (owners set disjoint bits); each
// thread builds the words of kRun consecutive rows in a register and ORs each word once
__global__ void k_select_bits(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t kcut, int64_t key0, int32_t W,
                              uint32_t *bits) {
    for (int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun; r0 < n;
         r0 += (int64_t)gridDim.x * blockDim.x * kRun) {
        int64_t word = -1;
        uint32_t m = 0;
        for (int64_t r = r0; r < r0 + kRun && r < n; ++r) {
            const uint32_t c = __ldg(fcnt + r);
            if (c == 0) continue;
            const uint32_t b = cnt_bin(c);
            const int64_t key = key0 + r * W;
            if (!(b > cstar || (b == cstar && key <= kcut))) continue;
            if ((key >> 5) != word) {
                if (m) atomicOr(bits + word, m);
                word = key >> 5;
                m = 0;
            }
            m |= 1u << (key & 31);
        }
        if (m) atomicOr(bits + word, m);
    }
}

// bitmap -> hot keys in ascending key order (slots grouped by pack: the key space is pack-major)
constexpr int kBitWords = 1024;  // words per block
__global__ void __launch_bounds__(kBitWords) k_bits_count(const uint32_t *bits, int64_t nw, int32_t *blk) {
    using BR = cub::BlockReduce<int32_t, kBitWords>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t w = (int64_t)blockIdx.x * kBitWords + threadIdx.x;
    const int32_t c = BR(tmp).Sum(w < nw ? __popc(bits[w]) : 0);
    if (threadIdx.x == 0) blk[blockIdx.x] = c;
}
__global__ void __launch_bounds__(1024) k_bits_scan(int32_t *blk, int64_t nb, int32_t *total) {
    using BS = cub::BlockScan<int32_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        const int64_t i = b0 + threadIdx.x;
        int32_t e, agg;
        BS(tmp).ExclusiveSum(i < nb ? blk[i] : 0, e, agg);
        if (i < nb) blk[i] = carry + e;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}
__global__ void __launch_bounds__(kBitWords) k_bits_emit(const uint32_t *bits, int64_t nw, const int32_t *blk,
                                                         unsigned long long *keys, int32_t kmax) {
    using BS = cub::BlockScan<int32_t, kBitWords>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t w = (int64_t)blockIdx.x * kBitWords + threadIdx.x;
    uint32_t x = w < nw ? bits[w] : 0u;
    int32_t e;
    BS(tmp).ExclusiveSum(__popc(x), e);
    int32_t o = blk[blockIdx.x] + e;
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        if (o < kmax) keys[o] = (unsigned long long)(w * 32 + b);
        ++o;
    }
}

// slot range of each pack (first hot key >= pack_key_off[p]) and each slot's staging offset
__global__ void k_hot_layout(const unsigned long long *keys, int32_t k, const int64_t *pack_key_off, int32_t P,
                             int32_t *pslot) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    int32_t lo = 0, hi = k;
    const unsigned long long v = (unsigned long long)pack_key_off[p];
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (keys[mid] < v) lo = mid + 1; else hi = mid;
    }
    pslot[p] = p == P ? k : lo;
}
__global__ void k_stage_idx(const int32_t *pslot, const int64_t *stage_off, const int32_t *pack_dim, int32_t P, int nst,
                            int32_t k, int64_t *stage_idx) {
    for (int32_t sl = blockIdx.x * blockDim.x + threadIdx.x; sl < k; sl += gridDim.x * blockDim.x) {
        int p = 0;
        while (p + 1 < P && pslot[p + 1] <= sl) ++p;
        stage_idx[sl] = stage_off[p] + (int64_t)(sl - pslot[p]) * nst * pack_dim[p];
    }
}

// new hot rows: owners pack their owned slots (w, s1, s2) in slot order into staging
template <int D>
__global__ void __launch_bounds__(256) k_pack_owned(MultiArgs m, int pack, const unsigned long long *keys,
                                                    const int64_t *stage_idx, const float *weight, const float *state1,
                                                    const float *state2, int nst, float *stage, int rank) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t s0 = m.hot_pslot[pack], s1e = m.hot_pslot[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t s = s0 + grp; s < s1e; s += ngrp) {
        const int64_t key = (int64_t)(keys[s] - (unsigned long long)m.pack_key_off[pack]);
        if (key % m.W != rank) continue;
        const int64_t lr = key / m.W;
        float *dst = stage + stage_idx[s];  // this slot's float offset in the staging
        const float *src[3] = {weight, state1, state2};
        for (int a = 0; a < nst; ++a)
#pragma unroll
            for (int q = 0; q < VPL; ++q)
                *reinterpret_cast<float4 *>(dst + a * D + li * 4 + q * LANES * 4) =
                    *reinterpret_cast<const float4 *>(src[a] + lr * D + li * 4 + q * LANES * 4);
    }
}

// staging (all owners' blocks) -> replica arena; rebuild the hot index (key -> slot)
template <int D>
__global__ void __launch_bounds__(256) k_place(MultiArgs m, int pack, const int64_t *stage_idx, const float *stage,
                                               int nst) {
    constexpr int V4 = D / 4, LANES = V4 < 32 ? V4 : 32, VPL = V4 / LANES;
    const int li = threadIdx.x % LANES;
    const int32_t s0 = m.hot_pslot[pack], s1e = m.hot_pslot[pack + 1];
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t s = s0 + grp; s < s1e; s += ngrp) {
        const int64_t i = s - s0;
        const float *src = stage + stage_idx[s];
        const int64_t off[3] = {m.hot_w_off[pack], m.hot_s1_off[pack], m.hot_s2_off[pack]};
        for (int a = 0; a < nst; ++a)
#pragma unroll
            for (int q = 0; q < VPL; ++q)
                *reinterpret_cast<float4 *>(m.hot_arena + off[a] + i * D + li * 4 + q * LANES * 4) =
                    *reinterpret_cast<const float4 *>(src + a * D + li * 4 + q * LANES * 4);
    }
}

__global__ void k_hot_index(Slot *index, uint32_t mask, const unsigned long long *keys, int32_t k) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const unsigned long long key = keys[s];
    uint32_t h = slot_hash(key) & mask;
    while (true) {
        const unsigned long long prev = atomicCAS(&index[h].key, kEmptyKey, key);
        if (prev == kEmptyKey) {
            index[h].minpos = (unsigned)s;
            return;
        }
        h = (h + 1) & mask;
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

void launch_hot_probe(const MultiArgs &m, int num_sms, cudaStream_t s) {
    k_hot_probe<<<(unsigned)num_sms * 4, 256, 0, s>>>(m);
}
void launch_hot_update(int D, const MultiArgs &m, int pack, int opt, float lr, float eps, float b1, float b2, float ss,
                       int num_sms, cudaStream_t s) {
#define CALL(DD) k_hot_update<DD><<<(unsigned)num_sms * 2, 256, 0, s>>>(m, pack, opt, lr, eps, b1, b2, ss)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_sum_ranks(const RankPtrs &src, int W, float *dst, int64_t n, cudaStream_t s) {
    if (n > 0) k_sum_ranks<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(src, W, dst, n);
}
void launch_sum_ranks_u32(const RankPtrs &src, int W, uint32_t *dst, int64_t n, cudaStream_t s) {
    if (n > 0) k_sum_ranks_u32<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(src, W, dst, n);
}
void launch_writeback(int D, const MultiArgs &m, int pack, const unsigned long long *keys, float *w, float *s1,
                      float *s2, int nst, const uint32_t *cnt_sum, int rank, int num_sms, cudaStream_t s) {
#define CALL(DD) k_writeback<DD><<<(unsigned)num_sms, 256, 0, s>>>(m, pack, keys, w, s1, s2, nst, cnt_sum, rank)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_count_hist(const uint32_t *fcnt, int64_t n, uint32_t *hist, int num_sms, cudaStream_t s) {
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kCntBins, s);
    if (n > 0) k_count_hist<<<(unsigned)num_sms * 4, 256, 0, s>>>(fcnt, n, hist);
}
int count_hist_bins() { return kCntBins; }
void launch_tie_keyhist(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                        uint32_t unit, uint32_t *hist, int num_sms, cudaStream_t s) {
    if (n > 0) k_tie_keyhist<<<(unsigned)num_sms * 4, 256, 0, s>>>(fcnt, n, cstar, key0, W, kshift, unit, hist);
}
void launch_tie_bin_collect(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                            int64_t bstar, unsigned long long *out, int32_t *out_n, int32_t cap, cudaStream_t s) {
    if (n > 0) k_tie_bin_collect<<<64, 256, 0, s>>>(fcnt, n, cstar, key0, W, kshift, bstar, out, out_n, cap);
}
void launch_select_bits(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t kcut, int64_t key0, int32_t W,
                        uint32_t *bits, int num_sms, cudaStream_t s) {
    if (n > 0) k_select_bits<<<(unsigned)num_sms * 4, 256, 0, s>>>(fcnt, n, cstar, kcut, key0, W, bits);
}
// bitmap (nw words) -> keys; blk: [nw / 1024 + 1] scratch; total: [1] device
void launch_bits_compact(const uint32_t *bits, int64_t nw, int32_t *blk, int32_t *total, unsigned long long *keys,
                         int32_t kmax, cudaStream_t s) {
    const int64_t nb = (nw + kBitWords - 1) / kBitWords;
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(int32_t), s);
        return;
    }
    k_bits_count<<<(unsigned)nb, kBitWords, 0, s>>>(bits, nw, blk);
    k_bits_scan<<<1, 1024, 0, s>>>(blk, nb, total);
    k_bits_emit<<<(unsigned)nb, kBitWords, 0, s>>>(bits, nw, blk, keys, kmax);
}
void launch_hot_layout(const unsigned long long *keys, int32_t k, const int64_t *pack_key_off, int32_t P,
                       int32_t *pslot, cudaStream_t s) {
    k_hot_layout<<<(unsigned)((P + 1 + 127) / 128), 128, 0, s>>>(keys, k, pack_key_off, P, pslot);
}
void launch_stage_idx(const int32_t *pslot, const int64_t *stage_off, const int32_t *pack_dim, int32_t P, int nst,
                      int32_t k, int64_t *stage_idx, cudaStream_t s) {
    if (k > 0) k_stage_idx<<<(unsigned)std::min<int64_t>((k + 255) / 256, 4096), 256, 0, s>>>(pslot, stage_off, pack_dim, P, nst, k, stage_idx);
}
void launch_pack_owned(int D, const MultiArgs &m, int pack, const unsigned long long *keys, const int64_t *stage_idx,
                       const float *w, const float *s1, const float *s2, int nst, float *stage, int rank, int num_sms,
                       cudaStream_t s) {
#define CALL(DD) k_pack_owned<DD><<<(unsigned)num_sms, 256, 0, s>>>(m, pack, keys, stage_idx, w, s1, s2, nst, stage, rank)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_place(int D, const MultiArgs &m, int pack, const int64_t *stage_idx, const float *stage, int nst,
                  int num_sms, cudaStream_t s) {
#define CALL(DD) k_place<DD><<<(unsigned)num_sms, 256, 0, s>>>(m, pack, stage_idx, stage, nst)
    PICASSO_DISPATCH_D(D, CALL)
#undef CALL
}
void launch_hot_index(Slot *index, uint32_t mask, const unsigned long long *keys, int32_t k, cudaStream_t s) {
    cudaMemsetAsync(index, 0xFF, sizeof(Slot) * ((size_t)mask + 1), s);
    if (k > 0) k_hot_index<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(index, mask, keys, k);
}

}  // namespace picasso
