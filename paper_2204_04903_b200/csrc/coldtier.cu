// coldtier.cu — HybridHash with a host-DRAM cold tier (Alg. 1),
// world == 1, opts.cold_tier = 1.
//
// "We refer to GPU device memory as the Hot-storage and DRAM as the Cold-storage" (L467-468):
// the packs' weights and optimizer state passed to picasso_bind live in pinned, device-mapped
// host memory (CStore; tables larger than HBM fit), and up to cache_max_bytes of HBM hold the
// top-k rows by FCounter (HStore), weights and state together.  Per step:
//   forward   index chain as usual (hash + Unique), then
//     k_ct_probe : per unique key, its hot slot (HStore index) or -1, and FCounter[key] += 1
//                  (Alg. 1; post-unique, reading O11)
//     k_ct_stage : cold rows copied from host memory (PCIe reads of whole rows) into the rows
//                  buffer; hot rows are read in place from HStore (row offsets)
//     pool       : the W > 1 pooling kernels over the row offsets (Stitch fused, as there)
//   backward  transpose + segment-sum (G rows in the rows buffer, pack layout), then
//     k_ct_update: per unique row, the optimizer step on HStore (hot) or on the host row itself
//                  (cold: read-modify-write over PCIe)
//   refresh (Alg. 1, called by the caller after bwd when itr >= warmup and
//   itr % flush == 0, reading O13):
//     k_ct_hist      : capacity cost of the rows at each FCounter value
//     (host)         : the count c* where the prefix of (count desc, pack asc, key asc) — the
//                      order of oracle_hot_select, reading O12 — stops fitting
//     k_ct_tiesum / k_ct_scan / k_ct_select : every row above c*, plus the rows at c* in
//                      ascending global key (= pack asc, key asc) while their cost prefix fits,
//                      compacted in that order (= the new slot order, pack-major)
//     k_ct_layout / k_ct_index : the new HStore layout and index (a second buffer)
//     k_ct_merge     : rows staying hot move HBM -> HBM to their new slots, rows entering are
//                      loaded from CStore, rows leaving are written back to it
// Results equal the uncached step's ("tier transparency"): a row is updated in exactly one
// tier, with the same arithmetic (optim.cuh), and written back when it leaves HStore (capacity
// 0 writes every hot row back: the host tables are then authoritative).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "ctx.h"
#include "optim.cuh"

namespace picasso {
namespace {

constexpr int kCountBuckets = 1 << 16;  // FCounter values >= 65535 share the top bucket

struct CtArgs {
    int32_t P;
    const int32_t *pack_ustart;             // [P+1]
    const unsigned long long *unique_gkey;  // [U]
    const int64_t *pack_key_off;            // [P+1]
    const int32_t *pack_dim;                // [P]
    const int64_t *pack_gbase;              // [P+1] float offset of each pack's rows in the rows buffer
    float *gbuf;                            // rows buffer (staged cold rows; later G rows)
    const Slot *index;                      // HStore index: key -> slot (minpos field)
    uint32_t mask;
    const int32_t *pslot;                   // [P+1] hot slots grouped by pack
    const int64_t *arena_off;               // [3P] float offset of pack p's w / s1 / s2 rows in the arena
    float *arena;
    int32_t *hslot;                         // [U]
    int64_t *row_off;                       // [U] float offset of the row relative to gbuf
    uint32_t *fcnt;                         // [sum pack_rows] FCounter, by global key
    unsigned long long *hits;               // [1] hot uniques of the last forward
    float *const *w;                        // [P] host (device-mapped) tables
    float *const *s1;
    float *const *s2;
    int32_t hot_k;
};

__device__ __forceinline__ int pack_of_gkey(const int64_t *pack_key_off, int P, unsigned long long k) {
    int lo = 0, hi = P;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((unsigned long long)__ldg(pack_key_off + mid) <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_ct_probe(CtArgs a) {
    const int32_t U = __ldg(a.pack_ustart + a.P);
    uint32_t nh = 0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = a.unique_gkey[u];
        int32_t hs = -1;
        if (a.hot_k > 0) {
            uint32_t s = slot_hash(key) & a.mask;
            for (uint32_t probe = 0; probe <= a.mask; ++probe) {
                const unsigned long long k = a.index[s].key;
                if (k == key) {
                    hs = (int32_t)a.index[s].minpos;
                    break;
                }
                if (k == kEmptyKey) break;
                s = (s + 1) & a.mask;
            }
        }
        a.hslot[u] = hs;
        nh += hs >= 0;
        atomicAdd(a.fcnt + key, 1u);  // FCounter(id) += 1, once per step per key (O11)
    }
    if (nh) atomicAdd(a.hits, (unsigned long long)nh);
}

// one thread per 4-float chunk of every unique row (rows buffer = pack layout)
__global__ void __launch_bounds__(256) k_ct_stage(CtArgs a) {
    const int64_t n4 = __ldg(a.pack_gbase + a.P) / 4;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = e * 4;
        int p = 0, hi = a.P;
        while (hi - p > 1) {
            const int mid = (p + hi) >> 1;
            if (__ldg(a.pack_gbase + mid) <= f) p = mid; else hi = mid;
        }
        const int D = __ldg(a.pack_dim + p);
        const int64_t rel = f - __ldg(a.pack_gbase + p);
        const int64_t u = __ldg(a.pack_ustart + p) + rel / D;
        const int c = (int)(rel % D);
        const int32_t hs = a.hslot[u];
        if (hs >= 0) {  // HStore: the pool reads the row in place
            if (c == 0)
                a.row_off[u] = (a.arena + a.arena_off[p] + (int64_t)(hs - a.pslot[p]) * D) - a.gbuf;
            continue;
        }
        if (c == 0) a.row_off[u] = f - c;
        const int64_t row = (int64_t)(a.unique_gkey[u] - (unsigned long long)__ldg(a.pack_key_off + p));
        *reinterpret_cast<float4 *>(a.gbuf + f) = *reinterpret_cast<const float4 *>(a.w[p] + row * D + c);  // CStore
    }
}

__global__ void __launch_bounds__(256) k_ct_update(CtArgs a, OptParams o) {
    const int64_t n4 = __ldg(a.pack_gbase + a.P) / 4;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = e * 4;
        int p = 0, hi = a.P;
        while (hi - p > 1) {
            const int mid = (p + hi) >> 1;
            if (__ldg(a.pack_gbase + mid) <= f) p = mid; else hi = mid;
        }
        const int D = __ldg(a.pack_dim + p);
        const int64_t rel = f - __ldg(a.pack_gbase + p);
        const int64_t u = __ldg(a.pack_ustart + p) + rel / D;
        const int c = (int)(rel % D);
        const int32_t hs = a.hslot[u];
        float *wp, *s1p, *s2p;
        if (hs >= 0) {
            const int64_t r = (int64_t)(hs - a.pslot[p]) * D + c;
            wp = a.arena + a.arena_off[p] + r;
            s1p = a.arena + a.arena_off[a.P + p] + r;
            s2p = a.arena + a.arena_off[2 * a.P + p] + r;
        } else {
            const int64_t r = (int64_t)(a.unique_gkey[u] - (unsigned long long)__ldg(a.pack_key_off + p)) * D + c;
            wp = a.w[p] + r;
            s1p = a.s1[p] + r;
            s2p = o.opt == 1 ? a.s2[p] + r : nullptr;
        }
        const float4 g = *reinterpret_cast<const float4 *>(a.gbuf + f);
        float4 w4 = *reinterpret_cast<float4 *>(wp), s14 = *reinterpret_cast<float4 *>(s1p);
        float4 s24 = o.opt == 1 ? *reinterpret_cast<float4 *>(s2p) : make_float4(0.f, 0.f, 0.f, 0.f);
        opt_step4(o, g, w4, s14, s24);
        *reinterpret_cast<float4 *>(wp) = w4;
        *reinterpret_cast<float4 *>(s1p) = s14;
        if (o.opt == 1) *reinterpret_cast<float4 *>(s2p) = s24;
    }
}

// capacity cost of the rows at each FCounter value (bucket kCountBuckets-1 collects the rest)
__global__ void __launch_bounds__(256) k_ct_hist(const uint32_t *fcnt, int64_t n, const int64_t *pack_key_off, int P,
                                                 const int32_t *pack_dim, int nst, unsigned long long *hist) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = fcnt[g];
        if (!c) continue;
        const int p = pack_of_gkey(pack_key_off, P, (unsigned long long)g);
        atomicAdd(hist + min(c, (uint32_t)kCountBuckets - 1u),
                  (unsigned long long)(4 * __ldg(pack_dim + p) * (1 + nst)));
    }
}

constexpr int kTieBlock = 1024;
__device__ __forceinline__ bool at_cstar(uint32_t c, uint32_t cstar) {
    return min(c, (uint32_t)kCountBuckets - 1u) == cstar;
}

// per block of kTieBlock global keys: the summed cost of the rows tied at c*
__global__ void __launch_bounds__(kTieBlock) k_ct_tiesum(const uint32_t *fcnt, int64_t n, const int64_t *pack_key_off,
                                                         int P, const int32_t *pack_dim, int nst, uint32_t cstar,
                                                         unsigned long long *bsum) {
    __shared__ unsigned long long s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const int64_t g = (int64_t)blockIdx.x * kTieBlock + threadIdx.x;
    if (g < n && at_cstar(fcnt[g], cstar)) {
        const int p = pack_of_gkey(pack_key_off, P, (unsigned long long)g);
        atomicAdd(&s, (unsigned long long)(4 * __ldg(pack_dim + p) * (1 + nst)));
    }
    __syncthreads();
    if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

// exclusive scan of the block sums, one block
__global__ void __launch_bounds__(1024) k_ct_scan(unsigned long long *v, int64_t n) {
    __shared__ unsigned long long carry, ws[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const unsigned long long x0 = i < n ? v[i] : 0ull;
        unsigned long long x = x0;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        if (w == 0) {
            unsigned long long y = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            ws[lane] = y;
        }
        __syncthreads();
        if (i < n) v[i] = carry + (w ? ws[w - 1] : 0ull) + x - x0;
        __syncthreads();
        if (threadIdx.x == 0) carry += ws[31];
        __syncthreads();
    }
}

// the new hot set: every row above c*, and the rows at c* whose cost prefix (ascending global
// key) fits `rem`.  Pass 0 counts the taken rows per block; pass 1 (after a scan of the counts)
// writes them in ascending global key order — the slot order, pack-major.
__global__ void __launch_bounds__(kTieBlock) k_ct_select(const uint32_t *fcnt, int64_t n, const int64_t *pack_key_off,
                                                         int P, const int32_t *pack_dim, int nst, uint32_t cstar,
                                                         unsigned long long rem, const unsigned long long *boff,
                                                         unsigned long long *bcnt, unsigned long long *out,
                                                         int64_t cap, int pass) {
    __shared__ unsigned long long ws[32], wt[32];
    const int64_t g = (int64_t)blockIdx.x * kTieBlock + threadIdx.x;
    const uint32_t c = g < n ? fcnt[g] : 0u;
    const uint32_t cb = min(c, (uint32_t)kCountBuckets - 1u);
    // inclusive prefix of the tie costs inside the block (key order)
    unsigned long long x = 0;
    if (c && cb == cstar) x = (unsigned long long)(4 * __ldg(pack_dim + pack_of_gkey(pack_key_off, P, g)) * (1 + nst));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long y = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        ws[lane] = y;
    }
    __syncthreads();
    const unsigned long long incl = boff[blockIdx.x] + (w ? ws[w - 1] : 0ull) + x;
    const bool take = c && (cb > cstar || (cb == cstar && incl <= rem));
    // rank of this row among the block's taken rows
    const unsigned tm = __ballot_sync(0xffffffffu, take);
    if (lane == 0) wt[w] = __popc(tm);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int k = 0; k < kTieBlock / 32; ++k) {
            const unsigned long long t = wt[k];
            wt[k] = run;
            run += t;
        }
        if (pass == 0) bcnt[blockIdx.x] = run;
    }
    __syncthreads();
    if (pass == 1 && take) {
        const unsigned long long i = bcnt[blockIdx.x] + wt[w] + __popc(tm & ((1u << lane) - 1u));
        if ((int64_t)i < cap) out[i] = (unsigned long long)g;
    }
}

// slots of each pack in the new (sorted) hot set, and the arena layout [w | s1 | s2], pack-major
__global__ void k_ct_layout(const unsigned long long *keys, const unsigned long long *nkeys, const int64_t *pack_key_off,
                            const int32_t *pack_dim, int P, int nst, int32_t *pslot, int64_t *arena_off) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t k = (int64_t)*nkeys;
    for (int p = 0; p <= P; ++p) {  // first slot whose key >= pack_key_off[p]
        const unsigned long long b = p == P ? ~0ull : (unsigned long long)pack_key_off[p];
        int64_t lo = 0, hi = k;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < b) lo = mid + 1; else hi = mid;
        }
        pslot[p] = (int32_t)(p == P ? k : lo);
    }
    int64_t off = 0;
    for (int arr = 0; arr < 3; ++arr)
        for (int p = 0; p < P; ++p) {
            arena_off[arr * P + p] = off;
            if (arr <= nst) off += (int64_t)(pslot[p + 1] - pslot[p]) * pack_dim[p];
        }
}

__device__ __forceinline__ int32_t ct_lookup(const Slot *index, uint32_t mask, unsigned long long key) {
    uint32_t s = slot_hash(key) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
        const unsigned long long k = index[s].key;
        if (k == key) return (int32_t)index[s].minpos;
        if (k == kEmptyKey) return -1;
        s = (s + 1) & mask;
    }
    return -1;
}

// New HStore from the old one (rows staying hot: HBM -> HBM) and from CStore (rows entering:
// host -> HBM); dir 0 instead writes back the old rows that leave (HBM -> host).  One thread per
// 4-float chunk of a slot's row in one of the 1 + nst arrays.
struct CtMerge {
    const unsigned long long *keys;        // the slots walked (new set for dir 1, old set for dir 0)
    int32_t k;
    const Slot *other_index;               // the other set's index (old for dir 1, new for dir 0)
    uint32_t other_mask;
    const int32_t *pslot, *other_pslot;
    const int64_t *aoff, *other_aoff;
    float *arena, *other_arena;
};
__global__ void __launch_bounds__(256) k_ct_merge(CtArgs a, CtMerge m, int nst, int maxD, int dir) {
    const int V4 = maxD / 4;
    const int64_t n = (int64_t)m.k * V4 * (1 + nst);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int arr = (int)(e / ((int64_t)m.k * V4));
        const int64_t r = e - (int64_t)arr * m.k * V4;
        const int32_t slot = (int32_t)(r / V4);
        const int c = (int)(r % V4) * 4;
        const unsigned long long key = m.keys[slot];
        const int p = pack_of_gkey(a.pack_key_off, a.P, key);
        const int D = __ldg(a.pack_dim + p);
        if (c >= D) continue;
        const int32_t os = ct_lookup(m.other_index, m.other_mask, key);
        float *mine = m.arena + m.aoff[arr * a.P + p] + (int64_t)(slot - m.pslot[p]) * D + c;
        const int64_t row = (int64_t)(key - (unsigned long long)__ldg(a.pack_key_off + p));
        float *host = (arr == 0 ? a.w[p] : arr == 1 ? a.s1[p] : a.s2[p]) + row * D + c;
        if (dir == 1) {  // fill the new slot
            const float *src = os >= 0
                ? m.other_arena + m.other_aoff[arr * a.P + p] + (int64_t)(os - m.other_pslot[p]) * D + c
                : host;
            *reinterpret_cast<float4 *>(mine) = *reinterpret_cast<const float4 *>(src);
        } else if (os < 0) {  // an old slot whose row leaves the hot set
            *reinterpret_cast<float4 *>(host) = *reinterpret_cast<const float4 *>(mine);
        }
    }
}

__global__ void k_ct_index(Slot *index, uint32_t mask, const unsigned long long *keys, int32_t k) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        uint32_t s = slot_hash(key) & mask;
        while (atomicCAS(&index[s].key, kEmptyKey, key) != kEmptyKey) s = (s + 1) & mask;
        index[s].minpos = (unsigned int)i;
    }
}

}  // namespace
}  // namespace picasso

using namespace picasso;

#define TCK(x)                                                                  \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_);      \
            return PICASSO_ERR_CUDA;                                            \
        }                                                                       \
    } while (0)

namespace picasso {
int launch_pool_all(picasso_ctx *ctx, PoolArgs pa, float *out, cudaStream_t s, int only_pack);
int launch_segsum_any(picasso_ctx *ctx, int D, const UpdateArgs &u, cudaStream_t s);
UpdateArgs make_update_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, const int32_t *su,
                            const int32_t *sseg);
IndexArgs make_index_args(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N);
void transpose_fork(picasso_ctx *ctx, cudaStream_t s);
void transpose_join(picasso_ctx *ctx, cudaStream_t s);
}  // namespace picasso

static int ct_nst(const picasso_ctx *ctx) { return ctx->opts.opt == PICASSO_OPT_ADAM_LAZY ? 2 : 1; }

static CtArgs ct_args(picasso_ctx *ctx) {
    CtArgs a{};
    a.P = ctx->P;
    a.pack_ustart = ctx->pack_ustart;
    a.unique_gkey = ctx->unique_gkey;
    a.pack_key_off = ctx->pack_key_off_d;
    a.pack_dim = ctx->pack_dim_d;
    a.pack_gbase = ctx->pack_gbase;
    a.gbuf = ctx->gbuf;
    a.index = ctx->ct_index;
    a.mask = ctx->ct_mask;
    a.pslot = ctx->ct_pslot_d;
    a.arena_off = ctx->ct_arena_off_d;
    a.arena = ctx->ct_arena;
    a.hslot = ctx->ct_hslot;
    a.row_off = ctx->ct_row_off;
    a.fcnt = ctx->ct_fcnt;
    a.hits = ctx->ct_hits;
    a.w = ctx->di_w;
    a.s1 = ctx->di_s1;
    a.s2 = ctx->di_s2;
    a.hot_k = ctx->ct_k;
    return a;
}

// forward, world == 1 with the host-DRAM cold tier
picasso_status ct_fwd(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t batch, int64_t n_ids,
                      float *out, cudaStream_t s) {
    IndexArgs a = make_index_args(ctx, ids, offsets, batch, n_ids);
    const uint32_t cap_step =
        (uint32_t)std::min<uint64_t>(ctx->cap, pow2_at_least((uint64_t)std::max<int64_t>(n_ids, 1) * 2));
    a.cap_mask = cap_step - 1;
    ctx->B = batch;
    ctx->N = n_ids;
    ctx->offsets = offsets;
    ctx->overlap = ctx->overlap_env >= 0 ? ctx->overlap_env != 0 : n_ids >= kOverlapMinIds;
    ctx->pool_sms = ctx->num_sms;
    ctx->mark(0, true, s);
    if (!a.region_base) TCK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
    launch_field_prep(a, s);
    launch_dedup_insert(a, s);
    launch_dedup_assign(a, s);
    ctx->mark(0, false, s);
    ctx->launches_fwd = 1 + (n_ids > 0 ? 4 : 0) + 1;
    transpose_fork(ctx, s);  // seg_of on s; the transpose beside the staging + pool when large
    CtArgs c = ct_args(ctx);
    TCK(cudaMemsetAsync(ctx->ct_hits, 0, sizeof(unsigned long long), s));
    ctx->mark(4, true, s);  // phase "owner_gather": probe + staging from host memory
    k_ct_probe<<<(unsigned)ctx->num_sms * 4, 256, 0, s>>>(c);
    k_ct_stage<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(c);
    ctx->mark(4, false, s);
    ctx->launches_fwd += 2;
    ctx->mark(1, true, s);
    PoolArgs pa{};
    pa.ids = ids;
    pa.offsets = offsets;
    pa.B = batch;
    pa.row_off = ctx->ct_row_off;
    pa.inverse = ctx->inverse;
    ctx->launches_fwd += launch_pool_all(ctx, pa, out, s, -1);
    ctx->mark(1, false, s);
    transpose_join(ctx, s);
    TCK(cudaGetLastError());
    ctx->fwd_done = true;
    ctx->last_stream = s;
    return PICASSO_OK;
}

picasso_status ct_bwd(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s) {
    ctx->launches_bwd = 0;
    UpdateArgs u = make_update_args(ctx, grad_out, lr, step, ctx->su, ctx->sseg);
    if (ctx->N > 0) {
        u.gbuf = ctx->gbuf;
        ctx->mark(3, true, s);
        for (int32_t p = 0; p < ctx->P; ++p) {
            u.pack = p;
            u.long_cnt = ctx->long_cnt + p;
            u.pack_key_off = ctx->pack_key_off[p];
            u.weight = ctx->w[p];
            u.state1 = ctx->s1[p];
            u.state2 = ctx->s2[p];
            ctx->launches_bwd += launch_segsum_any(ctx, ctx->pack_dim[p], u, s);
        }
        ctx->mark(3, false, s);
        ctx->mark(5, true, s);
        k_ct_update<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(ct_args(ctx),
                                                              OptParams{u.opt, u.lr, u.eps, u.beta1, u.beta2, u.adam_ss});
        ctx->mark(5, false, s);
        ctx->launches_bwd += 1;
    }
    TCK(cudaGetLastError());
    ctx->fwd_done = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

// Alg. 1: hot_ids = top-k(FCounter) within capacity_bytes; HStore <- CStore(hot_ids).
// Incremental: rows that stay hot move HBM -> HBM into their new slots (double-buffered HStore),
// rows that leave are written back to CStore, rows that enter are loaded from it.
picasso_status ct_refresh(picasso_ctx *ctx, size_t capacity, cudaStream_t s, picasso_cache_stats *stats) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const int nst = ct_nst(ctx);
    int maxD = 4;
    for (int32_t d : ctx->pack_dim) maxD = std::max(maxD, d);
    unsigned long long hits = 0;
    TCK(cudaMemcpyAsync(&hits, ctx->ct_hits, sizeof(hits), cudaMemcpyDeviceToHost, s));
    const int64_t n = ctx->ct_rows_total;
    const int b = ctx->ct_buf ^ 1;  // the new HStore's buffers
    unsigned long long *nkeys = ctx->ct_keys_b[b];
    int64_t knew = 0;
    TCK(cudaMemsetAsync(ctx->ct_nsel, 0, sizeof(unsigned long long), s));
    if (capacity > 0 && n > 0) {
        TCK(cudaMemsetAsync(ctx->ct_hist, 0, sizeof(unsigned long long) * kCountBuckets, s));
        k_ct_hist<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(ctx->ct_fcnt, n, ctx->pack_key_off_d, ctx->P,
                                                             ctx->pack_dim_d, nst, ctx->ct_hist);
        std::vector<unsigned long long> h(kCountBuckets);
        TCK(cudaMemcpyAsync(h.data(), ctx->ct_hist, sizeof(unsigned long long) * kCountBuckets,
                            cudaMemcpyDeviceToHost, s));
        TCK(cudaStreamSynchronize(s));
        // c* = the count where the (count desc) prefix stops fitting; everything above it fits
        unsigned long long above = 0;
        uint32_t cstar = 0;
        for (int c = kCountBuckets - 1; c >= 1; --c) {
            if (above + h[c] > capacity) {
                cstar = (uint32_t)c;
                break;
            }
            above += h[c];
        }
        const unsigned long long rem = capacity - above;  // room for rows tied at c* (cstar 0: no ties)
        const int64_t nb = (n + kTieBlock - 1) / kTieBlock;
        if (cstar > 0) {
            k_ct_tiesum<<<(unsigned)nb, kTieBlock, 0, s>>>(ctx->ct_fcnt, n, ctx->pack_key_off_d, ctx->P,
                                                           ctx->pack_dim_d, nst, cstar, ctx->ct_bsum);
            k_ct_scan<<<1, 1024, 0, s>>>(ctx->ct_bsum, nb);
        } else {
            TCK(cudaMemsetAsync(ctx->ct_bsum, 0, sizeof(unsigned long long) * nb, s));
        }
        k_ct_select<<<(unsigned)nb, kTieBlock, 0, s>>>(ctx->ct_fcnt, n, ctx->pack_key_off_d, ctx->P, ctx->pack_dim_d,
                                                       nst, cstar, rem, ctx->ct_bsum, ctx->ct_bcnt, nullptr, 0, 0);
        TCK(cudaMemsetAsync(ctx->ct_bcnt + nb, 0, sizeof(unsigned long long), s));
        k_ct_scan<<<1, 1024, 0, s>>>(ctx->ct_bcnt, nb + 1);  // [nb] = the number taken
        k_ct_select<<<(unsigned)nb, kTieBlock, 0, s>>>(ctx->ct_fcnt, n, ctx->pack_key_off_d, ctx->P, ctx->pack_dim_d,
                                                       nst, cstar, rem, ctx->ct_bsum, ctx->ct_bcnt, nkeys,
                                                       ctx->ct_kmax, 1);
        unsigned long long ns = 0;
        TCK(cudaMemcpyAsync(&ns, ctx->ct_bcnt + nb, sizeof(ns), cudaMemcpyDeviceToHost, s));
        TCK(cudaStreamSynchronize(s));
        if ((int64_t)ns > ctx->ct_kmax) {
            ctx->last_msg = "hot set larger than the workspace's HStore (cache_max_bytes)";
            return PICASSO_ERR_CAPACITY;
        }
        knew = (int64_t)ns;
        TCK(cudaMemcpyAsync(ctx->ct_nsel, ctx->ct_bcnt + nb, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    }
    const auto t1 = clk::now();
    // the new layout, index and rows
    k_ct_layout<<<1, 32, 0, s>>>(nkeys, ctx->ct_nsel, ctx->pack_key_off_d, ctx->pack_dim_d, ctx->P, nst,
                                 ctx->ct_pslot_b[b], ctx->ct_aoff_b[b]);
    TCK(cudaMemsetAsync(ctx->ct_index_b[b], 0xFF, sizeof(Slot) * ((size_t)ctx->ct_mask + 1), s));
    if (knew > 0)
        k_ct_index<<<(unsigned)ctx->num_sms * 2, 256, 0, s>>>(ctx->ct_index_b[b], ctx->ct_mask, nkeys, (int32_t)knew);
    const int o = ctx->ct_buf;
    CtArgs a = ct_args(ctx);
    if (knew > 0) {  // fill: staying rows from the old HStore, entering rows from CStore
        CtMerge m{nkeys, (int32_t)knew, ctx->ct_index_b[o], ctx->ct_mask, ctx->ct_pslot_b[b], ctx->ct_pslot_b[o],
                  ctx->ct_aoff_b[b], ctx->ct_aoff_b[o], ctx->ct_arena_b[b], ctx->ct_arena_b[o]};
        if (ctx->ct_k == 0) m.other_index = ctx->ct_index_b[o];  // empty (all 0xFF): every row loads
        k_ct_merge<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(a, m, nst, maxD, 1);
    }
    if (ctx->ct_k > 0) {  // write back the old rows that leave
        CtMerge m{ctx->ct_keys_b[o], ctx->ct_k, ctx->ct_index_b[b], ctx->ct_mask, ctx->ct_pslot_b[o], ctx->ct_pslot_b[b],
                  ctx->ct_aoff_b[o], ctx->ct_aoff_b[b], ctx->ct_arena_b[o], ctx->ct_arena_b[b]};
        k_ct_merge<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(a, m, nst, maxD, 0);
    }
    std::vector<int32_t> pslot(ctx->P + 1);
    TCK(cudaMemcpyAsync(pslot.data(), ctx->ct_pslot_b[b], sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost, s));
    TCK(cudaStreamSynchronize(s));
    // swap: the new buffers become the current HStore
    ctx->ct_buf = b;
    ctx->ct_k = (int32_t)knew;
    ctx->ct_pslot = pslot;
    ctx->ct_keys = ctx->ct_keys_b[b];
    ctx->ct_index = ctx->ct_index_b[b];
    ctx->ct_arena = ctx->ct_arena_b[b];
    ctx->ct_pslot_d = ctx->ct_pslot_b[b];
    ctx->ct_arena_off_d = ctx->ct_aoff_b[b];
    if (stats) {
        int64_t bytes = 0;
        for (int p = 0; p < ctx->P; ++p) bytes += (int64_t)(pslot[p + 1] - pslot[p]) * 4 * ctx->pack_dim[p] * (1 + nst);
        int64_t U = 0;
        std::vector<int32_t> us(ctx->P + 1);
        if (cudaMemcpy(us.data(), ctx->pack_ustart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost) ==
            cudaSuccess)
            U = us[ctx->P];
        const auto t2 = clk::now();
        stats->k = ctx->ct_k;
        stats->bytes = bytes;
        stats->hot_uniques = (int64_t)hits;
        stats->uniques = U;
        stats->hit_ratio_unique = U ? (double)hits / (double)U : 0.0;
        stats->refresh_ms = std::chrono::duration<double, std::milli>(t2 - t0).count();
        stats->propose_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();  // top-k selection
        stats->select_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();   // index + row moves
    }
    ctx->last_stream = s;
    return PICASSO_OK;
}

picasso_status ct_hot_keys(picasso_ctx *ctx, int32_t *pack, int64_t *key, int64_t cap, int64_t *n) {
    *n = ctx->ct_k;
    if (ctx->ct_k == 0 || !pack || !key) return PICASSO_OK;
    TCK(cudaStreamSynchronize(ctx->last_stream));
    std::vector<unsigned long long> k(ctx->ct_k);
    TCK(cudaMemcpy(k.data(), ctx->ct_keys, sizeof(unsigned long long) * ctx->ct_k, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < std::min<int64_t>(cap, ctx->ct_k); ++i) {
        const int p = (int)(std::upper_bound(ctx->pack_key_off.begin(), ctx->pack_key_off.begin() + ctx->P,
                                             (int64_t)k[i]) - ctx->pack_key_off.begin()) - 1;
        pack[i] = p;
        key[i] = (int64_t)(k[i] - (unsigned long long)ctx->pack_key_off[p]);
    }
    return PICASSO_OK;
}
