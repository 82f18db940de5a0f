// runtime.cu — the C ABI (include/picasso.h): context, workspace carving, step orchestration.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"

void p2p_release(picasso_ctx *ctx);  // p2p_host.cu
void nvls_release(picasso_ctx *ctx);  // nvls.cu

#define CK(x)                                                             \
    do {                                                                  \
        cudaError_t e_ = (x);                                             \
        if (e_ != cudaSuccess) {                                          \
            if (ctx) ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_); \
            return PICASSO_ERR_CUDA;                                      \
        }                                                                 \
    } while (0)

// The kernels are instantiated for these row widths; any other embedding dim (1..512: CAN's 8~200,
// MMoE's 12~128) is stored zero-padded to the next one — its rows, optimizer state,
// output / dY column block are kernel-dim wide, the padding stays 0 (its gradient is 0).
static int32_t kernel_dim(int32_t d) {
    static const int32_t ks[] = {4, 8, 16, 32, 64, 128, 256, 384, 512};
    for (int32_t k : ks)
        if (d >= 1 && d <= k) return k;
    return 0;
}

extern "C" picasso_status picasso_kernel_dim(int32_t dim, int32_t *kdim) {
    if (!kdim) return PICASSO_ERR_INVALID_ARG;
    *kdim = kernel_dim(dim);
    return *kdim ? PICASSO_OK : PICASSO_ERR_INVALID_ARG;
}

extern "C" picasso_status picasso_nccl_unique_id(uint8_t *out) {
    if (!out) return PICASSO_ERR_INVALID_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return PICASSO_ERR_NCCL;
    std::memcpy(out, &id, 128);
    return PICASSO_OK;
}

extern "C" picasso_status picasso_ctx_create(const picasso_plan_view *plan, int32_t rank, int32_t world,
                                             const uint8_t *nccl_uid, const picasso_ctx_opts *opts,
                                             picasso_ctx **out) {
    if (!plan || !opts || !out || plan->n_fields <= 0 || plan->n_tables <= 0 || plan->n_packs <= 0)
        return PICASSO_ERR_INVALID_ARG;
    if (world < 1 || world > 8 || rank < 0 || rank >= world) return PICASSO_ERR_INVALID_ARG;
    if (opts->max_batch <= 0 || opts->max_ids < 0 || opts->max_ids >= (int64_t)1 << 31) return PICASSO_ERR_INVALID_ARG;
    if (opts->max_recv < 0 || opts->max_recv >= (int64_t)1 << 31) return PICASSO_ERR_INVALID_ARG;
    if (opts->max_step_floats < 0 || opts->max_step_floats / 4 >= (int64_t)1 << 31) return PICASSO_ERR_INVALID_ARG;
    if (opts->max_step_unique < 0 || opts->max_step_unique >= (int64_t)1 << 31 ||
        (opts->max_step_unique > 0 && world != 1))
        return PICASSO_ERR_INVALID_ARG;
    if (opts->cold_tier < 0 || opts->cold_tier > 1 || (opts->cold_tier && world != 1)) return PICASSO_ERR_INVALID_ARG;
    if (opts->cold_tier && opts->max_step_unique > 0) return PICASSO_ERR_INVALID_ARG;  // not combined (yet)
    if (opts->cache_max_bytes < 0) return PICASSO_ERR_INVALID_ARG;
    if (opts->pool < 0 || opts->pool > 1 || opts->id_mode < 0 || opts->id_mode > 1 || opts->opt < 0 || opts->opt > 1 ||
        opts->exchange < 0 || opts->exchange > 1)
        return PICASSO_ERR_INVALID_ARG;
    if ((int64_t)plan->n_fields * opts->max_batch >= ((int64_t)1 << 31)) return PICASSO_ERR_INVALID_ARG;
    if ((int64_t)world * plan->n_packs > kMaxOwnerBlocks) return PICASSO_ERR_INVALID_ARG;
    auto *c = new picasso_ctx();
    if (world > 1) {
        c->mp.max_recv = opts->max_recv > 0 ? opts->max_recv : std::max<int64_t>(2 * opts->max_ids, 1024);
        if (nccl_uid) {
            std::memcpy(c->mp.uid, nccl_uid, 128);
            c->mp.has_uid = true;
        }
    }
    c->rank = rank;
    c->world = world;
    c->opts = *opts;
    c->F = plan->n_fields;
    c->T = plan->n_tables;
    c->P = plan->n_packs;
    c->f2t.assign(plan->field_to_table, plan->field_to_table + c->F);
    c->t2p.assign(plan->table_to_pack, plan->table_to_pack + c->T);
    c->tbase.assign(plan->table_base, plan->table_base + c->T);
    c->trows.assign(plan->table_rows, plan->table_rows + c->T);
    c->tdim.assign(plan->table_dim, plan->table_dim + c->T);
    for (int32_t t = 0; t < c->T; ++t) {  // the kernel (padded) dim: the layout of rows and columns
        const int32_t k = kernel_dim(c->tdim[t]);
        if (!k) {
            delete c;
            return PICASSO_ERR_PLAN_MISMATCH;
        }
        c->tdim[t] = k;
    }
    c->tsalt.assign(c->T, 0);
    if (plan->table_salt) c->tsalt.assign(plan->table_salt, plan->table_salt + c->T);
    c->fcol.assign(plan->field_col, plan->field_col + c->F);
    c->out_width = plan->out_width;
    // K-Interleaving barrier slots: every preset-excluded pack (-1) its own slot, first; then one slot
    // per group, groups contiguous and ascending in pack order
    c->pack_slot.assign(c->P, 0);
    {
        int32_t nex = 0, last = -1;
        bool grouped = false;
        for (int32_t p = 0; p < c->P; ++p) {
            const int32_t g = plan->pack_group ? plan->pack_group[p] : p;
            if (g < 0) {
                if (grouped) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }  // excluded packs come first
                c->pack_slot[p] = nex++;
                continue;
            }
            if (g != last && g != last + 1) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }
            grouped = true;
            last = g;
            c->pack_slot[p] = g;  // + nex below
        }
        for (int32_t p = 0; p < c->P; ++p)
            if (!plan->pack_group || plan->pack_group[p] >= 0) c->pack_slot[p] += nex;
        c->n_slots = c->P ? c->pack_slot[c->P - 1] + 1 : 0;
    }
    // validate plan: tables tile each pack's key range, dims agree, columns fit
    c->pack_dim.assign(c->P, -1);
    c->pack_rows.assign(c->P, 0);
    for (int32_t t = 0; t < c->T; ++t) {
        const int32_t p = c->t2p[t];
        if (p < 0 || p >= c->P || c->trows[t] <= 0) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }
        if (c->pack_dim[p] != -1 && c->pack_dim[p] != c->tdim[t]) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }
        c->pack_dim[p] = c->tdim[t];
        c->pack_rows[p] = std::max(c->pack_rows[p], c->tbase[t] + c->trows[t]);
    }
    for (int32_t p = 0; p < c->P; ++p)
        if (c->pack_dim[p] < 0) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }
    if (c->out_width % 4) { delete c; return PICASSO_ERR_PLAN_MISMATCH; }
    for (int32_t f = 0; f < c->F; ++f) {
        const int32_t t = c->f2t[f];
        if (t < 0 || t >= c->T || c->fcol[f] % 4 || c->fcol[f] < 0 || c->fcol[f] + c->tdim[t] > c->out_width) {
            delete c;
            return PICASSO_ERR_PLAN_MISMATCH;
        }
    }
    c->pack_key_off.assign(c->P + 1, 0);
    for (int32_t p = 0; p < c->P; ++p) c->pack_key_off[p + 1] = c->pack_key_off[p] + c->pack_rows[p];
    // pack-major field order (pack asc, field asc)
    c->pack_first_k.assign(c->P + 1, 0);
    for (int32_t p = 0; p < c->P; ++p) {
        c->pack_first_k[p] = (int32_t)c->pm_fields.size();
        for (int32_t f = 0; f < c->F; ++f)
            if (c->t2p[c->f2t[f]] == p) c->pm_fields.push_back(f);
    }
    c->pack_first_k[c->P] = c->F;
    // dedup table: per-table regions (<= 4 x max_ids + 64 per table) for the rank-local dedup, and a
    // pow2 >= 2 x max_recv global table for the NCCL owner dedup, in the same slots
    // per-table regions only when one global table would not stay in L2 (2 x max_ids x 16 B > ~64 MB):
    // below that the global table (load factor <= 1/4 here) has the shorter probe chains
    c->use_regions = opts->max_ids > ((int64_t)1 << 21);
    if (const char *e = std::getenv("PICASSO_DEDUP_REGIONS")) c->use_regions = std::atoi(e) != 0;
    c->region_shift = 1;
    uint64_t cap64 = pow2_at_least((uint64_t)std::max<int64_t>(std::max<int64_t>(opts->max_ids, c->mp.max_recv), 1) * 2);
    if (c->use_regions)
        cap64 = std::max<uint64_t>(cap64, ((uint64_t)opts->max_ids << (c->region_shift + 1)) + 64 * (uint64_t)c->T);
    // hash slots are int32 (slot_of, the device-side region bases): a table that would need more
    // than 2^31 - 1 slots (max_ids above ~2^28 with per-table regions) is refused up front
    if (cap64 > (uint64_t)INT32_MAX) {
        delete c;
        return PICASSO_ERR_CAPACITY;
    }
    c->cap = (uint32_t)cap64;
    if (world > 1) {  // local rows must fit int32 (received keys are int32 local rows)
        for (int32_t p = 0; p < c->P; ++p)
            if (c->pack_rows[p] / world >= ((int64_t)1 << 31)) {
                delete c;
                return PICASSO_ERR_PLAN_MISMATCH;
            }
        c->mp.row_base.assign(c->P + 1, 0);  // owned rows per pack, prefix (owner-row tables)
        for (int32_t p = 0; p < c->P; ++p) {
            const int64_t R = c->pack_rows[p];
            c->mp.row_base[p + 1] = c->mp.row_base[p] + (R > rank ? (R - rank + world - 1) / world : 0);
        }
        c->mp.rows_total = c->mp.row_base[c->P];
        if (opts->cache_max_bytes > 0) {  // HybridHash sizing: FCounter over owned rows, hot rows
            c->mp.fcnt_off = c->mp.row_base;
            int minD = 1 << 30;
            for (int32_t p = 0; p < c->P; ++p) minD = std::min(minD, c->pack_dim[p]);
            const int nst = opts->opt == PICASSO_OPT_ADAM_LAZY ? 2 : 1;
            c->mp.k_max = opts->cache_max_bytes / ((int64_t)4 * minD * (1 + nst));
            c->mp.hot_mask = (uint32_t)(pow2_at_least((uint64_t)std::max<int64_t>(c->mp.k_max, 1) * 2) - 1);
        }
    }
    if (const char *e = std::getenv("PICASSO_BWD")) c->fuse_pipe = std::strcmp(e, "split") != 0;
    if (const char *e = std::getenv("PICASSO_SEGSUM")) c->bulk_segsum = std::strcmp(e, "legacy") != 0;
    if (const char *e = std::getenv("PICASSO_SEGSUM_SMALL")) c->flat_small = std::strcmp(e, "legacy") != 0;
    c->seg_cfg = segsum_pipe_cfg();
    if (const char *e = std::getenv("PICASSO_POOL")) {
        c->pipe_pool = std::strcmp(e, "legacy") != 0;
        if (!std::strcmp(e, "flat")) c->pool_kind = 2;
        if (!std::strcmp(e, "pipe")) c->pool_kind = 1;
    }
    if (const char *e = std::getenv("PICASSO_OVERLAP")) c->overlap_env = std::strcmp(e, "0") != 0;
    if (c->overlap_env >= 0) c->overlap = c->overlap_env;
    if (const char *e = std::getenv("PICASSO_KINTERLEAVE")) c->kinterleave = std::atoi(e);
    // World == 1: the pool needs only the raw IDs (row = h(id)), so by default it starts at once
    // and streams rows on the caller's stream while the Unique chain and the backward's transpose
    // run beside it on the internal stream (C2: 0.291 -> 0.258 ms / step, round-2 measurement;
    // the pool alone then runs slower, sharing the SMs).  The pool leaves 74 of 148 SMs to that
    // chain (measured best at C2; PICASSO_POOL_RESERVE overrides).
    // PICASSO_EARLY_POOL=0: the serial order (dedup, then pool).
    // Chosen per forward (below kOverlapMinIds IDs; at C3's 83.5 M IDs the early pool measured
    // slower, 26.3 vs 25.6 ms, and the transpose alone goes beside the pool instead).
    if (const char *e = std::getenv("PICASSO_EARLY_POOL")) c->early_env = std::strcmp(e, "0") != 0;
    c->pool_reserve = 74;  // C2 sweep (round 2): 24 -> 0.283, 48 -> 0.270, 74 -> 0.258, 84 -> 0.267 ms / step
    if (const char *e = std::getenv("PICASSO_POOL_RESERVE")) c->pool_reserve = std::atoi(e);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    // fused segment-sum + optimizer (k_segsum_upd): world == 1, every tiled (D >= 64) pack of dim 64
    // or 128 — the tiles are then cut for its warps per CTA
    if (c->fuse_pipe) {
        bool ok = world == 1;
        for (int32_t d : c->pack_dim)
            if (d >= 64 && d != 64 && d != 128) ok = false;
        c->fuse_pipe = ok;
    }
    c->seg_nt = c->num_sms * (c->fuse_pipe ? segsum_upd_warps(opts->opt) : segsum_pipe_warps(c->seg_cfg));
    if (const char *e = std::getenv("PICASSO_FUSE_RW")) c->fuse_rw = std::max(1, std::atoi(e));
    // sort-based index: the backward must be the tiled one (the sort emits its tiles)
    c->sort_idx = world == 1 && !opts->cold_tier && c->bulk_segsum && c->pack_key_off[c->P] <= ((int64_t)1 << 32) &&
                  sortidx_scratch_ints(std::max<int64_t>(opts->max_ids, 1), c->P) <=
                      radix_hist2_ints(std::max<int64_t>(opts->max_ids, 1));
    c->sort_key_bits = c->pack_key_off[c->P] > 1 ? 64 - __builtin_clzll((unsigned long long)(c->pack_key_off[c->P] - 1)) : 1;
    if (const char *e = std::getenv("PICASSO_INDEX")) {
        if (!std::strcmp(e, "hash")) c->sort_idx = false;
        if (!std::strcmp(e, "sort")) c->sort_min_ids = 0;
    }
    if (const char *e = std::getenv("PICASSO_SORT_MIN_IDS")) c->sort_min_ids = std::atoll(e);
    if (const char *e = std::getenv("PICASSO_SORT_OVERLAP")) c->sort_overlap = std::strcmp(e, "0") != 0;
    if (const char *e = std::getenv("PICASSO_SORT_RESERVE")) c->sort_reserve = std::atoi(e);
    c->sort_w = world > 1 && !opts->cold_tier && c->bulk_segsum && c->pack_key_off[c->P] <= ((int64_t)1 << 32) &&
                sortidx_scratch_ints(std::max<int64_t>(opts->max_ids, 1), c->P) <=
                    radix_hist2_ints(std::max<int64_t>(opts->max_ids, 1));
    if (const char *e = std::getenv("PICASSO_INDEX"))
        if (!std::strcmp(e, "hash")) c->sort_w = false;
    if (const char *e = std::getenv("PICASSO_SORT_MIN_IDS_W")) c->sort_min_ids_w = std::atoll(e);
    // dY regrouped per pack before the world == 1 backward (several packs, disjoint columns)
    c->dy_stage = world == 1 && c->P > 1 && !opts->cold_tier;
    if (const char *e = std::getenv("PICASSO_DY_STAGE")) c->dy_stage = c->dy_stage && std::strcmp(e, "0") != 0;
    if (c->dy_stage) {
        std::vector<int32_t> owner(c->out_width / 4, -1);
        for (int32_t f = 0; f < c->F && c->dy_stage; ++f)
            for (int64_t q = c->fcol[f] / 4; q < (c->fcol[f] + c->tdim[c->f2t[f]]) / 4; ++q) {
                if (owner[q] >= 0) c->dy_stage = false;  // overlapping columns: read dY in place
                owner[q] = f;
            }
        c->dyp_off.assign(c->P + 1, 0);
        for (int32_t p = 0; p < c->P; ++p)
            c->dyp_off[p + 1] = c->dyp_off[p] + (int64_t)opts->max_batch * (c->pack_first_k[p + 1] - c->pack_first_k[p]) *
                                                     c->pack_dim[p];
    }
    c->pool_sms = c->num_sms;
    c->ws_bytes = c->carve(nullptr);
    *out = c;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_workspace_size(const picasso_ctx *ctx, size_t *bytes) {
    if (!ctx || !bytes) return PICASSO_ERR_INVALID_ARG;
    *bytes = ctx->ws_bytes;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_pack_local_rows(const picasso_ctx *ctx, int32_t pack, int64_t *rows) {
    if (!ctx || !rows || pack < 0 || pack >= ctx->P) return PICASSO_ERR_INVALID_ARG;
    const int64_t R = ctx->pack_rows[pack];
    *rows = R > ctx->rank ? (R - ctx->rank + ctx->world - 1) / ctx->world : 0;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_bind(picasso_ctx *ctx, void *workspace, size_t bytes, float *const *pack_weight,
                                       float *const *pack_state1, float *const *pack_state2) {
    if (!ctx || !workspace || !pack_weight || !pack_state1) return PICASSO_ERR_INVALID_ARG;
    if (bytes < ctx->ws_bytes) return PICASSO_ERR_CAPACITY;
    if (ctx->opts.opt == PICASSO_OPT_ADAM_LAZY && !pack_state2) return PICASSO_ERR_INVALID_ARG;
    char *base = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(workspace) + kAlign - 1) / kAlign * kAlign);
    if ((size_t)(base - reinterpret_cast<char *>(workspace)) + ctx->ws_bytes - kAlign > bytes) return PICASSO_ERR_CAPACITY;
    ctx->carve(base);
    ctx->w.assign(pack_weight, pack_weight + ctx->P);
    ctx->s1.assign(pack_state1, pack_state1 + ctx->P);
    ctx->s2.assign(ctx->P, nullptr);
    if (pack_state2) ctx->s2.assign(pack_state2, pack_state2 + ctx->P);
    for (int32_t p = 0; p < ctx->P; ++p) {
        if (!ctx->w[p] || !ctx->s1[p] || (ctx->opts.opt == PICASSO_OPT_ADAM_LAZY && !ctx->s2[p]))
            return PICASSO_ERR_INVALID_ARG;
        if ((reinterpret_cast<uintptr_t>(ctx->w[p]) | reinterpret_cast<uintptr_t>(ctx->s1[p])) & 15)
            return PICASSO_ERR_INVALID_ARG;
    }
    std::vector<FieldInfo> fi(ctx->F);
    for (int32_t f = 0; f < ctx->F; ++f) {
        const int32_t t = ctx->f2t[f];
        fi[f].base = ctx->tbase[t];
        fi[f].rows = ctx->trows[t];
        fi[f].salt = ctx->tsalt[t];
        fi[f].col = ctx->fcol[f];
        fi[f].pack = ctx->t2p[t];
        fi[f].dim = ctx->tdim[t];
        fi[f].table = t;
        fi[f].pad = 0;
    }
    CK(cudaMemcpy(ctx->finfo, fi.data(), sizeof(FieldInfo) * ctx->F, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->pm_fields_d, ctx->pm_fields.data(), sizeof(int32_t) * ctx->F, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->pack_first_k_d, ctx->pack_first_k.data(), sizeof(int32_t) * (ctx->P + 1), cudaMemcpyHostToDevice));
    {
        std::vector<int32_t> fk(ctx->F);
        for (int32_t p = 0; p < ctx->P; ++p)
            for (int32_t k = ctx->pack_first_k[p]; k < ctx->pack_first_k[p + 1]; ++k)
                fk[ctx->pm_fields[k]] = k - ctx->pack_first_k[p];
        CK(cudaMemcpy(ctx->field_k_d, fk.data(), sizeof(int32_t) * ctx->F, cudaMemcpyHostToDevice));
        if (ctx->dy_stage) {  // k_dy_pack's maps: chunk -> field, field -> its block in its pack's rows
            std::vector<int32_t> c4f(ctx->out_width / 4 + 1, -1), stride(ctx->F), col(ctx->F);
            std::vector<int64_t> base(ctx->F);
            for (int32_t f = 0; f < ctx->F; ++f) {
                const int32_t t = ctx->f2t[f], p = ctx->t2p[t], D = ctx->pack_dim[p];
                for (int64_t q = ctx->fcol[f] / 4; q < (ctx->fcol[f] + ctx->tdim[t]) / 4; ++q) c4f[q] = f;
                stride[f] = (ctx->pack_first_k[p + 1] - ctx->pack_first_k[p]) * D;
                col[f] = fk[f] * D;
                base[f] = ctx->dyp_off[p] + col[f];
            }
            CK(cudaMemcpy(ctx->col4_field_d, c4f.data(), sizeof(int32_t) * c4f.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(ctx->dyp_base_d, base.data(), sizeof(int64_t) * ctx->F, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(ctx->dyp_stride_d, stride.data(), sizeof(int32_t) * ctx->F, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(ctx->dyp_col_d, col.data(), sizeof(int32_t) * ctx->F, cudaMemcpyHostToDevice));
        }
    }
    CK(cudaMemcpy(ctx->pack_key_off_d, ctx->pack_key_off.data(), sizeof(int64_t) * (ctx->P + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->pack_dim_d, ctx->pack_dim.data(), sizeof(int32_t) * ctx->P, cudaMemcpyHostToDevice));
    CK(cudaMemset(ctx->err, 0, sizeof(int)));
    if (ctx->ct_fcnt) {  // cold tier: FCounter zero, HStore empty
        CK(cudaMemset(ctx->ct_fcnt, 0, sizeof(uint32_t) * std::max<int64_t>(ctx->ct_rows_total, 1)));
        for (int b = 0; b < 2; ++b) {
            CK(cudaMemset(ctx->ct_index_b[b], 0xFF, sizeof(Slot) * ((size_t)ctx->ct_mask + 1)));
            CK(cudaMemset(ctx->ct_pslot_b[b], 0, sizeof(int32_t) * (ctx->P + 1)));
            CK(cudaMemset(ctx->ct_aoff_b[b], 0, sizeof(int64_t) * 3 * ctx->P));
        }
        ctx->ct_k = 0;
        ctx->ct_pslot.assign(ctx->P + 1, 0);
    }
    if (ctx->di_w) {  // D-Interleaving / cold tier: kernels reach every pack's rows
        CK(cudaMemcpy(ctx->di_w, ctx->w.data(), sizeof(float *) * ctx->P, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->di_s1, ctx->s1.data(), sizeof(float *) * ctx->P, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->di_s2, ctx->s2.data(), sizeof(float *) * ctx->P, cudaMemcpyHostToDevice));
    }
    if (ctx->world > 1 && !ctx->mp.cnt_send_h) {
        const int WP = ctx->world * ctx->P;
        CK(cudaMallocHost(&ctx->mp.cnt_send_h, sizeof(int32_t) * (WP + 1)));
        CK(cudaMallocHost(&ctx->mp.cnt_recv_h, sizeof(int32_t) * WP));
        CK(cudaMallocHost(&ctx->mp.oblk_h, sizeof(OwnerBlock) * WP));
        CK(cudaMallocHost(&ctx->mp.ostart_h, sizeof(int64_t) * (ctx->P + 1)));
        CK(cudaMallocHost(&ctx->mp.og_h, sizeof(int32_t) * (ctx->P + 1)));
    }
    if (ctx->world > 1)
        CK(cudaMemcpy(ctx->mp.row_base_d, ctx->mp.row_base.data(), sizeof(int64_t) * (ctx->P + 1),
                      cudaMemcpyHostToDevice));
    if (ctx->world > 1 && ctx->opts.cache_max_bytes > 0) {  // HybridHash: FCounter, empty hot set
        MultiState &mp = ctx->mp;
        CK(cudaMemcpy(mp.fcnt_off_d, mp.fcnt_off.data(), sizeof(int64_t) * (ctx->P + 1), cudaMemcpyHostToDevice));
        CK(cudaMemset(mp.fcnt, 0, sizeof(uint32_t) * std::max<int64_t>(mp.rows_total, 1)));
        CK(cudaMemset(mp.hot_cnt, 0, sizeof(uint32_t) * std::max<int64_t>(mp.k_max, 1)));
        CK(cudaMemset(mp.hot_index, 0xFF, sizeof(Slot) * ((size_t)mp.hot_mask + 1)));
        CK(cudaMemset(mp.hot_pslot_d, 0, sizeof(int32_t) * (ctx->P + 1)));
        CK(cudaMemset(mp.hot_off_d, 0, sizeof(int64_t) * 4 * ctx->P));
        mp.hot_k = 0;
    }
    if (ctx->world > 1 && ctx->mp.has_uid && !ctx->mp.comm) {  // one rank per process: NCCL
        ncclUniqueId id;
        std::memcpy(&id, ctx->mp.uid, 128);
        if (ncclCommInitRank(&ctx->mp.comm, ctx->world, id, ctx->rank) != ncclSuccess) {
            ctx->last_msg = "ncclCommInitRank failed";
            return PICASSO_ERR_NCCL;
        }
        if (ctx->opts.cache_max_bytes > 0) {  // set up the AllReduce path now, not in the first hot step
            if (ncclAllReduce(ctx->mp.hot_touch, ctx->mp.hot_touch, 1, ncclFloat32, ncclSum, ctx->mp.comm, 0) !=
                ncclSuccess)
                return PICASSO_ERR_NCCL;
            CK(cudaStreamSynchronize(0));
        }
    }
    if (!ctx->side) {  // internal streams: the forward's overlapped transpose, K-Interleaving
        // the internal stream carries the latency-bound Unique / transpose chain beside the pool:
        // highest priority, so its blocks are scheduled first whenever SMs free up
        int lo_prio = 0, hi_prio = 0;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        static const char *pe = std::getenv("PICASSO_SIDE_PRIO");
        if (pe && std::atoi(pe) == 0)
            CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        else
            CK(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi_prio));
        CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_fp, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_seg, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_fork2, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join2, cudaEventDisableTiming));
    }
    ctx->bound = true;
    ctx->fwd_done = false;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_ctx_destroy(picasso_ctx *ctx) {
    if (!ctx) return PICASSO_OK;
    if (ctx->mp.nvls_mc) nvls_release(ctx);
    p2p_release(ctx);
    if (ctx->side) {
        cudaStreamDestroy(ctx->side);
        cudaEventDestroy(ctx->ev_fork);
        cudaEventDestroy(ctx->ev_join);
        cudaEventDestroy(ctx->ev_fp);
        cudaEventDestroy(ctx->ev_seg);
        cudaStreamDestroy(ctx->side2);
        cudaEventDestroy(ctx->ev_fork2);
        cudaEventDestroy(ctx->ev_join2);
    }
    if (ctx->mp.comm) ncclCommDestroy(ctx->mp.comm);
    if (ctx->mp.cnt_send_h) {
        cudaFreeHost(ctx->mp.cnt_send_h);
        cudaFreeHost(ctx->mp.cnt_recv_h);
        cudaFreeHost(ctx->mp.oblk_h);
        cudaFreeHost(ctx->mp.ostart_h);
        cudaFreeHost(ctx->mp.og_h);
    }
    delete ctx;
    return PICASSO_OK;
}

namespace picasso {
IndexArgs make_index_args(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N);
UpdateArgs make_update_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, const int32_t *su,
                            const int32_t *sseg);
int launch_segsum_any(picasso_ctx *ctx, int D, const UpdateArgs &u, cudaStream_t s);  // returns #launches
void launch_csr_any(picasso_ctx *ctx, const int32_t *su, int64_t N, cudaStream_t s);
int launch_pool_all(picasso_ctx *ctx, PoolArgs pa, float *out, cudaStream_t s, int only_pack = -1);  // #launches
void transpose_fork(picasso_ctx *ctx, cudaStream_t s);
void transpose_on(picasso_ctx *ctx, cudaStream_t t);
void transpose_join(picasso_ctx *ctx, cudaStream_t s);
}
picasso_status multi_fwd_nccl(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                              float *out, cudaStream_t s);
picasso_status multi_bwd_nccl(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s);
picasso_status multi_fwd_p2p(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                             float *out, cudaStream_t s);
picasso_status multi_bwd_p2p(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s);
picasso_status ct_fwd(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t batch, int64_t n_ids,
                      float *out, cudaStream_t s);  // coldtier.cu
picasso_status ct_bwd(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s);

static IndexArgs index_args(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N) {
    return picasso::make_index_args(ctx, ids, offsets, B, N);
}

IndexArgs picasso::make_index_args(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N) {
    IndexArgs a{};
    a.ids = ids;
    a.offsets = offsets;
    a.B = B;
    a.N = N;
    a.F = ctx->F;
    a.P = ctx->P;
    a.id_mode = ctx->opts.id_mode;
    a.finfo = ctx->finfo;
    a.pm_fields = ctx->pm_fields_d;
    a.pack_first_k = ctx->pack_first_k_d;
    a.pack_key_off = ctx->pack_key_off_d;
    a.id_start = ctx->id_start;
    a.gstart_pm = ctx->gstart_pm;
    a.field_gstart = ctx->field_gstart;
    a.pack_gstart = ctx->pack_gstart;
    a.table = ctx->table;
    a.slot_of = ctx->slot_of;
    a.fmask = ctx->fmask;
    a.T = ctx->T;
    a.region_base = ctx->use_regions ? ctx->region_base : nullptr;
    a.region_mask = ctx->region_mask;
    a.region_shift = ctx->region_shift;
    a.empty_pack = ctx->empty_pack;
    a.seg_limit = ctx->seg_limit;
    a.tocc = ctx->tocc;
    a.seg_of = ctx->seg_of;
    a.inverse = ctx->inverse;
    a.blk_cnt = ctx->blk_cnt;
    a.blk_off = ctx->blk_off;
    a.d_total = ctx->d_total;
    a.unique_gkey = ctx->unique_gkey;
    a.pack_ustart = ctx->pack_ustart;
    a.pack_dim = ctx->pack_dim_d;
    a.pack_gbase = ctx->pack_gbase;
    ctx->splan = make_sort_plan(std::max<int64_t>(N, 1));
    a.sort_bits0 = ctx->splan.bits[0];
    a.sort_hist0 = ctx->hist0;
    a.err = ctx->err;
    return a;
}

static SortIdxArgs sort_idx_args(picasso_ctx *ctx, const int64_t *ids, int32_t B, int64_t N) {
    SortIdxArgs x{};
    x.ids = ids;
    x.seg_of = ctx->seg_of;
    x.B = B;
    x.N = N;
    x.id_mode = ctx->opts.id_mode;
    x.finfo = ctx->finfo;
    x.id_start = ctx->id_start;
    x.field_gstart = ctx->field_gstart;
    x.pack_key_off = ctx->pack_key_off_d;
    x.err = ctx->err;
    x.keys = reinterpret_cast<uint32_t *>(ctx->slot_of);
    x.hist = ctx->hist0;
    x.rowtot = ctx->rowtot;
    const int64_t nb1 = (N + kTile - 1) / kTile + 1;  // scratch (hist1): tile arrays, views, word ranks
    x.tile_heads = ctx->blk_cnt;
    x.run_base = ctx->blk_off;
    x.tile_last = ctx->hist1;
    x.carry = ctx->hist1 + nb1;
    x.pack_hb = ctx->hist1 + 2 * nb1;
    x.view_scratch = x.pack_hb + ctx->P + 1;
    x.wpref = x.view_scratch + 2 * nb1;
    x.bm = reinterpret_cast<uint32_t *>(ctx->fmask);
    x.d_total = ctx->d_total;
    x.inverse = ctx->inverse;
    x.ustart = ctx->ustart;
    x.run_key = ctx->run_keys();
    x.unique_gkey = ctx->unique_gkey;
    x.P = ctx->P;
    x.pack_gstart = ctx->pack_gstart;
    x.pack_ustart = ctx->pack_ustart;
    x.pack_gbase = ctx->pack_gbase;
    x.pack_dim = ctx->pack_dim_d;
    x.nt = ctx->seg_nt;
    x.rw = ctx->fuse_pipe ? ctx->fuse_rw : 1;
    x.tile_start = ctx->tile_start;
    x.long_cnt = ctx->long_cnt;
    return x;
}

// Row-sharded step (world > 1) indexed by sort: field layout, segment map + keys, the sort (the
// backward's run-order rows and tiles), and at once the reading-O1 views the exchange works in
// (Unique in first-occurrence order, inverse, per-pack uid ranges) plus run -> uid.  multi_host.cu.
picasso_status w_sorted_index(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                              cudaStream_t s) {
    IndexArgs a = index_args(ctx, ids, offsets, B, N);
    a.region_base = nullptr;
    a.keys = reinterpret_cast<uint32_t *>(ctx->slot_of);
    launch_field_prep(a, s);
    const SegKeyArgs ka{ids, ctx->pack_key_off_d, ctx->opts.id_mode, a.keys};
    launch_seg_of(offsets, B, ctx->F, ctx->field_gstart, ctx->id_start, ctx->seg_of, s, ctx->finfo, ctx->empty_pack,
                  ctx->seg_limit, ctx->err, &ka);
    SortIdxArgs x = sort_idx_args(ctx, ids, B, N);
    x.run_uid = ctx->run_uid;
    ctx->w_runx = ctx->mp.p2p && std::getenv("PICASSO_W_UIDORDER") == nullptr;  // (measurement aid)
    if (ctx->w_runx) x.inv_run = ctx->inverse;
    const SortIdxPlan plan = make_sortidx_plan(N, ctx->sort_key_bits, ctx->num_sms);
    uint64_t *sorted = nullptr, *other = nullptr;
    ctx->launches_fwd += 2 + launch_sort_index(x, plan, reinterpret_cast<uint64_t *>(ctx->k_a),
                                               reinterpret_cast<uint64_t *>(ctx->k_b), &sorted, &other, s);
    ctx->views_ready = false;
    if (!ctx->w_runx) {
        ctx->launches_fwd += launch_sort_views(x, sorted, s);
        ctx->views_ready = true;
    }
    ctx->su = reinterpret_cast<int32_t *>(other);
    ctx->sseg = ctx->su + N;
    ctx->sorted_items = sorted;
    CK(cudaGetLastError());
    return PICASSO_OK;
}

// the reading-O1 views of a sorted step (Unique in first-occurrence order, inverse), on request
static picasso_status ensure_views(picasso_ctx *ctx) {
    const bool sorted = ctx->world > 1 ? ctx->w_runorder : ctx->sort_step;
    if (!sorted || ctx->views_ready) return PICASSO_OK;
    const SortIdxArgs x = sort_idx_args(ctx, nullptr, ctx->B, ctx->N);
    launch_sort_views(x, ctx->sorted_items, ctx->last_stream);
    CK(cudaGetLastError());
    ctx->views_ready = true;
    return PICASSO_OK;
}

// World == 1, sort-based index (k_sortidx.cu): field layout + segment of every position, then the
// sort chain on the internal stream beside the pool (which needs only the IDs and seg_of); the
// forward joins both.  The chain emits Unique / inverse (reading O1) and the backward's CSR + tiles.
static picasso_status fwd_sorted(picasso_ctx *ctx, IndexArgs a, float *out, cudaStream_t s) {
    const int64_t N = a.N;
    ctx->B = a.B;
    ctx->N = N;
    ctx->offsets = a.offsets;
    a.region_base = nullptr;  // no dedup table
    a.keys = reinterpret_cast<uint32_t *>(ctx->slot_of);
    launch_field_prep(a, s);
    const SegKeyArgs ka{a.ids, ctx->pack_key_off_d, ctx->opts.id_mode, a.keys};
    launch_seg_of(a.offsets, a.B, ctx->F, ctx->field_gstart, ctx->id_start, ctx->seg_of, s, ctx->finfo,
                  ctx->empty_pack, ctx->seg_limit, ctx->err, &ka);
    ctx->launches_fwd += 2;
    cudaStream_t t = s;
    if (ctx->sort_overlap && ctx->side) {
        CK(cudaEventRecord(ctx->ev_fork, s));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        t = ctx->side;
    }
    SortIdxArgs x = sort_idx_args(ctx, a.ids, a.B, N);
    const SortIdxPlan plan = make_sortidx_plan(N, ctx->sort_key_bits, ctx->num_sms);
    uint64_t *sorted = nullptr, *other = nullptr;
    ctx->mark(0, true, t);
    ctx->launches_fwd += launch_sort_index(x, plan, reinterpret_cast<uint64_t *>(ctx->k_a),
                                           reinterpret_cast<uint64_t *>(ctx->k_b), &sorted, &other, t);
    ctx->mark(0, false, t);
    ctx->su = reinterpret_cast<int32_t *>(other);
    ctx->sseg = ctx->su + N;
    ctx->sorted_items = sorted;
    ctx->views_ready = false;
    if (t != s) CK(cudaEventRecord(ctx->ev_join, t));
    // the pool leaves sort_reserve SMs to the sort chain running beside it (C2 sweep)
    ctx->pool_sms = t != s ? std::max(ctx->num_sms / 4, ctx->num_sms - ctx->sort_reserve) : ctx->num_sms;
    ctx->mark(1, true, s);
    {
        PoolArgs pa{};
        pa.ids = a.ids;
        pa.offsets = a.offsets;
        pa.B = a.B;
        ctx->launches_fwd += launch_pool_all(ctx, pa, out, s);
    }
    ctx->mark(1, false, s);
    if (t != s) CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    CK(cudaGetLastError());
    ctx->fwd_done = true;
    ctx->last_stream = s;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_packed_lookup_fwd(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets,
                                                    int32_t batch, int64_t n_ids, float *out, void *stream) {
    NvtxRange nvtx("picasso_fwd");
    if (!ctx || !offsets || (!out && batch > 0) || batch < 0 || n_ids < 0 || (n_ids > 0 && !ids))
        return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound) return PICASSO_ERR_STATE;
    if (batch > ctx->opts.max_batch || n_ids > ctx->opts.max_ids) return PICASSO_ERR_CAPACITY;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ctx->launches_fwd = 0;
    if (ctx->world > 1) {
        // loopback groups step through picasso_group_fwd; the NCCL exchange and the HybridHash
        // AllReduce need the communicator; the peer-memory exchange alone needs only the windows
        if (ctx->mp.group) return PICASSO_ERR_STATE;
        if (!ctx->mp.comm && (!ctx->mp.p2p || ctx->opts.cache_max_bytes > 0)) return PICASSO_ERR_STATE;
        if (ctx->opts.exchange == 0 && !ctx->mp.p2p) {
            ctx->last_msg = "peer-memory exchange: picasso_p2p_handle / picasso_p2p_open not done";
            return PICASSO_ERR_STATE;
        }
        return ctx->mp.p2p ? multi_fwd_p2p(ctx, ids, offsets, batch, n_ids, out, s)
                           : multi_fwd_nccl(ctx, ids, offsets, batch, n_ids, out, s);
    }
    if (ctx->opts.cold_tier) return ct_fwd(ctx, ids, offsets, batch, n_ids, out, s);
    IndexArgs a = index_args(ctx, ids, offsets, batch, n_ids);
    ctx->sort_step = ctx->sort_idx && batch > 0 && n_ids >= ctx->sort_min_ids;
    if (ctx->sort_step) return fwd_sorted(ctx, a, out, s);
    const uint32_t cap_step =
        (uint32_t)std::min<uint64_t>(ctx->cap, pow2_at_least((uint64_t)std::max<int64_t>(n_ids, 1) * 2));
    a.cap_mask = cap_step - 1;
    ctx->B = batch;
    ctx->N = n_ids;
    ctx->offsets = offsets;
    // world == 1: the transpose beside the pool pays only for large batches.  Below kOverlapMinIds
    // the persistent pool (one CTA per SM, static tiles) waits for SMs the transpose's blocks
    // hold, and the serial order is faster (C2: 0.283 vs 0.294 ms; C3, 83.5 M IDs: 26.2 vs
    // 26.6 ms the other way round).  PICASSO_OVERLAP=0/1 forces either; the early pool needs it.
    ctx->early_pool = ctx->early_env >= 0 ? ctx->early_env != 0 : n_ids < kOverlapMinIds;
    if (ctx->overlap_env < 0) ctx->overlap = ctx->early_pool || n_ids >= kOverlapMinIds;
    ctx->pool_sms = (ctx->early_pool && ctx->overlap && ctx->side)
                        ? std::max(ctx->num_sms / 4, ctx->num_sms - ctx->pool_reserve)
                        : ctx->num_sms;
    if (ctx->overlap && ctx->side && ctx->early_pool) {
        // At world == 1 the pool needs only the raw IDs (row = h(id)), not the dedup: the index
        // work (Unique, inverse) and the backward's transpose run on the internal stream while
        // the pool streams rows on the caller's stream; the forward joins both before returning.
        if (!a.region_base) CK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
        launch_field_prep(a, s);
        launch_seg_of(offsets, batch, ctx->F, ctx->field_gstart, ctx->id_start, ctx->seg_of, s, ctx->finfo,
                      ctx->empty_pack, ctx->seg_limit, ctx->err);
        CK(cudaEventRecord(ctx->ev_fork, s));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        cudaStream_t t = ctx->side;
        ctx->mark(0, true, t);
        launch_dedup_insert(a, t);
        launch_dedup_assign(a, t);
        ctx->mark(0, false, t);
        picasso::transpose_on(ctx, t);
        CK(cudaEventRecord(ctx->ev_join, t));
        ctx->launches_fwd += 2 + (n_ids > 0 ? 4 : 0) + 1;  // prep, seg_of, insert+flag+scan+assign, inverse
    } else if (ctx->overlap && ctx->side) {
        // the internal stream takes seg_of (needs only the field layout) beside the dedup chain,
        // then the transpose beside the pool
        ctx->mark(0, true, s);
        if (!a.region_base) CK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
        launch_field_prep(a, s);  // (+ the table regions' clear)
        CK(cudaEventRecord(ctx->ev_fp, s));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fp, 0));
        launch_seg_of(offsets, batch, ctx->F, ctx->field_gstart, ctx->id_start, ctx->seg_of, ctx->side, ctx->finfo,
                      ctx->empty_pack, ctx->seg_limit, ctx->err);
        CK(cudaEventRecord(ctx->ev_seg, ctx->side));
        launch_dedup_insert(a, s);
        launch_dedup_assign(a, s);
        ctx->mark(0, false, s);
        ctx->launches_fwd += 2 + (n_ids > 0 ? 4 : 0) + 1;  // prep, seg_of, insert+flag+scan+assign, inverse
        CK(cudaEventRecord(ctx->ev_fork, s));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        picasso::transpose_on(ctx, ctx->side);
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
        CK(cudaStreamWaitEvent(s, ctx->ev_seg, 0));  // the pool reads seg_of
    } else {
        ctx->mark(0, true, s);
        if (!a.region_base) CK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
        launch_field_prep(a, s);  // (+ the table regions' clear)
        launch_dedup_insert(a, s);
        launch_dedup_assign(a, s);
        ctx->mark(0, false, s);
        ctx->launches_fwd += 1 + (n_ids > 0 ? 4 : 0) + 1;  // prep, insert+flag+scan+assign, inverse
        picasso::transpose_fork(ctx, s);
    }
    ctx->mark(1, true, s);
    {
        PoolArgs pa{};
        pa.ids = ids;
        pa.offsets = offsets;
        pa.B = batch;
        ctx->launches_fwd += launch_pool_all(ctx, pa, out, s);
    }
    ctx->mark(1, false, s);
    picasso::transpose_join(ctx, s);
    CK(cudaGetLastError());
    ctx->fwd_done = true;
    ctx->last_stream = s;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_packed_lookup_bwd_update(picasso_ctx *ctx, const float *grad_out, float lr,
                                                           int64_t step, void *stream) {
    NvtxRange nvtx("picasso_bwd_update");
    if (!ctx || step < 1) return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound || !ctx->fwd_done || ctx->di_active) return PICASSO_ERR_STATE;
    if (!grad_out && ctx->B > 0) return PICASSO_ERR_INVALID_ARG;  // an empty batch has no dY
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ctx->launches_bwd = 0;
    if (ctx->world > 1) {
        if (ctx->mp.group) return PICASSO_ERR_STATE;  // loopback: picasso_group_bwd_update
        if (!ctx->mp.comm && (!ctx->mp.p2p || ctx->opts.cache_max_bytes > 0)) return PICASSO_ERR_STATE;
        return ctx->mp.p2p ? multi_bwd_p2p(ctx, grad_out, lr, step, s) : multi_bwd_nccl(ctx, grad_out, lr, step, s);
    }
    if (ctx->opts.cold_tier) return ct_bwd(ctx, grad_out, lr, step, s);
    const int64_t N = ctx->N;
    ctx->mark(3, true, s);  // the transpose ran in the forward (transpose_fork)
    UpdateArgs u = picasso::make_update_args(ctx, grad_out, lr, step, ctx->su, ctx->sseg);
    if (N > 0) {
        if (ctx->dy_stage) {
            launch_dy_pack(grad_out, ctx->B, ctx->out_width, ctx->col4_field_d, ctx->finfo, ctx->dyp_base_d,
                           ctx->dyp_stride_d, ctx->dyp, s);
            ctx->launches_bwd += 1;
            u.dy_col = ctx->dyp_col_d;
        }
        for (int32_t p = 0; p < ctx->P; ++p) {  // packs in stream order share the long-row scratch
            ctx->mark_pack(1, p, true, s);
            u.pack = p;
            if (ctx->dy_stage) {  // this pack's rows of the regrouped dY
                u.dy = ctx->dyp + ctx->dyp_off[p];
                u.dy_stride = (int64_t)(ctx->pack_first_k[p + 1] - ctx->pack_first_k[p]) * ctx->pack_dim[p];
            }
            u.long_cnt = ctx->long_cnt + p;
            u.pack_key_off = ctx->pack_key_off[p];
            u.weight = ctx->w[p];
            u.state1 = ctx->s1[p];
            u.state2 = ctx->s2[p];
            int fl = 0;
            if (ctx->fuse_pipe && ctx->bulk_segsum) fl = launch_segsum_fused(ctx->pack_dim[p], u, ctx->num_sms, s);
            if (fl) {  // segment-sum and optimizer in one pass over the rows
                ctx->launches_bwd += fl;
            } else {
                ctx->launches_bwd += 1 + launch_segsum_any(ctx, ctx->pack_dim[p], u, s);
                ctx->mark(3, false, s);
                ctx->mark(5, true, s);
                launch_update_rows(ctx->pack_dim[p], u, ctx->num_sms, s);
                ctx->mark(5, false, s);
                ctx->mark(3, true, s);
            }
            ctx->mark_pack(1, p, false, s);
        }
    }
    ctx->mark(3, false, s);
    if (ctx->prof) ++ctx->prof_calls;
    CK(cudaGetLastError());
    ctx->fwd_done = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

// The backward's transpose (stable sort of the inverse index by uid, row starts, tiles) depends
// only on the forward's index phase: the forward launches it right after that phase, on an
// internal stream, so it overlaps the Gather / exchange / pool; the forward joins it before it
// returns (a forward stays self-contained, e.g. inside a CUDA graph capture).  k_seg_of first:
// segment of every packed position, for the sort and the pool.
void picasso::transpose_fork(picasso_ctx *ctx, cudaStream_t s) {
    launch_seg_of(ctx->offsets, ctx->B, ctx->F, ctx->field_gstart, ctx->id_start, ctx->seg_of, s, ctx->finfo,
                  ctx->empty_pack, ctx->seg_limit, ctx->err);
    ctx->launches_fwd += (int64_t)ctx->F * ctx->B > 0 ? 1 : 0;
    cudaStream_t t = s;
    if (ctx->overlap && ctx->side) {
        cudaEventRecord(ctx->ev_fork, s);
        cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
        t = ctx->side;
    }
    transpose_on(ctx, t);
    if (t != s) cudaEventRecord(ctx->ev_join, t);
}

// the transpose itself, on stream t (seg_of and the pass-0 histogram already written)
void picasso::transpose_on(picasso_ctx *ctx, cudaStream_t t) {
    ctx->mark(2, true, t);
    int32_t *su = nullptr, *sseg = nullptr;
    radix_sort_pairs2(ctx->inverse, ctx->seg_of, ctx->k_a, ctx->v_a, ctx->k_b, ctx->v_b, &su, &sseg, ctx->N,
                      ctx->splan, ctx->hist0, ctx->hist1, ctx->rowtot, t, &ctx->launches_fwd);
    launch_csr_any(ctx, su, ctx->N, t);
    ctx->launches_fwd += ctx->N > 0 ? 1 : 0;
    ctx->mark(2, false, t);
    ctx->su = su;
    ctx->sseg = sseg;
}

void picasso::transpose_join(picasso_ctx *ctx, cudaStream_t s) {
    if (ctx->world > 1 && ctx->w_runorder) return;  // no transpose was forked (sort-indexed step)
    if (ctx->overlap && ctx->side) cudaStreamWaitEvent(s, ctx->ev_join, 0);
}

void picasso::launch_csr_any(picasso_ctx *ctx, const int32_t *su, int64_t N, cudaStream_t s) {
    if (ctx->bulk_segsum)
        launch_csr_tiles(su, N, ctx->ustart, ctx->long_cnt, ctx->pack_gstart, ctx->pack_ustart, ctx->P, ctx->seg_nt,
                         ctx->tile_start, s, ctx->fuse_pipe ? ctx->fuse_rw : 1);
    else
        launch_csr_bounds(su, N, ctx->ustart, ctx->long_cnt, ctx->P, s);
}

// Gather + Stitch + pool of every pack (base: ids / offsets / B, plus row_off / inverse at W > 1,
// where the rows come from the received-rows buffer instead of the local tables).
int picasso::launch_pool_all(picasso_ctx *ctx, PoolArgs pa, float *out, cudaStream_t s, int only_pack) {
    int n = 0;
    pa.finfo = ctx->finfo;
    pa.field_gstart = ctx->field_gstart;
    pa.id_start = ctx->id_start;
    pa.seg_of = ctx->seg_of;
    pa.id_mode = ctx->opts.id_mode;
    pa.pool_mean = ctx->opts.pool == PICASSO_POOL_MEAN;
    pa.out = out;
    pa.out_stride = ctx->out_width;
    pa.err = ctx->err;
    pa.pack_gstart = ctx->pack_gstart;
    pa.field_k = ctx->pipe_pool ? ctx->field_k_d : nullptr;
    pa.empty_pack = ctx->empty_pack;
    pa.n_ids = ctx->N;
    for (int32_t p = 0; p < ctx->P; ++p) {  // seg_of: written by transpose_fork (k_seg_of)
        if (only_pack >= 0 && p != only_pack) continue;
        pa.pack = p;
        pa.Fp = ctx->pack_first_k[p + 1] - ctx->pack_first_k[p];
        pa.pack_fields = ctx->pm_fields_d + ctx->pack_first_k[p];
        pa.weight = pa.row_off ? ctx->gbuf : ctx->w[p];
        if ((int64_t)pa.Fp * pa.B == 0) continue;
        {   // 32-B row / output chunks (k_pool_flat8): local rows, 32-B aligned columns and table
            bool ok = !pa.row_off && ctx->out_width % 8 == 0 && ((uintptr_t)pa.weight & 31) == 0 &&
                      ((uintptr_t)out & 31) == 0;
            for (int32_t k = ctx->pack_first_k[p]; ok && k < ctx->pack_first_k[p + 1]; ++k)
                ok = ctx->fcol[ctx->pm_fields[k]] % 8 == 0;
            pa.vec8 = ok;
        }
        ctx->mark_pack(0, p, true, s);
        if (ctx->pool_kind == 2) {
            n += launch_pool_flat(ctx->pack_dim[p], pa, ctx->num_sms, s);
        } else if (pool_pipe_supported(ctx->pack_dim[p], pa)) {  // D >= 64: the cp.async ring
            n += launch_pool_pipe(ctx->pack_dim[p], pa, ctx->pool_sms, s);  // (+ its empty segments)
        } else if (ctx->pipe_pool) {  // narrow rows: one thread per 16-B chunk (C4: 20 -> 6 ms)
            n += launch_pool_flat(ctx->pack_dim[p], pa, ctx->num_sms, s);
        } else {  // PICASSO_POOL=legacy
            launch_pool(ctx->pack_dim[p], pa, ctx->num_sms, s);
            ++n;
        }
        ctx->mark_pack(0, p, false, s);
    }
    return n;
}

int picasso::launch_segsum_any(picasso_ctx *ctx, int D, const UpdateArgs &u, cudaStream_t s) {
    if (ctx->bulk_segsum && segsum_bulk_supported(D, u))
        return launch_segsum_bulk(ctx->seg_cfg, D, u, ctx->num_sms, s);
    launch_segsum(D, u, ctx->num_sms, s, ctx->flat_small);
    return 1 + launch_long_update(D, u, ctx->num_sms, s);
}

UpdateArgs picasso::make_update_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step,
                                     const int32_t *su, const int32_t *sseg) {
    UpdateArgs u{};
    u.sorted_u = su;
    u.sorted_seg = sseg;
    u.ustart = ctx->ustart;
    u.pack_ustart = ctx->pack_ustart;
    u.unique_gkey = ctx->row_keys();
    u.offsets = ctx->offsets;
    u.B = ctx->B;
    u.finfo = ctx->finfo;
    u.dy = grad_out;
    u.dy_stride = ctx->out_width;
    u.pool_mean = ctx->opts.pool == PICASSO_POOL_MEAN;
    u.opt = ctx->opts.opt;
    u.lr = lr;
    u.eps = ctx->opts.eps;
    u.beta1 = ctx->opts.beta1;
    u.beta2 = ctx->opts.beta2;
    {   // SparseAdam step size, in double then rounded once (torch: lr*sqrt(bc2)/bc1)
        const double bc1 = 1.0 - std::pow((double)ctx->opts.beta1, (double)step);
        const double bc2 = 1.0 - std::pow((double)ctx->opts.beta2, (double)step);
        u.adam_ss = (float)((double)lr * std::sqrt(bc2) / bc1);
    }
    u.long_list = ctx->long_list;
    u.chunk_off = ctx->chunk_off;
    u.partial = ctx->partial;
    u.chunk_row = ctx->chunk_row;
    u.gbuf = ctx->split_bwd ? ctx->gbuf : nullptr;
    u.pack_gbase = ctx->pack_gbase;
    u.tile_start = ctx->bulk_segsum ? ctx->tile_start : nullptr;
    u.nt = ctx->seg_nt;
    u.split = ctx->split;
    return u;
}

extern "C" picasso_status picasso_last_error(picasso_ctx *ctx, char *msg, size_t len) {
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    picasso_status st = PICASSO_OK;
    std::string m = ctx->last_msg;
    if (ctx->bound) {
        cudaError_t e = cudaStreamSynchronize(ctx->last_stream);
        if (e != cudaSuccess) {
            m = cudaGetErrorString(e);
            st = PICASSO_ERR_CUDA;
        } else {
            int h = 0;
            if (cudaMemcpy(&h, ctx->err, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && h) {
                if (h & ERR_PEER_TIMEOUT) { st = PICASSO_ERR_STATE; m = "peer timeout: a rank never reached a barrier (sticky: destroy the context)"; }
                else if (h & ERR_ID_RANGE) { st = PICASSO_ERR_ID_RANGE; m = "raw ID outside [0, V_t) in ROWS mode"; }
                else if (h & ERR_OFFSETS) { st = PICASSO_ERR_INVALID_ARG; m = "offsets are not a CSR over n_ids IDs"; }
                else if (h & ERR_CAPACITY) { st = PICASSO_ERR_CAPACITY; m = "device capacity overflow"; }
                // ID-range / capacity / offsets errors belong to the step that raised them; a peer
                // timeout is sticky (the ranks' barrier epochs no longer agree: destroy the context)
                cudaMemset(ctx->err, 0, sizeof(int));
                if (h & ERR_PEER_TIMEOUT) {
                    const int keep = ERR_PEER_TIMEOUT;
                    cudaMemcpy(ctx->err, &keep, sizeof(int), cudaMemcpyHostToDevice);
                }
            }
        }
    }
    if (msg && len) {
        std::snprintf(msg, len, "%s", m.c_str());
    }
    return st;
}

extern "C" picasso_status picasso_get_unique(picasso_ctx *ctx, int32_t pack, int64_t *dst, int64_t cap, int64_t *n) {
    if (!ctx || !n || pack < 0 || pack >= ctx->P || !ctx->bound) return PICASSO_ERR_INVALID_ARG;
    if (picasso_status st = ensure_views(ctx)) return st;
    CK(cudaStreamSynchronize(ctx->last_stream));
    std::vector<int32_t> us(ctx->P + 1);
    CK(cudaMemcpy(us.data(), ctx->pack_ustart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost));
    const int64_t U = us[pack + 1] - us[pack];
    *n = U;
    if (dst && cap > 0 && U > 0) {
        std::vector<unsigned long long> g(U);
        CK(cudaMemcpy(g.data(), ctx->unique_gkey + us[pack], sizeof(unsigned long long) * U, cudaMemcpyDeviceToHost));
        std::vector<int64_t> k(U);
        for (int64_t i = 0; i < U; ++i) k[i] = (int64_t)(g[i] - (unsigned long long)ctx->pack_key_off[pack]);
        CK(cudaMemcpy(dst, k.data(), sizeof(int64_t) * std::min(U, cap), cudaMemcpyHostToDevice));
    }
    return PICASSO_OK;
}

extern "C" picasso_status picasso_get_inverse(picasso_ctx *ctx, int32_t pack, int32_t *dst, int64_t cap, int64_t *n) {
    if (!ctx || !n || pack < 0 || pack >= ctx->P || !ctx->bound) return PICASSO_ERR_INVALID_ARG;
    if (picasso_status st = ensure_views(ctx)) return st;
    CK(cudaStreamSynchronize(ctx->last_stream));
    std::vector<int32_t> gs(ctx->P + 1), us(ctx->P + 1);
    CK(cudaMemcpy(gs.data(), ctx->pack_gstart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(us.data(), ctx->pack_ustart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost));
    const int64_t Np = gs[pack + 1] - gs[pack];
    *n = Np;
    if (dst && cap > 0 && Np > 0) {
        std::vector<int32_t> v(Np);
        CK(cudaMemcpy(v.data(), ctx->inverse + gs[pack], sizeof(int32_t) * Np, cudaMemcpyDeviceToHost));
        for (auto &x : v) x -= us[pack];
        CK(cudaMemcpy(dst, v.data(), sizeof(int32_t) * std::min(Np, cap), cudaMemcpyHostToDevice));
    }
    return PICASSO_OK;
}

extern "C" picasso_status picasso_profile_enable(picasso_ctx *ctx, int32_t on) {
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    if (on == 2 && !ctx->prof_graph) {  // start of a graph capture: fresh event list, kept afterwards
        for (int ph = 0; ph < picasso_ctx::kAllPhases; ++ph) ctx->ev_used[ph] = 0;
        ctx->prof_calls = 0;
    }
    ctx->prof = on != 0;
    ctx->prof_graph = on == 2;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_profile_read(picasso_ctx *ctx, float *ms, int64_t *calls) {
    if (!ctx || !ms) return PICASSO_ERR_INVALID_ARG;
    for (int ph = 0; ph < picasso_ctx::kPhases; ++ph) {
        float tot = 0.f;
        for (size_t i = 0; i < ctx->ev_used[ph]; ++i) {
            CK(cudaEventSynchronize(ctx->ev[ph][i].second));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, ctx->ev[ph][i].first, ctx->ev[ph][i].second));
            tot += t;
        }
        ms[ph] = tot;
        if (!ctx->prof_graph) ctx->ev_used[ph] = 0;  // graph mode: the replayed nodes re-record them
    }
    if (!ctx->prof_graph)
        for (int ph = picasso_ctx::kPhases; ph < picasso_ctx::kAllPhases; ++ph) ctx->ev_used[ph] = 0;
    if (calls) *calls = ctx->prof_graph ? 1 : ctx->prof_calls;
    if (!ctx->prof_graph) ctx->prof_calls = 0;
    return PICASSO_OK;
}

// per pack (first kPackPhases packs): its pool and its backward kernels since the last read; call
// before picasso_profile_read, which resets them
extern "C" picasso_status picasso_profile_read_packs(picasso_ctx *ctx, float *pool_ms, float *bwd_ms, int32_t cap) {
    if (!ctx || !pool_ms || !bwd_ms || cap < 0) return PICASSO_ERR_INVALID_ARG;
    for (int32_t p = 0; p < cap; ++p) {
        for (int which = 0; which < 2; ++which) {
            float tot = 0.f;
            if (p < picasso_ctx::kPackPhases) {
                const int ph = picasso_ctx::kPhases + which * picasso_ctx::kPackPhases + p;
                for (size_t i = 0; i < ctx->ev_used[ph]; ++i) {
                    CK(cudaEventSynchronize(ctx->ev[ph][i].second));
                    float t = 0.f;
                    CK(cudaEventElapsedTime(&t, ctx->ev[ph][i].first, ctx->ev[ph][i].second));
                    tot += t;
                }
            }
            (which ? bwd_ms : pool_ms)[p] = tot;
        }
    }
    return PICASSO_OK;
}

extern "C" picasso_status picasso_unique_offsets(picasso_ctx *ctx, int32_t *dst, void *stream) {
    if (!ctx || !dst || !ctx->bound) return PICASSO_ERR_INVALID_ARG;
    CK(cudaMemcpyAsync(dst, ctx->pack_ustart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDefault,
                       reinterpret_cast<cudaStream_t>(stream)));
    return PICASSO_OK;
}

extern "C" picasso_status picasso_launch_count(const picasso_ctx *ctx, int64_t *fwd, int64_t *bwd) {
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    if (fwd) *fwd = ctx->launches_fwd;
    if (bwd) *bwd = ctx->launches_bwd;
    return PICASSO_OK;
}
