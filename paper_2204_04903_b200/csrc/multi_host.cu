// multi_host.cu — host orchestration of the row-sharded step (world W > 1).
//
// The step is written as phases separated by exchange points (AllToAllv):
//   fwd:  A  dedup + Partition (send layout, bucket counts)        -> exchange counts
//         B  host: offsets + capacity checks, owner block table     -> exchange keys (IDs)
//         C  owner: dedup of received keys, contribution index, gather rows -> exchange rows
//         D  pool from the received rows (Stitch fused, L380-382)
//   bwd:  E  transpose + segment-sum -> gradient rows in the send layout -> exchange gradients
//         F  owner: reduce <= W contributions per row (source order) + optimizer
// Two drivers run the phases: one rank per process with NCCL grouped send/recv (the exchange
// of a rank is issued on its stream), or all ranks in one process ("loopback": exchanges
// are device copies between the ranks' buffers, used to test W up to 8 on one GPU).
#include "ctx.h"

#define MCK(x)                                                                    \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_);        \
            return PICASSO_ERR_CUDA;                                              \
        }                                                                         \
    } while (0)
#define NCK(x)                                                                    \
    do {                                                                          \
        ncclResult_t r_ = (x);                                                    \
        if (r_ != ncclSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + ncclGetErrorString(r_);        \
            return PICASSO_ERR_NCCL;                                              \
        }                                                                         \
    } while (0)

namespace picasso {
IndexArgs make_index_args(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N);
UpdateArgs make_update_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, const int32_t *su,
                            const int32_t *sseg);
int launch_segsum_any(picasso_ctx *ctx, int D, const UpdateArgs &u, cudaStream_t s);  // returns #launches
void launch_csr_any(picasso_ctx *ctx, const int32_t *su, int64_t N, cudaStream_t s);
int launch_pool_all(picasso_ctx *ctx, PoolArgs pa, float *out, cudaStream_t s, int only_pack = -1);  // #launches
void transpose_fork(picasso_ctx *ctx, cudaStream_t s);
void transpose_join(picasso_ctx *ctx, cudaStream_t s);
}
picasso_status hot_update_all(picasso_ctx *ctx, float lr, float ss, cudaStream_t s);
picasso_status group_fwd_p2p(picasso_group *g, const int64_t *const *ids, const int32_t *const *offsets,
                             const int32_t *batch, const int64_t *n_ids, float *const *out, cudaStream_t s);
picasso_status group_bwd_p2p(picasso_group *g, const float *const *grad_out, float lr, int64_t step,
                             cudaStream_t s);

static MultiArgs multi_args(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    MultiArgs m{};
    m.W = ctx->world;
    m.P = ctx->P;
    m.nblk = (std::max<int64_t>(ctx->N, 1) + kTile - 1) / kTile;
    int bb = 1;
    while ((1 << bb) < ctx->world * ctx->P) ++bb;
    m.bucket_bits = bb;
    m.pack_dim = ctx->pack_dim_d;
    m.pack_key_off = ctx->pack_key_off_d;
    m.d_total = ctx->d_total;
    m.pack_ustart = ctx->pack_ustart;
    m.unique_gkey = ctx->w_runorder && ctx->w_runx ? ctx->run_keys() : ctx->unique_gkey;  // (uid = run index)
    m.bkey = mp.bkey;
    m.bval = mp.bval;
    m.bhist = mp.bhist;
    m.bcount = mp.bcount;
    m.bstart = mp.bstart;
    m.sroff = mp.sroff;
    m.send_uid = mp.send_uid;
    m.send_pos = mp.send_pos;
    m.send_keys = mp.send_keys;
    m.row_off = mp.row_off;
    m.R = mp.R;
    m.oblk = mp.oblk_d;
    m.pack_ostart = mp.opack_ostart_d;
    m.recv_keys = mp.recv_keys;
    m.opos_map = mp.opos_map;
    m.oslot = mp.oslot;
    m.oinv = mp.oinv;
    m.ouid_key = mp.ouid_key;
    m.opack_ustart = mp.opack_ustart;
    m.contrib = mp.contrib;
    m.rsend_off = mp.rsend_off;
    m.rows_send = mp.rows_send;
    while ((1 << m.bucket_bits) < ctx->world * ctx->P + 1) ++m.bucket_bits;  // + the hot bucket
    m.hot_k = mp.hot_k;
    m.hot_index = mp.hot_index;
    m.hot_mask = mp.hot_mask;
    m.hslot = mp.hslot;
    m.hot_pslot = mp.hot_pslot_d;
    m.hot_w_off = mp.hot_off_d;
    m.hot_s1_off = mp.hot_off_d + ctx->P;
    m.hot_s2_off = mp.hot_off_d + 2 * ctx->P;
    m.hot_g_off = mp.hot_off_d + 3 * ctx->P;
    m.hot_arena = mp.hot_arena;
    m.hot_g = mp.hot_g;
    m.hot_touch = mp.hot_touch;
    m.hot_cnt = mp.hot_cnt;
    m.gbuf_base = ctx->gbuf;
    m.fcnt = mp.fcnt;
    m.fcnt_off = mp.fcnt_off_d;
    return m;
}

MultiArgs picasso_multi_args(picasso_ctx *ctx) { return multi_args(ctx); }

namespace picasso {
void launch_hot_probe(const MultiArgs &m, int num_sms, cudaStream_t s);
void launch_hot_update(int D, const MultiArgs &m, int pack, int opt, float lr, float eps, float b1, float b2, float ss,
                       int num_sms, cudaStream_t s);
void launch_sum_ranks(const RankPtrs &src, int W, float *dst, int64_t n, cudaStream_t s);
}  // namespace picasso

// ---- phase A: dedup (as at W = 1) + Partition into the owner-major send layout -------------
picasso_status w_sorted_index(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                              cudaStream_t s);  // runtime.cu

picasso_status mfwd_a(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                      cudaStream_t s) {
    MultiState &mp = ctx->mp;
    ctx->N = N;
    ctx->B = B;
    ctx->offsets = offsets;
    ctx->w_runorder = ctx->sort_w && B > 0 && N >= ctx->sort_min_ids_w;
    ctx->mark(0, true, s);
    if (ctx->w_runorder) {  // sort-based index: no dedup table, no uid transpose later
        picasso_status st = w_sorted_index(ctx, ids, offsets, B, N, s);
        if (st) return st;
    } else {
        IndexArgs a = make_index_args(ctx, ids, offsets, B, N);
        const uint32_t cap_step =
            (uint32_t)std::min<uint64_t>(ctx->cap, pow2_at_least((uint64_t)std::max<int64_t>(N, 1) * 2));
        a.cap_mask = cap_step - 1;
        if (!a.region_base) MCK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
        launch_field_prep(a, s);  // (+ the table regions' clear)
        launch_dedup_insert(a, s);
        launch_dedup_assign(a, s);
    }
    MultiArgs m = multi_args(ctx);
    if (mp.hot_k > 0) launch_hot_probe(m, ctx->num_sms, s);  // hot keys skip the exchange
    if (mp.p2p) {  // slot order inside a bucket is free: counts + placement, no sort
        launch_partition_p2p(m, ctx->num_sms, s);
    } else {       // first-occurrence order inside a bucket (the owner dedup's order, reading O2)
        launch_bucket(m, s);
        bucket_sort_pass(mp.bkey, mp.bval, mp.bsorted, mp.send_uid, std::max<int64_t>(N, 1), ctx->d_total,
                         m.bucket_bits, mp.bhist, mp.bcount, s);
        launch_bucket_prefix(m, s);
        launch_send_prep(m, ctx->num_sms, s);
    }
    // bucket counts (+ the hot bucket: the hit statistic of HybridHash); the peer-memory driver
    // never needs them on the host inside a step (p2p_host_counts copies them on request)
    if (!mp.p2p)
        MCK(cudaMemcpyAsync(mp.cnt_send_h, mp.bcount, sizeof(int32_t) * (ctx->world * ctx->P + 1),
                            cudaMemcpyDeviceToHost, s));
    ctx->mark(0, false, s);
    ctx->launches_fwd += 1 + (N > 0 ? 4 : 0) + 1 + 5;
    if (!ctx->w_runorder) transpose_fork(ctx, s);  // (the sort already gave the backward's rows)
    return PICASSO_OK;
}

// run-order backward of a sort-indexed row-sharded step: the per-row destination arrays the
// segment-sum indexes by row, gathered from their uid-indexed originals
static void run_order_args(picasso_ctx *ctx, UpdateArgs &u, cudaStream_t s) {
    if (!ctx->w_runorder) return;
    u.unique_gkey = ctx->run_keys();
    if (ctx->w_runx) return;  // rows were numbered in run order from the start
    launch_run_gather(ctx->run_uid, ctx->d_total, ctx->N, u.hslot, ctx->hs_run, u.row_off, ctx->ro_run, u.dst_rank,
                      ctx->dr_run, u.dst_off, ctx->do_run, ctx->num_sms, s);
    ctx->launches_bwd += 1;
    if (u.hslot) u.hslot = ctx->hs_run;
    if (u.row_off) u.row_off = ctx->ro_run;
    if (u.dst_rank) u.dst_rank = ctx->dr_run;
    if (u.dst_off) u.dst_off = ctx->do_run;
    u.unique_gkey = ctx->run_keys();
}

// ---- phase B: counts known -> offsets, capacity check, owner block table ------------------
picasso_status mfwd_b(picasso_ctx *ctx, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int W = ctx->world, P = ctx->P;
    MCK(cudaMemcpyAsync(mp.cnt_recv_h, mp.cnt_recv_d, sizeof(int32_t) * W * P, cudaMemcpyDeviceToHost, s));
    MCK(cudaStreamSynchronize(s));  // NCCL needs host-side sizes (SURVEY hard part 5)
    mp.skoff.assign(W + 1, 0);
    mp.sk.assign(W, 0);
    mp.rkoff.assign(W + 1, 0);
    mp.rk.assign(W, 0);
    mp.srow_off.assign(W + 1, 0);
    mp.srow_n.assign(W, 0);
    mp.rrow_off.assign(W + 1, 0);
    mp.rrow_n.assign(W, 0);
    for (int r = 0; r < W; ++r) {
        for (int p = 0; p < P; ++p) {
            const int64_t cs = mp.cnt_send_h[r * P + p], cr = mp.cnt_recv_h[r * P + p];
            mp.sk[r] += cs;
            mp.rk[r] += cr;
            mp.srow_n[r] += cs * ctx->pack_dim[p];
            mp.rrow_n[r] += cr * ctx->pack_dim[p];
        }
        mp.skoff[r + 1] = mp.skoff[r] + mp.sk[r];
        mp.rkoff[r + 1] = mp.rkoff[r] + mp.rk[r];
        mp.srow_off[r + 1] = mp.srow_off[r] + mp.srow_n[r];
        mp.rrow_off[r + 1] = mp.rrow_off[r] + mp.rrow_n[r];
    }
    mp.R = mp.rkoff[W];
    mp.last_hot_uniques = mp.hot_k > 0 ? mp.cnt_send_h[W * P] : 0;
    mp.last_uniques = mp.skoff[W] + mp.last_hot_uniques;
    mp.U_send = mp.skoff[W];
    if (mp.R > mp.max_recv) {
        ctx->last_msg = "received keys exceed max_recv";
        return PICASSO_ERR_CAPACITY;
    }
    // owner stream blocks, pack-major: (pack p, source src)
    mp.opack_ostart.assign(P + 1, 0);
    int64_t o = 0;
    for (int p = 0; p < P; ++p) {
        mp.opack_ostart[p] = o;
        for (int src = 0; src < W; ++src) {
            int64_t rs = mp.rkoff[src], rr = mp.rrow_off[src];
            for (int q = 0; q < p; ++q) {
                rs += mp.cnt_recv_h[src * P + q];
                rr += (int64_t)mp.cnt_recv_h[src * P + q] * ctx->pack_dim[q];
            }
            OwnerBlock &b = mp.oblk_h[p * W + src];
            b.ostart = o;
            b.rstart = rs;
            b.rroff = rr;
            b.pack = p;
            b.src = src;
            o += mp.cnt_recv_h[src * P + p];
        }
    }
    mp.opack_ostart[P] = o;
    for (int p = 0; p <= P; ++p) mp.ostart_h[p] = mp.opack_ostart[p];
    MCK(cudaMemcpyAsync(mp.oblk_d, mp.oblk_h, sizeof(OwnerBlock) * W * P, cudaMemcpyHostToDevice, s));
    MCK(cudaMemcpyAsync(mp.opack_ostart_d, mp.ostart_h, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
    return PICASSO_OK;
}

// ---- phase C: owner side: dedup of received keys, contribution index, gather ---------------
picasso_status mfwd_c(picasso_ctx *ctx, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int W = ctx->world, P = ctx->P;
    const int64_t R = mp.R;
    MultiArgs m = multi_args(ctx);
    // owner dedup reuses the index kernels on the owner stream (positions pack-major)
    IndexArgs a{};
    a.N = R;
    a.P = P;
    a.table = ctx->table;
    a.slot_of = mp.oslot;
    a.fmask = ctx->fmask;
    a.blk_cnt = ctx->blk_cnt;
    a.blk_off = ctx->blk_off;
    a.d_total = mp.od_total;
    a.unique_gkey = mp.ouid_key;
    a.pack_gstart = mp.opack_gstart;
    a.pack_ustart = mp.opack_ustart;
    a.inverse = mp.oinv;
    a.pack_dim = ctx->pack_dim_d;
    a.pack_gbase = mp.ogbase_scratch;
    a.sort_bits0 = 1;
    a.sort_hist0 = ctx->osort_hist;
    a.err = ctx->err;
    for (int p = 0; p <= P; ++p) mp.og_h[p] = (int32_t)mp.opack_ostart[p];
    MCK(cudaMemcpyAsync(mp.opack_gstart, mp.og_h, sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice, s));
    const uint32_t cap_step = (uint32_t)std::min<uint64_t>(ctx->cap, pow2_at_least((uint64_t)std::max<int64_t>(R, 1) * 2));
    ctx->mark(4, true, s);
    MCK(cudaMemsetAsync(ctx->table, 0xFF, sizeof(Slot) * cap_step, s));
    launch_owner_insert(m, ctx->table, cap_step - 1, ctx->err, s);
    launch_dedup_assign(a, s);
    MCK(cudaMemsetAsync(mp.contrib, 0xFF, sizeof(int32_t) * std::max<int64_t>(R, 1) * W, s));
    launch_contrib(m, s);
    for (int p = 0; p < P; ++p)
        if (mp.opack_ostart[p + 1] > mp.opack_ostart[p]) launch_gather(ctx->pack_dim[p], m, ctx->w[p], p, ctx->num_sms, s);
    ctx->mark(4, false, s);
    ctx->launches_fwd += (R > 0 ? 2 + 4 : 1) + P;
    return PICASSO_OK;
}

// ---- phase D: pool from the received rows ----------------------------------------------------
picasso_status mfwd_d(picasso_ctx *ctx, float *out, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    ctx->mark(1, true, s);
    {
        PoolArgs pa{};
        pa.ids = nullptr;
        pa.offsets = ctx->offsets;
        pa.B = ctx->B;
        pa.row_off = mp.row_off;
        pa.inverse = ctx->inverse;
        ctx->launches_fwd += launch_pool_all(ctx, pa, out, s);
    }
    ctx->mark(1, false, s);
    transpose_join(ctx, s);
    MCK(cudaGetLastError());
    ctx->fwd_done = true;
    ctx->last_stream = s;
    return PICASSO_OK;
}

// ---- phase E: transpose + segment-sum into the send layout -----------------------------------
// arguments of the phase-E segment-sum (hot buffers zeroed on s when the cache is on)
UpdateArgs mbwd_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s) {
    UpdateArgs u = make_update_args(ctx, grad_out, lr, step, ctx->su, ctx->sseg);
    MultiState &mp = ctx->mp;
    if (mp.hot_k > 0) {  // this rank's hot-row gradients and occurrence counts (AllReduced next)
        cudaMemsetAsync(mp.hot_g, 0, sizeof(float) * mp.hot_g_floats, s);
        cudaMemsetAsync(mp.hot_touch, 0, sizeof(float) * mp.hot_k, s);
        u.hslot = mp.hslot;
        u.hot_g = mp.hot_g;
        u.hot_g_off = mp.hot_off_d + 3 * ctx->P;
        u.hot_pslot = mp.hot_pslot_d;
        u.hot_touch = mp.hot_touch;
    }
    u.gbuf = ctx->gbuf;
    u.row_off = ctx->mp.row_off;
    if (mp.p2p) {  // G rows straight into the owners' receive buffers (p2p.cu)
        u.dst_rank = mp.dst_rank;
        u.dst_off = mp.dst_off;
        for (int q = 0; q < ctx->world; ++q) u.dst_buf[q] = mp.peers.ogbuf[q];
    }
    run_order_args(ctx, u, s);
    return u;
}

// segment-sum of one pack (phase E)
int mbwd_segsum_pack(picasso_ctx *ctx, UpdateArgs u, int p, cudaStream_t s) {
    if (ctx->N == 0) return 0;
    u.pack = p;
    u.long_cnt = ctx->long_cnt + p;
    u.pack_key_off = ctx->pack_key_off[p];
    return launch_segsum_any(ctx, ctx->pack_dim[p], u, s);
}

picasso_status mbwd_e(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s) {
    const int64_t N = ctx->N;
    ctx->mark(3, true, s);  // the transpose ran in the forward (transpose_fork)
    UpdateArgs u = make_update_args(ctx, grad_out, lr, step, ctx->su, ctx->sseg);
    MultiState &mp = ctx->mp;
    if (mp.hot_k > 0) {  // this rank's hot-row gradients and occurrence counts (AllReduced next)
        MCK(cudaMemsetAsync(mp.hot_g, 0, sizeof(float) * mp.hot_g_floats, s));
        MCK(cudaMemsetAsync(mp.hot_touch, 0, sizeof(float) * mp.hot_k, s));
        u.hslot = mp.hslot;
        u.hot_g = mp.hot_g;
        u.hot_g_off = mp.hot_off_d + 3 * ctx->P;
        u.hot_pslot = mp.hot_pslot_d;
        u.hot_touch = mp.hot_touch;
    }
    u.gbuf = ctx->gbuf;
    u.row_off = ctx->mp.row_off;
    if (mp.p2p) {  // G rows straight into the owners' receive buffers (p2p.cu)
        u.dst_rank = mp.dst_rank;
        u.dst_off = mp.dst_off;
        for (int q = 0; q < ctx->world; ++q) u.dst_buf[q] = mp.peers.ogbuf[q];
    }
    run_order_args(ctx, u, s);
    if (N > 0) {
        for (int32_t p = 0; p < ctx->P; ++p) {
            u.pack = p;
            u.long_cnt = ctx->long_cnt + p;
            u.pack_key_off = ctx->pack_key_off[p];
            ctx->launches_bwd += launch_segsum_any(ctx, ctx->pack_dim[p], u, s);
        }
    }
    ctx->mark(3, false, s);
    return PICASSO_OK;
}

// HybridHash replicas: the same update on every rank (after the hot-gradient AllReduce)
picasso_status hot_update_all(picasso_ctx *ctx, float lr, float ss, cudaStream_t s) {
    if (ctx->mp.hot_k == 0) return PICASSO_OK;
    MultiArgs m = multi_args(ctx);
    for (int32_t p = 0; p < ctx->P; ++p)
        if (ctx->mp.hot_pslot[p + 1] > ctx->mp.hot_pslot[p]) {
            launch_hot_update(ctx->pack_dim[p], m, p, ctx->opts.opt, lr, ctx->opts.eps, ctx->opts.beta1,
                              ctx->opts.beta2, ss, ctx->num_sms, s);
            ctx->launches_bwd += 1;
        }
    MCK(cudaGetLastError());
    return PICASSO_OK;
}

// ---- phase F: owner reduce (source order) + optimizer ----------------------------------------
picasso_status mbwd_f(picasso_ctx *ctx, float lr, int64_t step, cudaStream_t s) {
    MultiArgs m = multi_args(ctx);
    const double bc1 = 1.0 - std::pow((double)ctx->opts.beta1, (double)step);
    const double bc2 = 1.0 - std::pow((double)ctx->opts.beta2, (double)step);
    const float ss = (float)((double)lr * std::sqrt(bc2) / bc1);
    ctx->mark(5, true, s);
    for (int32_t p = 0; p < ctx->P; ++p) {
        launch_owner_update(ctx->pack_dim[p], m, p, ctx->w[p], ctx->s1[p], ctx->s2[p], ctx->opts.opt, lr,
                            ctx->opts.eps, ctx->opts.beta1, ctx->opts.beta2, ss, ctx->num_sms, s);
        ctx->launches_bwd += 1;
    }
    picasso_status st = hot_update_all(ctx, lr, ss, s);
    if (st) return st;
    ctx->mark(5, false, s);
    if (ctx->prof) ++ctx->prof_calls;
    MCK(cudaGetLastError());
    ctx->fwd_done = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

// ------------------------------------------------------------------------------------------
// NCCL driver: one rank per process
static picasso_status a2av_nccl(picasso_ctx *ctx, const void *send, const std::vector<int64_t> &soff,
                                const std::vector<int64_t> &sn, void *recv, const std::vector<int64_t> &roff,
                                const std::vector<int64_t> &rn, ncclDataType_t dt, size_t esz, cudaStream_t s) {
    NCK(ncclGroupStart());
    for (int r = 0; r < ctx->world; ++r) {
        if (sn[r] > 0) NCK(ncclSend(static_cast<const char *>(send) + soff[r] * esz, sn[r], dt, r, ctx->mp.comm, s));
        if (rn[r] > 0) NCK(ncclRecv(static_cast<char *>(recv) + roff[r] * esz, rn[r], dt, r, ctx->mp.comm, s));
    }
    NCK(ncclGroupEnd());
    return PICASSO_OK;
}

picasso_status multi_fwd_nccl(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                              float *out, cudaStream_t s) {
    const int W = ctx->world, P = ctx->P;
    picasso_status st;
    if ((st = mfwd_a(ctx, ids, offsets, B, N, s))) return st;
    std::vector<int64_t> cn(W, P), co(W + 1);
    for (int r = 0; r <= W; ++r) co[r] = (int64_t)r * P;
    if ((st = a2av_nccl(ctx, ctx->mp.bcount, co, cn, ctx->mp.cnt_recv_d, co, cn, ncclInt32, 4, s))) return st;
    if ((st = mfwd_b(ctx, s))) return st;
    MultiState &mp = ctx->mp;
    if ((st = a2av_nccl(ctx, mp.send_keys, mp.skoff, mp.sk, mp.recv_keys, mp.rkoff, mp.rk, ncclInt32, 4, s))) return st;
    if ((st = mfwd_c(ctx, s))) return st;
    if ((st = a2av_nccl(ctx, mp.rows_send, mp.rrow_off, mp.rrow_n, ctx->gbuf, mp.srow_off, mp.srow_n, ncclFloat32, 4,
                        s)))
        return st;
    return mfwd_d(ctx, out, s);
}

picasso_status multi_bwd_nccl(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s) {
    picasso_status st;
    MultiState &mp = ctx->mp;
    if ((st = mbwd_e(ctx, grad_out, lr, step, s))) return st;
    if ((st = a2av_nccl(ctx, ctx->gbuf, mp.srow_off, mp.srow_n, mp.rows_send, mp.rrow_off, mp.rrow_n, ncclFloat32, 4,
                        s)))
        return st;
    if (mp.hot_k > 0) {  // HybridHash: hot-row gradients and occurrence counts summed over ranks
        NCK(ncclGroupStart());
        NCK(ncclAllReduce(mp.hot_g, mp.hot_g, mp.hot_g_floats, ncclFloat32, ncclSum, mp.comm, s));
        NCK(ncclAllReduce(mp.hot_touch, mp.hot_touch, mp.hot_k, ncclFloat32, ncclSum, mp.comm, s));
        NCK(ncclGroupEnd());
    }
    return mbwd_f(ctx, lr, step, s);
}

// loopback AllReduce of the hot-row gradients / occurrence counts: rank-order sum into rank 0's
// scratch, then a copy to every rank (all replicas then apply identical arithmetic)
static picasso_status hot_allreduce_loop(std::vector<picasso_ctx *> &cs, cudaStream_t s) {
    picasso_ctx *ctx = cs[0];
    const int W = (int)cs.size();
    MultiState &m0 = ctx->mp;
    if (m0.hot_k == 0) return PICASSO_OK;
    RankPtrs pg{}, pt{};
    for (int r = 0; r < W; ++r) {
        pg.p[r] = cs[r]->mp.hot_g;
        pt.p[r] = cs[r]->mp.hot_touch;
    }
    launch_sum_ranks(pg, W, m0.hot_gsum, m0.hot_g_floats, s);
    launch_sum_ranks(pt, W, m0.stage, m0.hot_k, s);
    for (int r = 0; r < W; ++r) {
        MCK(cudaMemcpyAsync(cs[r]->mp.hot_g, m0.hot_gsum, sizeof(float) * m0.hot_g_floats, cudaMemcpyDeviceToDevice, s));
        MCK(cudaMemcpyAsync(cs[r]->mp.hot_touch, m0.stage, sizeof(float) * m0.hot_k, cudaMemcpyDeviceToDevice, s));
    }
    return PICASSO_OK;
}

picasso_status hot_allreduce_group(std::vector<picasso_ctx *> &cs, cudaStream_t s) { return hot_allreduce_loop(cs, s); }

// ------------------------------------------------------------------------------------------
// Loopback driver: all W ranks in this process, on one device; exchanges are device copies.

static picasso_status a2av_loop(picasso_group *g, int which, cudaStream_t s) {
    const int W = (int)g->ctx.size();
    for (int src = 0; src < W; ++src)
        for (int dst = 0; dst < W; ++dst) {
            picasso_ctx *a = g->ctx[src], *b = g->ctx[dst];
            picasso_ctx *ctx = a;
            const int P = a->P;
            const void *from = nullptr;
            void *to = nullptr;
            size_t bytes = 0;
            if (which == 0) {  // counts: src's bucket row for dst -> dst's receive row for src
                from = a->mp.bcount + dst * P;
                to = b->mp.cnt_recv_d + src * P;
                bytes = sizeof(int32_t) * P;
            } else if (which == 1) {  // keys
                from = a->mp.send_keys + a->mp.skoff[dst];
                to = b->mp.recv_keys + b->mp.rkoff[src];
                bytes = sizeof(int32_t) * a->mp.sk[dst];
            } else if (which == 2) {  // rows: owner src -> requester dst
                from = a->mp.rows_send + a->mp.rrow_off[dst];
                to = b->gbuf + b->mp.srow_off[src];
                bytes = sizeof(float) * a->mp.rrow_n[dst];
            } else {  // gradients: requester src -> owner dst
                from = a->gbuf + a->mp.srow_off[dst];
                to = b->mp.rows_send + b->mp.rrow_off[src];
                bytes = sizeof(float) * a->mp.srow_n[dst];
            }
            if (bytes) MCK(cudaMemcpyAsync(to, from, bytes, cudaMemcpyDeviceToDevice, s));
        }
    return PICASSO_OK;
}

extern "C" picasso_status picasso_group_create(picasso_ctx *const *ctxs, int32_t world, picasso_group **out) {
    if (!ctxs || !out || world < 2) return PICASSO_ERR_INVALID_ARG;
    auto *g = new picasso_group();
    for (int r = 0; r < world; ++r) {
        picasso_ctx *c = ctxs[r];
        if (!c || c->world != world || c->rank != r || c->mp.comm || !c->bound) {
            delete g;
            return PICASSO_ERR_INVALID_ARG;
        }
        g->ctx.push_back(c);
    }
    for (auto *c : g->ctx) c->mp.group = g;
    *out = g;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_group_destroy(picasso_group *g) {
    if (g)
        for (auto *c : g->ctx) c->mp.group = nullptr;
    delete g;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_group_fwd(picasso_group *g, const int64_t *const *ids, const int32_t *const *offsets,
                                            const int32_t *batch, const int64_t *n_ids, float *const *out,
                                            void *stream) {
    if (!g) return PICASSO_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int W = (int)g->ctx.size();
    picasso_status st;
    for (int r = 0; r < W; ++r) {
        picasso_ctx *c = g->ctx[r];
        if (batch[r] > c->opts.max_batch || n_ids[r] > c->opts.max_ids) return PICASSO_ERR_CAPACITY;
        c->launches_fwd = 0;
        if (c->mp.p2p) continue;
        if (c->opts.exchange == 0) return PICASSO_ERR_STATE;  // picasso_group_p2p not called
        if ((st = mfwd_a(c, ids[r], offsets[r], batch[r], n_ids[r], s))) return st;
    }
    if (g->ctx[0]->mp.p2p) return group_fwd_p2p(g, ids, offsets, batch, n_ids, out, s);
    if ((st = a2av_loop(g, 0, s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = mfwd_b(g->ctx[r], s))) return st;
    if ((st = a2av_loop(g, 1, s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = mfwd_c(g->ctx[r], s))) return st;
    if ((st = a2av_loop(g, 2, s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = mfwd_d(g->ctx[r], out[r], s))) return st;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_group_bwd_update(picasso_group *g, const float *const *grad_out, float lr,
                                                   int64_t step, void *stream) {
    if (!g || step < 1) return PICASSO_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int W = (int)g->ctx.size();
    picasso_status st;
    for (int r = 0; r < W; ++r) {
        picasso_ctx *c = g->ctx[r];
        if (!c->fwd_done) return PICASSO_ERR_STATE;
        c->launches_bwd = 0;
        if (c->mp.p2p) continue;
        if ((st = mbwd_e(c, grad_out[r], lr, step, s))) return st;
    }
    if (g->ctx[0]->mp.p2p) return group_bwd_p2p(g, grad_out, lr, step, s);
    if ((st = a2av_loop(g, 3, s))) return st;
    if ((st = hot_allreduce_loop(g->ctx, s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = mbwd_f(g->ctx[r], lr, step, s))) return st;
    return PICASSO_OK;
}
