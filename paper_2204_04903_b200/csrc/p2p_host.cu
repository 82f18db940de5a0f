#include <cstdlib>
// p2p_host.cu — host orchestration of the row-sharded step over NVLink peer memory.
//
//   fwd:  A  dedup + Partition (multi_host.cu)                 -> barrier 0 (send lists ready)
//         C' owner: block table from the peers' counts, keys read from the requesters' send
//            lists into a direct (row, source) table, rows stored into the requesters' rows
//            buffers -> barrier 1
//         D  pool from the local rows buffer (multi_host.cu)
//   bwd:  E  transpose + segment-sum, G rows stored into the owners' receive buffers -> barrier 2
//         (HybridHash hot rows: AllReduce as in the NCCL driver)
//         F' owner: per requested row, the pushed G rows reduced in source order, optimizer
// No host synchronisation inside the step (sizes live on the device), so a step can be captured
// in a CUDA graph.  Barrier 0 also orders every owner's F' pulls of the previous step before
// any rank's buffers are rewritten (a rank signals it only after its own F').  Windows are
// exchanged with CUDA IPC handles (one process per GPU) or, for the loopback group, are plain
// pointers on one device (the host then runs each phase for every rank before the next one,
// which is the barrier).
#include "ctx.h"

#define PCK(x)                                                                    \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_);        \
            return PICASSO_ERR_CUDA;                                              \
        }                                                                         \
    } while (0)
#define PNCK(x)                                                                   \
    do {                                                                          \
        ncclResult_t r_ = (x);                                                    \
        if (r_ != ncclSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + ncclGetErrorString(r_);        \
            return PICASSO_ERR_NCCL;                                              \
        }                                                                         \
    } while (0)

// phases shared with the NCCL driver (multi_host.cu)
picasso_status mfwd_a(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                      cudaStream_t s);
picasso_status mfwd_d(picasso_ctx *ctx, float *out, cudaStream_t s);
picasso_status mbwd_e(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s);
picasso_status hot_allreduce_group(std::vector<picasso_ctx *> &cs, cudaStream_t s);
picasso_status hot_update_all(picasso_ctx *ctx, float lr, float ss, cudaStream_t s);
picasso_status nvls_allreduce(picasso_ctx *ctx, cudaStream_t s);  // nvls.cu
UpdateArgs mbwd_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s);
int mbwd_segsum_pack(picasso_ctx *ctx, UpdateArgs u, int p, cudaStream_t s);
namespace picasso {
int launch_pool_all(picasso_ctx *ctx, PoolArgs pa, float *out, cudaStream_t s, int only_pack = -1);  // #launches
void transpose_join(picasso_ctx *ctx, cudaStream_t s);
}

namespace {

int max_dim(const picasso_ctx *ctx) {
    int maxD = 4;
    for (int32_t d : ctx->pack_dim) maxD = std::max(maxD, d);
    return maxD;
}

constexpr size_t kFlagBytes = sizeof(uint32_t) * kP2PFlags * kP2PMaxW;

// window: [flags | bcount | send_keys | gbuf | ogbuf], the same layout on every rank (same plan,
// max_ids, max_recv)
void window_layout(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    const int64_t N = std::max<int64_t>(ctx->opts.max_ids, 1);
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    size_t o = up(kFlagBytes);
    mp.win_bcount = o;
    o = up(o + sizeof(int32_t) * kMaxRadix);
    mp.win_keys = o;
    o = up(o + sizeof(int32_t) * N);
    mp.win_gbuf = o;
    o = up(o + sizeof(float) * (size_t)N * max_dim(ctx));
    mp.win_ogbuf = o;
    o = up(o + sizeof(float) * (size_t)std::max<int64_t>(mp.max_recv, 1) * max_dim(ctx));
    mp.win_bytes = o;
}

void set_peer(picasso_ctx *ctx, int q, char *base) {
    MultiState &mp = ctx->mp;
    mp.peers.flags[q] = reinterpret_cast<uint32_t *>(base);
    mp.peers.bcount[q] = reinterpret_cast<int32_t *>(base + mp.win_bcount);
    mp.peers.send_keys[q] = reinterpret_cast<int32_t *>(base + mp.win_keys);
    mp.peers.gbuf[q] = reinterpret_cast<float *>(base + mp.win_gbuf);
    mp.peers.ogbuf[q] = reinterpret_cast<float *>(base + mp.win_ogbuf);
}

// allocate this rank's window and move the shared buffers (bucket counts, send list, rows / G
// buffer) into it
picasso_status window_alloc(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    if (mp.win) return PICASSO_OK;
    window_layout(ctx);
    PCK(cudaMalloc(&mp.win, mp.win_bytes));
    PCK(cudaMalloc(&mp.dtab, sizeof(int32_t) * (size_t)std::max<int64_t>(mp.rows_total, 1) * ctx->world));
    PCK(cudaMemset(mp.dtab, 0xFF, sizeof(int32_t) * (size_t)std::max<int64_t>(mp.rows_total, 1) * ctx->world));
    PCK(cudaMemset(mp.R_d, 0, sizeof(int32_t)));
    PCK(cudaMemset(mp.win, 0, mp.win_bcount));
    set_peer(ctx, ctx->rank, mp.win);
    mp.bcount = mp.peers.bcount[ctx->rank];
    mp.send_keys = mp.peers.send_keys[ctx->rank];
    ctx->gbuf = mp.peers.gbuf[ctx->rank];
    PCK(cudaMemset(mp.epoch_d, 0, sizeof(uint32_t) * 2 * kP2PFlags));
    return PICASSO_OK;
}

P2PArgs make_p2p_args(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    P2PArgs a{};
    a.W = ctx->world;
    a.P = ctx->P;
    a.rank = ctx->rank;
    a.max_recv = mp.max_recv;
    a.peer = mp.peers;
    a.epoch = mp.epoch_d;
    a.err = ctx->err;
    a.pack_dim = ctx->pack_dim_d;
    a.pack_key_off = ctx->pack_key_off_d;
    a.oblk = mp.oblk_d;
    a.pack_ostart = mp.opack_ostart_d;
    a.opack_gstart = mp.opack_gstart;
    a.R = mp.R_d;
    a.cnt_recv = mp.cnt_recv_d;
    a.lrow = mp.recv_keys;
    a.osrc = mp.opos_map;
    a.roff = mp.rsend_off;
    a.dtab = mp.dtab;
    a.olist = mp.oslot;     // (W > 2) the hash-dedup scratch of the NCCL driver, unused here
    a.ocount = mp.od_total;
    a.row_base = mp.row_base_d;
    a.pack_fbase = mp.pack_fbase_d;
    a.d_total = ctx->d_total;
    a.bkey = mp.bkey;
    a.send_pos = mp.send_pos;
    a.bstart = mp.bstart;
    a.dbase = mp.dbase_d;
    a.dst_rank = mp.dst_rank;
    a.dst_off = mp.dst_off;
    a.fcnt = ctx->opts.cache_max_bytes > 0 ? mp.fcnt : nullptr;
    a.fcnt_off = mp.fcnt_off_d;
    return a;
}

void barrier(picasso_ctx *ctx, int phase, cudaStream_t s) {
    if (ctx->mp.p2p_loop) return;
    const P2PArgs a = make_p2p_args(ctx);
    launch_p2p_signal(a, phase * kP2PMaxGroups, s);
    launch_p2p_wait(a, phase * kP2PMaxGroups, s);
    ctx->launches_fwd += 2;
}
// split barrier of one K-Interleaving group: signal where the group's data is produced, wait
// where it is consumed (another stream)
void signal_group(picasso_ctx *ctx, int phase, int group, cudaStream_t s) {
    launch_p2p_signal(make_p2p_args(ctx), phase * kP2PMaxGroups + group, s);
}
void wait_group(picasso_ctx *ctx, int phase, int group, cudaStream_t s) {
    launch_p2p_wait(make_p2p_args(ctx), phase * kP2PMaxGroups + group, s);
}

// K-Interleaving over the packs: pack p's exchange overlaps pack p-1's pool
// (forward) and owner update (backward); one barrier per (phase, pack).  Needs >= 2 packs, no
// HybridHash, one process per GPU.
bool interleaved(const picasso_ctx *ctx) {
    return ctx->kinterleave && ctx->n_slots >= 2 && ctx->n_slots <= kP2PMaxGroups && ctx->opts.cache_max_bytes == 0 &&
           !ctx->mp.p2p_loop && ctx->side2;
}
// last pack of its barrier slot (a group's packs are contiguous)
bool slot_end(const picasso_ctx *ctx, int p) { return p + 1 == ctx->P || ctx->pack_slot[p + 1] != ctx->pack_slot[p]; }

// ---- C': owner side --------------------------------------------------------------------------
// W > 2: a leader-listing pass, then the update walks the listed rows; at W = 2 the update walks
// the owner positions and elects each row's leader itself (C2 loopback: the listing pass cost more
// than the update's extra lanes at W = 2; at N = 4 the fused form's idle lanes cost more: update
// 0.074 -> 0.096 ms vs owner phase 0.132 -> 0.120 ms)
static bool owner_list(const picasso_ctx *ctx) {
    static const char *e = std::getenv("PICASSO_P2P_LIST");  // measurement aid: 0 / 1 forces
    if (e) return e[0] == '1';
    return ctx->world > 2;
}

// 32-B chunks when every pack's rows are (the receive buffer's pack blocks then start on 32 B too)
static bool rows_vec8(const picasso_ctx *ctx, int p) {
    static const bool off = std::getenv("PICASSO_P2P_VEC4") != nullptr;  // measurement aid
    if (off) return false;
    for (int32_t d : ctx->pack_dim)
        if (d % 8) return false;
    auto al = [](const float *q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 31) == 0; };
    return al(ctx->w[p]) && al(ctx->s1[p]) && (ctx->opts.opt != 1 || al(ctx->s2[p]));
}

picasso_status p2p_c(picasso_ctx *ctx, cudaStream_t s, bool kil) {
    const int P = ctx->P;
    const P2PArgs a = make_p2p_args(ctx);
    ctx->mark(4, true, s);
    if (ctx->mp.reset_forked) {  // the reset ran beside unique + partition (multi_fwd_p2p)
        PCK(cudaStreamWaitEvent(s, ctx->ev_join2, 0));
        ctx->mp.reset_forked = false;
    } else {
        launch_p2p_reset(a, ctx->num_sms, s);  // the previous forward's direct-table entries
    }
    launch_p2p_tables(a, s);
    launch_p2p_dst_insert(a, ctx->num_sms, s);
    if (owner_list(ctx)) launch_p2p_leaders(a, ctx->num_sms, s);
    static const bool split = std::getenv("PICASSO_PROF_SPLIT") != nullptr;  // measurement aid
    if (split) ctx->mark(4, false, s);
    if (kil) {  // the pools start on the second stream once the prep is done
        PCK(cudaEventRecord(ctx->ev_fork2, s));
        PCK(cudaStreamWaitEvent(ctx->side2, ctx->ev_fork2, 0));
    }
    int nsig = 0;
    for (int p = 0; p < P; ++p) {
        launch_p2p_gather(ctx->pack_dim[p], a, ctx->w[p], p, ctx->num_sms, s, rows_vec8(ctx, p));
        if (kil && slot_end(ctx, p)) {  // the slot's rows are in every requester's buffer
            signal_group(ctx, 1, ctx->pack_slot[p], s);
            ++nsig;
        }
    }
    if (!split) ctx->mark(4, false, s);
    ctx->launches_fwd += 3 + (owner_list(ctx) ? 1 : 0) + P + nsig;
    PCK(cudaGetLastError());
    return PICASSO_OK;
}

// ---- F': owner reduce (pulled G rows, source order) + optimizer -------------------------------
float adam_step(const picasso_ctx *ctx, float lr, int64_t step) {
    const double bc1 = 1.0 - std::pow((double)ctx->opts.beta1, (double)step);
    const double bc2 = 1.0 - std::pow((double)ctx->opts.beta2, (double)step);
    return (float)((double)lr * std::sqrt(bc2) / bc1);
}

void p2p_update_pack(picasso_ctx *ctx, const P2PArgs &a, int p, float lr, float ss, cudaStream_t s) {
    launch_p2p_update(ctx->pack_dim[p], a, p, ctx->w[p], ctx->s1[p], ctx->s2[p], ctx->opts.opt, lr, ctx->opts.eps,
                      ctx->opts.beta1, ctx->opts.beta2, ss, ctx->num_sms, s, rows_vec8(ctx, p), owner_list(ctx));
    ctx->launches_bwd += 1;
}

picasso_status p2p_f(picasso_ctx *ctx, float lr, int64_t step, cudaStream_t s) {
    const P2PArgs a = make_p2p_args(ctx);
    const float ss = adam_step(ctx, lr, step);
    ctx->mark(5, true, s);
    for (int32_t p = 0; p < ctx->P; ++p) p2p_update_pack(ctx, a, p, lr, ss, s);
    picasso_status st = hot_update_all(ctx, lr, ss, s);
    if (st) return st;
    ctx->mark(5, false, s);
    if (ctx->prof) ++ctx->prof_calls;
    PCK(cudaGetLastError());
    ctx->fwd_done = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

}  // namespace

// ---- drivers ---------------------------------------------------------------------------------
picasso_status multi_fwd_p2p(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets, int32_t B, int64_t N,
                             float *out, cudaStream_t s) {
    picasso_status st;
    // the previous step's direct-table entries are cleared on the second stream while the
    // index work runs (it touches none of dtab / lrow / osrc / R); p2p_c joins it before the
    // tables kernel rewrites R
    ctx->mp.reset_forked = false;
    if (ctx->side2) {
        PCK(cudaEventRecord(ctx->ev_fork2, s));
        PCK(cudaStreamWaitEvent(ctx->side2, ctx->ev_fork2, 0));
        launch_p2p_reset(make_p2p_args(ctx), ctx->num_sms, ctx->side2);
        PCK(cudaEventRecord(ctx->ev_join2, ctx->side2));
        ctx->mp.reset_forked = true;
    }
    if ((st = mfwd_a(ctx, ids, offsets, B, N, s))) {
        if (ctx->mp.reset_forked) {  // keep the stream joined on the error path
            cudaStreamWaitEvent(s, ctx->ev_join2, 0);
            ctx->mp.reset_forked = false;
        }
        return st;
    }
    barrier(ctx, 0, s);
    const bool kil = interleaved(ctx);
    if ((st = p2p_c(ctx, s, kil))) return st;
    if (!kil) {
        barrier(ctx, 1, s);
        return mfwd_d(ctx, out, s);
    }
    // pool of pack p as soon as every owner has stored pack p's rows (gathers of later packs
    // still running on s)
    PoolArgs pa{};
    pa.ids = nullptr;
    pa.offsets = ctx->offsets;
    pa.B = ctx->B;
    pa.row_off = ctx->mp.row_off;
    pa.inverse = ctx->inverse;
    cudaStream_t t = ctx->side2;
    for (int p = 0; p < ctx->P; ++p) {
        if (p == 0 || ctx->pack_slot[p] != ctx->pack_slot[p - 1]) {  // the slot's first pack
            wait_group(ctx, 1, ctx->pack_slot[p], t);
            ctx->launches_fwd += 1;
        }
        ctx->mark(1, true, t);
        ctx->launches_fwd += launch_pool_all(ctx, pa, out, t, p);
        ctx->mark(1, false, t);
    }
    PCK(cudaEventRecord(ctx->ev_join2, t));
    PCK(cudaStreamWaitEvent(s, ctx->ev_join2, 0));
    transpose_join(ctx, s);
    PCK(cudaGetLastError());
    ctx->fwd_done = true;
    ctx->last_stream = s;
    return PICASSO_OK;
}

picasso_status multi_bwd_p2p(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, cudaStream_t s) {
    picasso_status st;
    MultiState &mp = ctx->mp;
    if (interleaved(ctx)) {  // owner update of pack p once every requester has stored pack p's G
        UpdateArgs u = mbwd_args(ctx, grad_out, lr, step, s);
        PCK(cudaEventRecord(ctx->ev_fork2, s));
        PCK(cudaStreamWaitEvent(ctx->side2, ctx->ev_fork2, 0));
        ctx->mark(3, true, s);
        for (int p = 0; p < ctx->P; ++p) {
            ctx->launches_bwd += mbwd_segsum_pack(ctx, u, p, s);
            if (slot_end(ctx, p)) {
                signal_group(ctx, 2, ctx->pack_slot[p], s);
                ctx->launches_bwd += 1;
            }
        }
        ctx->mark(3, false, s);
        const P2PArgs a = make_p2p_args(ctx);
        const float ss = adam_step(ctx, lr, step);
        cudaStream_t t = ctx->side2;
        for (int p = 0; p < ctx->P; ++p) {
            if (p == 0 || ctx->pack_slot[p] != ctx->pack_slot[p - 1]) {
                wait_group(ctx, 2, ctx->pack_slot[p], t);
                ctx->launches_bwd += 1;
            }
            ctx->mark(5, true, t);
            p2p_update_pack(ctx, a, p, lr, ss, t);
            ctx->mark(5, false, t);
        }
        PCK(cudaEventRecord(ctx->ev_join2, t));
        PCK(cudaStreamWaitEvent(s, ctx->ev_join2, 0));
        if (ctx->prof) ++ctx->prof_calls;
        PCK(cudaGetLastError());
        ctx->fwd_done = false;
        ctx->last_stream = s;
        return PICASSO_OK;
    }
    if ((st = mbwd_e(ctx, grad_out, lr, step, s))) return st;
    barrier(ctx, 2, s);
    if (mp.hot_k > 0 && mp.nvls) {  // HybridHash over NVLS: in-switch reduce + multicast broadcast
        if ((st = nvls_allreduce(ctx, s))) return st;
        barrier(ctx, 3, s);  // every rank's broadcast landed before any hot-row update reads it
    } else if (mp.hot_k > 0) {  // HybridHash: hot-row gradients and occurrence counts summed over ranks
        PNCK(ncclGroupStart());
        PNCK(ncclAllReduce(mp.hot_g, mp.hot_g, mp.hot_g_floats, ncclFloat32, ncclSum, mp.comm, s));
        PNCK(ncclAllReduce(mp.hot_touch, mp.hot_touch, mp.hot_k, ncclFloat32, ncclSum, mp.comm, s));
        PNCK(ncclGroupEnd());
    }
    return p2p_f(ctx, lr, step, s);
}

picasso_status group_fwd_p2p(picasso_group *g, const int64_t *const *ids, const int32_t *const *offsets,
                             const int32_t *batch, const int64_t *n_ids, float *const *out, cudaStream_t s) {
    const int W = (int)g->ctx.size();
    picasso_status st;
    for (int r = 0; r < W; ++r)
        if ((st = mfwd_a(g->ctx[r], ids[r], offsets[r], batch[r], n_ids[r], s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = p2p_c(g->ctx[r], s, false))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = mfwd_d(g->ctx[r], out[r], s))) return st;
    return PICASSO_OK;
}

picasso_status group_bwd_p2p(picasso_group *g, const float *const *grad_out, float lr, int64_t step,
                             cudaStream_t s) {
    const int W = (int)g->ctx.size();
    picasso_status st;
    for (int r = 0; r < W; ++r)
        if ((st = mbwd_e(g->ctx[r], grad_out[r], lr, step, s))) return st;
    if ((st = hot_allreduce_group(g->ctx, s))) return st;
    for (int r = 0; r < W; ++r)
        if ((st = p2p_f(g->ctx[r], lr, step, s))) return st;
    return PICASSO_OK;
}

// ---- C ABI: window exchange ------------------------------------------------------------------
extern "C" picasso_status picasso_p2p_handle(picasso_ctx *ctx, void *handle_out) {
    if (!ctx || !handle_out || ctx->world < 2 || !ctx->bound || ctx->mp.group || ctx->opts.exchange != 0)
        return PICASSO_ERR_INVALID_ARG;
    picasso_status st = window_alloc(ctx);
    if (st) return st;
    cudaIpcMemHandle_t h;
    PCK(cudaIpcGetMemHandle(&h, ctx->mp.win));
    std::memcpy(handle_out, &h, sizeof(h));
    return PICASSO_OK;
}

extern "C" picasso_status picasso_p2p_open(picasso_ctx *ctx, const void *handles) {
    if (!ctx || !handles || ctx->world < 2 || !ctx->mp.win || ctx->mp.p2p) return PICASSO_ERR_INVALID_ARG;
    MultiState &mp = ctx->mp;
    for (int q = 0; q < ctx->world; ++q) {
        if (q == ctx->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char *>(handles) + (size_t)q * sizeof(h), sizeof(h));
        void *base = nullptr;
        PCK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        mp.peer_base[q] = base;
        set_peer(ctx, q, static_cast<char *>(base));
    }
    mp.p2p = true;
    mp.p2p_loop = false;
    PCK(cudaDeviceSynchronize());
    return PICASSO_OK;
}

extern "C" picasso_status picasso_group_p2p(picasso_group *g) {
    if (!g || g->ctx.empty()) return PICASSO_ERR_INVALID_ARG;
    for (auto *ctx : g->ctx)
        if (ctx->opts.exchange != 0) return PICASSO_ERR_INVALID_ARG;
    for (auto *ctx : g->ctx) {
        picasso_status st = window_alloc(ctx);
        if (st) return st;
    }
    for (auto *ctx : g->ctx) {
        for (auto *peer : g->ctx) set_peer(ctx, peer->rank, peer->mp.win);
        ctx->mp.p2p = true;
        ctx->mp.p2p_loop = true;
    }
    return PICASSO_OK;
}

void p2p_release(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    for (int q = 0; q < kP2PMaxW; ++q)
        if (mp.peer_base[q]) {
            cudaIpcCloseMemHandle(mp.peer_base[q]);
            mp.peer_base[q] = nullptr;
        }
    if (mp.win) cudaFree(mp.win);
    if (mp.dtab) cudaFree(mp.dtab);
    mp.win = nullptr;
    mp.dtab = nullptr;
    mp.p2p = false;
}

// host view of this step's send counts (the P2P step never synchronises for them)
void p2p_host_counts(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    if (!mp.p2p || !mp.cnt_send_h) return;
    cudaStreamSynchronize(ctx->last_stream);
    cudaMemcpy(mp.cnt_send_h, mp.bcount, sizeof(int32_t) * (ctx->world * ctx->P + 1), cudaMemcpyDeviceToHost);
    const int W = ctx->world, P = ctx->P;
    mp.sk.assign(W, 0);
    int64_t tot = 0;
    for (int r = 0; r < W; ++r)
        for (int p = 0; p < P; ++p) {
            mp.sk[r] += mp.cnt_send_h[r * P + p];
            tot += mp.cnt_send_h[r * P + p];
        }
    mp.last_hot_uniques = mp.hot_k > 0 ? mp.cnt_send_h[W * P] : 0;
    mp.last_uniques = tot + mp.last_hot_uniques;
    mp.U_send = tot;
}
