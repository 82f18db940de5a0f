// cache_host.cu — picasso_hot_cache_refresh: Alg. 1 L514-517 on the row-sharded step.
//
//   1. replicas -> owners' shards; the ranks' hot-hit counts are summed (AllReduce) and added
//      to the owners' FCounter;
//   2. top-k (L515) without moving candidates: every owner histograms its rows' counts per pack,
//      the histograms are summed over the ranks (AllReduce), and every rank finds the same count
//      c* at which the selection by (count desc, key asc) reaches the capacity; the rows at c*
//      are cut in ascending key by a second AllReduced histogram over key bins and, inside the
//      bin where the budget runs out, the few tie keys themselves (AllGather);
//   3. owners set their selected rows in a bitmap over the global key space; summed over the
//      ranks (disjoint bits) it is the hot set, compacted on every rank into the hot keys in
//      ascending key (slots grouped by pack) — equal as a set to oracle_hot_select;
//   4. owners write their new hot rows into a slot-major staging buffer, the staging is summed
//      over the ranks as 32-bit words (each word has one non-zero contributor: an exact copy),
//      and every rank places it into its replica arena and rebuilds the key -> slot index.
// Everything but a few KB of histograms stays on the devices.  capacity_bytes = 0 writes back
// and drops the hot set (checkpoint / disable).
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "ctx.h"

void p2p_host_counts(picasso_ctx *ctx);  // p2p_host.cu

#define HCK(x)                                                                    \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_);        \
            return PICASSO_ERR_CUDA;                                              \
        }                                                                         \
    } while (0)
#define HNK(x)                                                                    \
    do {                                                                          \
        ncclResult_t r_ = (x);                                                    \
        if (r_ != ncclSuccess) {                                                  \
            ctx->last_msg = std::string(#x ": ") + ncclGetErrorString(r_);        \
            return PICASSO_ERR_NCCL;                                              \
        }                                                                         \
    } while (0)

MultiArgs picasso_multi_args(picasso_ctx *ctx);
namespace picasso {
void launch_sum_ranks_u32(const RankPtrs &src, int W, uint32_t *dst, int64_t n, cudaStream_t s);
void launch_writeback(int D, const MultiArgs &m, int pack, const unsigned long long *keys, float *w, float *s1,
                      float *s2, int nst, const uint32_t *cnt_sum, int rank, int num_sms, cudaStream_t s);
void launch_count_hist(const uint32_t *fcnt, int64_t n, uint32_t *hist, int num_sms, cudaStream_t s);
int count_hist_bins();
void launch_tie_keyhist(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                        uint32_t unit, uint32_t *hist, int num_sms, cudaStream_t s);
void launch_tie_bin_collect(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t key0, int32_t W, int kshift,
                            int64_t bstar, unsigned long long *out, int32_t *out_n, int32_t cap, cudaStream_t s);
void launch_select_bits(const uint32_t *fcnt, int64_t n, uint32_t cstar, int64_t kcut, int64_t key0, int32_t W,
                        uint32_t *bits, int num_sms, cudaStream_t s);
void launch_bits_compact(const uint32_t *bits, int64_t nw, int32_t *blk, int32_t *total, unsigned long long *keys,
                         int32_t kmax, cudaStream_t s);
void launch_hot_layout(const unsigned long long *keys, int32_t k, const int64_t *pack_key_off, int32_t P,
                       int32_t *pslot, cudaStream_t s);
void launch_stage_idx(const int32_t *pslot, const int64_t *stage_off, const int32_t *pack_dim, int32_t P, int nst,
                      int32_t k, int64_t *stage_idx, cudaStream_t s);
void launch_pack_owned(int D, const MultiArgs &m, int pack, const unsigned long long *keys, const int64_t *stage_idx,
                       const float *w, const float *s1, const float *s2, int nst, float *stage, int rank, int num_sms,
                       cudaStream_t s);
void launch_place(int D, const MultiArgs &m, int pack, const int64_t *stage_idx, const float *stage, int nst,
                  int num_sms, cudaStream_t s);
void launch_hot_index(Slot *index, uint32_t mask, const unsigned long long *keys, int32_t k, cudaStream_t s);
}  // namespace picasso

namespace {

int nst_of(const picasso_ctx *ctx) { return ctx->opts.opt == PICASSO_OPT_ADAM_LAZY ? 2 : 1; }

int pack_of_key(const picasso_ctx *ctx, unsigned long long gkey) {
    int p = 0;
    while (p + 1 < ctx->P && (unsigned long long)ctx->pack_key_off[p + 1] <= gkey) ++p;
    return p;
}

// step 1b (after the counts AllReduce): write replicas back, merge counts, drop the hot set
picasso_status refresh_writeback(picasso_ctx *ctx, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    if (mp.hot_k == 0) return PICASSO_OK;
    MultiArgs m = picasso_multi_args(ctx);
    const int nst = 1 + nst_of(ctx);  // weights + state arrays
    for (int p = 0; p < ctx->P; ++p)
        if (mp.hot_pslot[p + 1] > mp.hot_pslot[p])
            launch_writeback(ctx->pack_dim[p], m, p, mp.hot_keys, ctx->w[p], ctx->s1[p], ctx->s2[p], nst, mp.cnt_sum,
                             ctx->rank, ctx->num_sms, s);
    HCK(cudaMemsetAsync(mp.hot_cnt, 0, sizeof(uint32_t) * std::max<int64_t>(mp.k_max, 1), s));
    mp.hot_k = 0;
    launch_hot_index(mp.hot_index, mp.hot_mask, mp.hot_keys, 0, s);
    return PICASSO_OK;
}

// ---- the ranks of one refresh: NCCL (one local ctx) or the loopback group (all ctxs here) ----
struct Ranks {
    std::vector<picasso_ctx *> cs;  // the ctxs this process drives
    ncclComm_t comm = nullptr;      // NCCL mode
};

// sum of a u32 buffer over the ranks, into every rank's copy (the same buffer of each ctx)
template <typename F>
picasso_status allreduce_u32(const Ranks &R, F buf, int64_t n, cudaStream_t s) {
    picasso_ctx *ctx = R.cs[0];
    if (n <= 0) return PICASSO_OK;
    if (R.comm) {
        HNK(ncclAllReduce(buf(ctx), buf(ctx), (size_t)n, ncclUint32, ncclSum, R.comm, s));
        return PICASSO_OK;
    }
    RankPtrs pc{};
    const int W = (int)R.cs.size();
    for (int r = 0; r < W; ++r) pc.p[r] = buf(R.cs[r]);
    launch_sum_ranks_u32(pc, W, buf(ctx), n, s);  // in place into rank 0 (element-wise), then copies
    for (int r = 1; r < W; ++r)
        HCK(cudaMemcpyAsync(buf(R.cs[r]), buf(ctx), sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    return PICASSO_OK;
}

int64_t key_space(const picasso_ctx *ctx) { return ctx->pack_key_off[ctx->P]; }

// steps 2-4 (capacity > 0); identical decisions on every rank
picasso_status refresh_select_all(const Ranks &R, size_t capacity, cudaStream_t s, double *t_threshold) {
    using clk = std::chrono::steady_clock;
    static const bool trace = std::getenv("PICASSO_REFRESH_TRACE") != nullptr;  // measurement aid
    auto tlast = clk::now();
    auto mark = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        const auto t = clk::now();
        std::fprintf(stderr, "[refresh r%d] %-22s %9.3f ms\n", R.cs[0]->rank, what,
                     std::chrono::duration<double, std::milli>(t - tlast).count());
        tlast = t;
    };
    mark("(queued work)");
    const auto t0 = clk::now();
    picasso_ctx *ctx = R.cs[0];
    picasso_status st;
    const int P = ctx->P, W = ctx->world, nst = 1 + nst_of(ctx), bins = count_hist_bins();
    std::vector<int64_t> unit(P);  // 16-byte units of one hot row (weights + state) per pack
    for (int p = 0; p < P; ++p) unit[p] = (int64_t)ctx->pack_dim[p] * nst / 4;
    const int64_t cap_units = (int64_t)(capacity / 16);
    // 2a. per-pack count histograms of the owned rows, summed over the ranks
    for (picasso_ctx *c : R.cs)
        for (int p = 0; p < P; ++p)
            launch_count_hist(c->mp.fcnt + c->mp.fcnt_off[p], c->mp.fcnt_off[p + 1] - c->mp.fcnt_off[p],
                              c->mp.phist + (size_t)p * bins, c->num_sms, s);
    mark("count histograms");
    if ((st = allreduce_u32(R, [](picasso_ctx *c) { return c->mp.phist; }, (int64_t)P * bins, s))) return st;
    mark("histogram allreduce");
    std::vector<uint32_t> h((size_t)P * bins);
    HCK(cudaMemcpyAsync(h.data(), ctx->mp.phist, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    // 2b. c*: the count at which the (count desc) order reaches the capacity
    auto units_at = [&](int b) {
        int64_t u = 0;
        for (int p = 0; p < P; ++p) u += (int64_t)h[(size_t)p * bins + b] * unit[p];
        return u;
    };
    uint32_t cstar = 0;
    int64_t kcut = INT64_MAX, above = 0;
    int b = bins - 1;
    for (; b >= 1; --b) {
        const int64_t u = units_at(b);
        if (above + u > cap_units) break;
        above += u;
    }
    if (b >= 1) {  // rows at count b only partly fit: cut them in ascending key
        cstar = (uint32_t)b;
        const int64_t rem = cap_units - above;
        const int64_t KT = key_space(ctx);
        int kbits = 1;
        while (kbits < 40 && ((int64_t)1 << kbits) < KT) ++kbits;
        const int kshift = std::max(0, kbits - 16);
        const int64_t nkb = (KT >> kshift) + 1;
        for (picasso_ctx *c : R.cs) {
            HCK(cudaMemsetAsync(c->mp.khist, 0, sizeof(uint32_t) * nkb, s));
            for (int p = 0; p < P; ++p)
                launch_tie_keyhist(c->mp.fcnt + c->mp.fcnt_off[p], c->mp.fcnt_off[p + 1] - c->mp.fcnt_off[p], cstar,
                                   ctx->pack_key_off[p] + c->rank, W, kshift, (uint32_t)unit[p], c->mp.khist,
                                   c->num_sms, s);
        }
        mark("tie key histogram");
        if ((st = allreduce_u32(R, [](picasso_ctx *c) { return c->mp.khist; }, nkb, s))) return st;
        mark("tie allreduce");
        std::vector<uint32_t> kh(nkb);
        HCK(cudaMemcpyAsync(kh.data(), ctx->mp.khist, sizeof(uint32_t) * nkb, cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        int64_t acc = 0, bstar = 0;
        for (; bstar < nkb; ++bstar) {
            if (acc + (int64_t)kh[bstar] > rem) break;
            acc += kh[bstar];
        }
        kcut = (bstar << kshift) - 1;  // every tie key below bin b* fits
        if (bstar < nkb) {           // inside b*: the tie keys themselves, in ascending order
            const int32_t tcap = (int32_t)(((int64_t)1 << kshift) / W + 2);
            std::vector<unsigned long long> keys;
            for (picasso_ctx *c : R.cs) {
                HCK(cudaMemsetAsync(c->mp.tie_n, 0, sizeof(int32_t), s));
                for (int p = 0; p < P; ++p)
                    launch_tie_bin_collect(c->mp.fcnt + c->mp.fcnt_off[p], c->mp.fcnt_off[p + 1] - c->mp.fcnt_off[p],
                                           cstar, ctx->pack_key_off[p] + c->rank, W, kshift, bstar,
                                           c->mp.tie_keys + (size_t)c->rank * tcap, c->mp.tie_n, tcap, s);
                if (R.comm) {  // [W, tcap] keys + [W] counts on every rank
                    HCK(cudaMemcpyAsync(c->mp.tie_keys + (size_t)W * tcap + c->rank, c->mp.tie_n, sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, s));
                    HNK(ncclGroupStart());
                    HNK(ncclAllGather(c->mp.tie_keys + (size_t)c->rank * tcap, c->mp.tie_keys, tcap, ncclUint64,
                                      R.comm, s));
                    HNK(ncclAllGather(reinterpret_cast<int32_t *>(c->mp.tie_keys + (size_t)W * tcap) + c->rank,
                                      reinterpret_cast<int32_t *>(c->mp.tie_keys + (size_t)W * tcap), 1, ncclInt32,
                                      R.comm, s));
                    HNK(ncclGroupEnd());
                    std::vector<unsigned long long> all((size_t)W * tcap);
                    std::vector<int32_t> cnt(W);
                    HCK(cudaMemcpyAsync(all.data(), c->mp.tie_keys, sizeof(unsigned long long) * all.size(),
                                        cudaMemcpyDeviceToHost, s));
                    HCK(cudaMemcpyAsync(cnt.data(), c->mp.tie_keys + (size_t)W * tcap, sizeof(int32_t) * W,
                                        cudaMemcpyDeviceToHost, s));
                    HCK(cudaStreamSynchronize(s));
                    for (int r = 0; r < W; ++r)
                        keys.insert(keys.end(), all.begin() + (size_t)r * tcap,
                                    all.begin() + (size_t)r * tcap + std::min(cnt[r], tcap));
                } else {
                    int32_t n = 0;
                    HCK(cudaMemcpyAsync(&n, c->mp.tie_n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                    HCK(cudaStreamSynchronize(s));
                    std::vector<unsigned long long> mine(std::min(n, tcap));
                    HCK(cudaMemcpy(mine.data(), c->mp.tie_keys + (size_t)c->rank * tcap,
                                   sizeof(unsigned long long) * mine.size(), cudaMemcpyDeviceToHost));
                    keys.insert(keys.end(), mine.begin(), mine.end());
                }
            }
            mark("tie bin keys");
            std::sort(keys.begin(), keys.end());
            for (unsigned long long k : keys) {
                int p = 0;
                while (p + 1 < P && (unsigned long long)ctx->pack_key_off[p + 1] <= k) ++p;
                if (acc + unit[p] > rem) break;  // the longest prefix that fits (oracle_hot_select)
                acc += unit[p];
                kcut = (int64_t)k;
            }
        }
    }
    if (t_threshold) *t_threshold = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    // 3. the selection bitmap over the global key space, summed over the ranks; hot keys
    const int64_t nw = key_space(ctx) / 32 + 1;
    for (picasso_ctx *c : R.cs) {
        HCK(cudaMemsetAsync(c->mp.sel_bits, 0, sizeof(uint32_t) * nw, s));
        for (int p = 0; p < P; ++p)
            launch_select_bits(c->mp.fcnt + c->mp.fcnt_off[p], c->mp.fcnt_off[p + 1] - c->mp.fcnt_off[p], cstar, kcut,
                               ctx->pack_key_off[p] + c->rank, W, c->mp.sel_bits, c->num_sms, s);
    }
    mark("selection bits");
    if ((st = allreduce_u32(R, [](picasso_ctx *c) { return c->mp.sel_bits; }, nw, s))) return st;
    mark("bits allreduce");
    for (picasso_ctx *c : R.cs) {
        MultiState &mp = c->mp;
        launch_bits_compact(mp.sel_bits, nw, mp.bits_blk, mp.bits_blk + nw / 1024 + 1, mp.hot_keys,
                            (int32_t)mp.k_max, s);
        int32_t k = 0;
        HCK(cudaMemcpyAsync(&k, mp.bits_blk + nw / 1024 + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        if (k > mp.k_max) {
            c->last_msg = "hot set larger than the workspace's k_max";
            return PICASSO_ERR_CAPACITY;
        }
        launch_hot_layout(mp.hot_keys, k, c->pack_key_off_d, P, mp.hot_pslot_d, s);
        mp.hot_pslot.assign(P + 1, 0);
        HCK(cudaMemcpyAsync(mp.hot_pslot.data(), mp.hot_pslot_d, sizeof(int32_t) * (P + 1), cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        // replica arena (per pack: w, s1, s2 blocks) + G offsets; slot-major staging
        mp.hot_off.assign(4 * P, 0);
        std::vector<int64_t> soff(P);
        int64_t cur = 0, g = 0, so = 0;
        for (int p = 0; p < P; ++p) {
            const int64_t kp = mp.hot_pslot[p + 1] - mp.hot_pslot[p], D = c->pack_dim[p];
            mp.hot_off[p] = cur;
            cur += kp * D;
            mp.hot_off[P + p] = cur;
            cur += kp * D;
            mp.hot_off[2 * P + p] = nst == 3 ? cur : mp.hot_off[P + p];
            if (nst == 3) cur += kp * D;
            mp.hot_off[3 * P + p] = g;
            g += kp * D;
            soff[p] = so;
            so += kp * D * nst;
        }
        mp.hot_g_floats = g;
        mp.stage_floats = so;
        HCK(cudaMemcpyAsync(mp.hot_off_d, mp.hot_off.data(), sizeof(int64_t) * 4 * P, cudaMemcpyHostToDevice, s));
        HCK(cudaMemcpyAsync(mp.stage_off_d, soff.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, s));
        launch_stage_idx(mp.hot_pslot_d, mp.stage_off_d, c->pack_dim_d, P, nst, k, mp.stage_idx, s);
        HCK(cudaStreamSynchronize(s));  // soff goes out of scope
        mp.new_k = k;
        // 4. owners write their new hot rows into the staging (others' slots stay zero)
        HCK(cudaMemsetAsync(mp.stage, 0, sizeof(float) * std::max<int64_t>(so, 1), s));
        MultiArgs m = picasso_multi_args(c);
        for (int p = 0; p < P; ++p)
            if (mp.hot_pslot[p + 1] > mp.hot_pslot[p])
                launch_pack_owned(c->pack_dim[p], m, p, mp.hot_keys, mp.stage_idx, c->w[p], c->s1[p], c->s2[p], nst,
                                  mp.stage, c->rank, c->num_sms, s);
    }
    mark("compact + stage");
    st = allreduce_u32(R, [](picasso_ctx *c) { return reinterpret_cast<uint32_t *>(c->mp.stage); },
                       ctx->mp.stage_floats, s);
    mark("stage allreduce");
    return st;
}

// step 4b: staging (all owners' blocks now present) -> replicas; index; counters
picasso_status refresh_place(picasso_ctx *ctx, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int nst = 1 + nst_of(ctx);
    MultiArgs m = picasso_multi_args(ctx);
    for (int p = 0; p < ctx->P; ++p)
        if (mp.hot_pslot[p + 1] > mp.hot_pslot[p])
            launch_place(ctx->pack_dim[p], m, p, mp.stage_idx, mp.stage, nst, ctx->num_sms, s);
    launch_hot_index(mp.hot_index, mp.hot_mask, mp.hot_keys, mp.new_k, s);
    HCK(cudaMemsetAsync(mp.hot_cnt, 0, sizeof(uint32_t) * std::max<int64_t>(mp.k_max, 1), s));
    mp.hot_k = mp.new_k;
    HCK(cudaGetLastError());
    return PICASSO_OK;
}

void fill_stats(picasso_ctx *ctx, picasso_cache_stats *st) {
    if (!st) return;
    p2p_host_counts(ctx);
    MultiState &mp = ctx->mp;
    st->k = mp.hot_k;
    int64_t bytes = 0;
    for (int p = 0; p < ctx->P && !mp.hot_pslot.empty(); ++p)
        bytes += (int64_t)(mp.hot_pslot[p + 1] - mp.hot_pslot[p]) * 4 * ctx->pack_dim[p] * (1 + nst_of(ctx));
    st->bytes = mp.hot_k ? bytes : 0;
    st->hot_uniques = mp.last_hot_uniques;
    st->uniques = mp.last_uniques;
    st->hit_ratio_unique = mp.last_uniques ? (double)mp.last_hot_uniques / (double)mp.last_uniques : 0.0;
}

picasso_status check_refresh_args(picasso_ctx *ctx, size_t capacity) {
    if (!ctx->bound) return PICASSO_ERR_STATE;
    if (ctx->opts.cache_max_bytes <= 0) return capacity ? PICASSO_ERR_CAPACITY : PICASSO_OK;
    if ((int64_t)capacity > ctx->opts.cache_max_bytes) return PICASSO_ERR_CAPACITY;
    return PICASSO_OK;
}

}  // namespace

// ---- NCCL: one rank per process -----------------------------------------------------------
picasso_status ct_refresh(picasso_ctx *ctx, size_t capacity, cudaStream_t s, picasso_cache_stats *stats);  // coldtier.cu
picasso_status ct_hot_keys(picasso_ctx *ctx, int32_t *pack, int64_t *key, int64_t cap, int64_t *n);

extern "C" picasso_status picasso_hot_cache_refresh(picasso_ctx *ctx, size_t capacity_bytes, void *stream,
                                                    picasso_cache_stats *stats) {
    NvtxRange nvtx("picasso_hot_cache_refresh");
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    picasso_status st = check_refresh_args(ctx, capacity_bytes);
    if (st) return st;
    if (ctx->world == 1 && ctx->opts.cold_tier) return ct_refresh(ctx, capacity_bytes, s, stats);  // host-DRAM tier
    if (ctx->world == 1 || ctx->opts.cache_max_bytes <= 0) {  // no shard to skip: the table is the hot storage
        if (stats) *stats = picasso_cache_stats{0, 0, 0, 0, 0.0};
        return PICASSO_OK;
    }
    if (ctx->mp.group || !ctx->mp.comm) return PICASSO_ERR_STATE;
    MultiState &mp = ctx->mp;
    using clk = std::chrono::steady_clock;
    HCK(cudaStreamSynchronize(s));  // the steps queued before it are not the refresh's cost
    const auto t0 = clk::now();
    auto t1 = t0, t2 = t0;
    if (mp.hot_k > 0)
        HNK(ncclAllReduce(mp.hot_cnt, mp.cnt_sum, mp.hot_k, ncclUint32, ncclSum, mp.comm, s));
    if ((st = refresh_writeback(ctx, s))) return st;
    double t_thr = 0.0;
    if (capacity_bytes > 0) {
        Ranks R;
        R.cs = {ctx};
        R.comm = mp.comm;
        if ((st = refresh_select_all(R, capacity_bytes, s, &t_thr))) return st;
        t1 = t0 + std::chrono::duration_cast<clk::duration>(std::chrono::duration<double, std::milli>(t_thr));
        t2 = clk::now();
        if ((st = refresh_place(ctx, s))) return st;
    }
    HCK(cudaStreamSynchronize(s));
    fill_stats(ctx, stats);
    if (stats) {
        const auto t3 = clk::now();
        stats->refresh_ms = std::chrono::duration<double, std::milli>(t3 - t0).count();
        stats->propose_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        stats->select_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    }
    return PICASSO_OK;
}

// ---- loopback group -------------------------------------------------------------------------
extern "C" picasso_status picasso_group_hot_cache_refresh(picasso_group *g, size_t capacity_bytes, void *stream,
                                                          picasso_cache_stats *stats) {
    if (!g || g->ctx.empty()) return PICASSO_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int W = (int)g->ctx.size();
    picasso_ctx *ctx = g->ctx[0];
    picasso_status st;
    for (auto *c : g->ctx)
        if ((st = check_refresh_args(c, capacity_bytes))) return st;
    if (ctx->opts.cache_max_bytes <= 0) return PICASSO_OK;
    if (ctx->mp.hot_k > 0) {  // AllReduce of the hit counts: rank-order sum into every rank
        RankPtrs pc{};
        for (int r = 0; r < W; ++r) pc.p[r] = g->ctx[r]->mp.hot_cnt;
        launch_sum_ranks_u32(pc, W, ctx->mp.cnt_sum + ctx->mp.k_max, ctx->mp.hot_k, s);
        for (int r = 0; r < W; ++r)
            HCK(cudaMemcpyAsync(g->ctx[r]->mp.cnt_sum, ctx->mp.cnt_sum + ctx->mp.k_max,
                                sizeof(uint32_t) * ctx->mp.hot_k, cudaMemcpyDeviceToDevice, s));
    }
    for (auto *c : g->ctx)
        if ((st = refresh_writeback(c, s))) return st;
    if (capacity_bytes > 0) {
        Ranks R;
        R.cs = g->ctx;
        if ((st = refresh_select_all(R, capacity_bytes, s, nullptr))) return st;
        for (auto *c : g->ctx)
            if ((st = refresh_place(c, s))) return st;
    }
    for (int r = 0; r < W; ++r) fill_stats(g->ctx[r], stats ? stats + r : nullptr);
    return PICASSO_OK;
}

extern "C" picasso_status picasso_get_hot_keys(picasso_ctx *ctx, int32_t *pack, int64_t *key, int64_t cap,
                                               int64_t *n) {
    if (!ctx || !n) return PICASSO_ERR_INVALID_ARG;
    if (ctx->opts.cold_tier) return ct_hot_keys(ctx, pack, key, cap, n);
    MultiState &mp = ctx->mp;
    *n = mp.hot_k;
    if (mp.hot_k == 0 || !pack || !key) return PICASSO_OK;
    if (cudaStreamSynchronize(ctx->last_stream) != cudaSuccess) return PICASSO_ERR_CUDA;
    std::vector<unsigned long long> k(mp.hot_k);
    if (cudaMemcpy(k.data(), mp.hot_keys, sizeof(unsigned long long) * mp.hot_k, cudaMemcpyDeviceToHost) != cudaSuccess)
        return PICASSO_ERR_CUDA;
    for (int64_t i = 0; i < std::min<int64_t>(cap, mp.hot_k); ++i) {
        const int p = pack_of_key(ctx, k[i]);
        pack[i] = p;
        key[i] = (int64_t)(k[i] - (unsigned long long)ctx->pack_key_off[p]);
    }
    return PICASSO_OK;
}
