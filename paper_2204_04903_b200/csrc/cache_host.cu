// cache_host.cu — picasso_hot_cache_refresh: Alg. 1 L514-517 on the row-sharded step.
//
//   1. replicas -> owners' shards; the ranks' hot-hit counts are summed (AllReduce) and added
//      to the owners' FCounter;
//   2. each owner proposes its local top-kc rows by (count desc, key asc) — kc = the most rows
//      the capacity can hold — found with a count histogram, a threshold and an ordered tie
//      cut, so the union of proposals contains the global top-k;
//   3. the proposals are gathered; every rank merges them on the host in the same
//      deterministic order and keeps the longest prefix whose rows (weights + optimizer state)
//      fit the capacity (readings O12/O13; equals oracle_hot_select);
//   4. owners pack their new hot rows, every rank receives every owner's block (broadcasts),
//      places the rows into its replica arena and rebuilds the key -> slot index.
// capacity_bytes = 0 writes back and drops the hot set (checkpoint / disable).
#include <chrono>

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
void launch_tie_count(const uint32_t *fcnt, int64_t n, uint32_t cstar, int32_t *tile_cnt, cudaStream_t s);
void launch_collect(const uint32_t *fcnt, int64_t n, uint32_t cstar, int32_t m_ties, const int32_t *tile_off,
                    const int64_t *row_key, int32_t nseg, const int64_t *seg_start, unsigned long long *out_key,
                    uint32_t *out_cnt, int32_t *out_n, cudaStream_t s);
void launch_pack_owned(int D, const MultiArgs &m, int pack, const unsigned long long *keys, const int32_t *stage_idx,
                       const float *w, const float *s1, const float *s2, int nst, float *stage, int rank, int num_sms,
                       cudaStream_t s);
void launch_place(int D, const MultiArgs &m, int pack, const int32_t *stage_idx, const float *stage, int nst,
                  int num_sms, cudaStream_t s);
void launch_hot_index(Slot *index, uint32_t mask, const unsigned long long *keys, int32_t k, cudaStream_t s);
}  // namespace picasso

namespace {

struct Cand {
    uint32_t cnt;
    unsigned long long key;
};

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

// step 2: this owner's proposals (host vector), kc = most rows the capacity can hold
picasso_status refresh_propose(picasso_ctx *ctx, int64_t kc, std::vector<Cand> &out, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int64_t n = mp.rows_total;
    out.clear();
    if (kc <= 0 || n == 0) return PICASSO_OK;
    const int bins = count_hist_bins();
    launch_count_hist(mp.fcnt, n, mp.cnt_hist, ctx->num_sms, s);
    std::vector<uint32_t> h(bins);
    HCK(cudaMemcpyAsync(h.data(), mp.cnt_hist, sizeof(uint32_t) * bins, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    // cstar: the kc-th largest count; above it all rows are taken, at it the first m_ties
    int64_t above = 0;
    uint32_t cstar = 0;
    int64_t m_ties = 0;
    for (int c = bins - 1; c >= 1; --c) {
        if (above + h[c] >= kc) {
            cstar = (uint32_t)c;
            m_ties = kc - above;
            break;
        }
        above += h[c];
    }
    if (cstar == 0) {  // fewer than kc rows were ever counted: propose all of them
        cstar = 1;
        m_ties = h[1];
        above -= h[1];
    }
    const int64_t ntile = (n + kTile - 1) / kTile;
    launch_tie_count(mp.fcnt, n, cstar, mp.tie_cnt, s);
    launch_scan_exclusive(mp.tie_cnt, mp.tie_cnt, ntile, ctx->hot_scan_scratch, nullptr, s);
    std::vector<int64_t> rk(2 * ctx->P), seg(ctx->P + 1);
    for (int p = 0; p < ctx->P; ++p) {
        rk[2 * p] = ctx->pack_key_off[p] + ctx->rank;  // global key of local row lr: rk0 + lr * W
        rk[2 * p + 1] = ctx->world;
        seg[p] = mp.fcnt_off[p];
    }
    seg[ctx->P] = mp.fcnt_off[ctx->P];
    HCK(cudaMemcpyAsync(mp.row_key_d, rk.data(), sizeof(int64_t) * 2 * ctx->P, cudaMemcpyHostToDevice, s));
    HCK(cudaMemcpyAsync(mp.fcnt_off_d, seg.data(), sizeof(int64_t) * (ctx->P + 1), cudaMemcpyHostToDevice, s));
    HCK(cudaMemsetAsync(mp.cand_n, 0, sizeof(int32_t), s));
    launch_collect(mp.fcnt, n, cstar, (int32_t)m_ties, mp.tie_cnt, mp.row_key_d, ctx->P, mp.fcnt_off_d, mp.cand_key,
                   mp.cand_cnt, mp.cand_n, s);
    int32_t nc = 0;
    HCK(cudaMemcpyAsync(&nc, mp.cand_n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    nc = std::min<int32_t>(nc, (int32_t)mp.k_max);
    std::vector<unsigned long long> k(nc);
    std::vector<uint32_t> c(nc);
    HCK(cudaMemcpy(k.data(), mp.cand_key, sizeof(unsigned long long) * nc, cudaMemcpyDeviceToHost));
    HCK(cudaMemcpy(c.data(), mp.cand_cnt, sizeof(uint32_t) * nc, cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < nc; ++i) out.push_back({c[i], k[i]});
    return PICASSO_OK;
}

// step 3 + layout: identical on every rank given the same proposals
picasso_status refresh_select(picasso_ctx *ctx, std::vector<Cand> all, size_t capacity, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int P = ctx->P, W = ctx->world, nst = 1 + nst_of(ctx);
    std::sort(all.begin(), all.end(), [](const Cand &a, const Cand &b) {
        if (a.cnt != b.cnt) return a.cnt > b.cnt;
        return a.key < b.key;  // (pack asc, key asc) == global key asc
    });
    std::vector<std::vector<unsigned long long>> by_pack(P);
    uint64_t used = 0;
    for (const Cand &c : all) {
        const int p = pack_of_key(ctx, c.key);
        const uint64_t cost = (uint64_t)4 * ctx->pack_dim[p] * nst;
        if (used + cost > capacity) break;  // longest prefix that fits (oracle_hot_select)
        used += cost;
        by_pack[p].push_back(c.key);
    }
    std::vector<unsigned long long> keys;
    mp.hot_pslot.assign(P + 1, 0);
    mp.hot_off.assign(4 * P, 0);
    int64_t cur = 0, g = 0;
    for (int p = 0; p < P; ++p) {
        mp.hot_pslot[p] = (int32_t)keys.size();
        keys.insert(keys.end(), by_pack[p].begin(), by_pack[p].end());
        const int64_t kp = (int64_t)by_pack[p].size(), D = ctx->pack_dim[p];
        mp.hot_off[p] = cur;
        cur += kp * D;
        mp.hot_off[P + p] = cur;
        cur += kp * D;
        mp.hot_off[2 * P + p] = nst == 3 ? cur : mp.hot_off[P + p];
        if (nst == 3) cur += kp * D;
        mp.hot_off[3 * P + p] = g;
        g += kp * D;
    }
    mp.hot_pslot[P] = (int32_t)keys.size();
    mp.hot_g_floats = g;
    const int32_t k = (int32_t)keys.size();
    // staging: owner-major blocks, each owned slot's w|s1|s2 rows in slot order
    std::vector<int32_t> sidx(k);
    std::vector<int64_t> blk(W + 1, 0);
    int64_t off = 0;
    for (int o = 0; o < W; ++o) {
        blk[o] = off;
        for (int p = 0; p < P; ++p)
            for (int32_t sl = mp.hot_pslot[p]; sl < mp.hot_pslot[p + 1]; ++sl)
                if ((int64_t)((keys[sl] - (unsigned long long)ctx->pack_key_off[p]) % W) == o) {
                    sidx[sl] = (int32_t)off;
                    off += (int64_t)nst * ctx->pack_dim[p];
                }
    }
    blk[W] = off;
    mp.stage_blk = blk;
    if (k > 0) {
        HCK(cudaMemcpyAsync(mp.hot_keys, keys.data(), sizeof(unsigned long long) * k, cudaMemcpyHostToDevice, s));
        HCK(cudaMemcpyAsync(mp.stage_idx, sidx.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, s));
    }
    HCK(cudaMemcpyAsync(mp.hot_pslot_d, mp.hot_pslot.data(), sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice, s));
    HCK(cudaMemcpyAsync(mp.hot_off_d, mp.hot_off.data(), sizeof(int64_t) * 4 * P, cudaMemcpyHostToDevice, s));
    HCK(cudaStreamSynchronize(s));  // the host vectors above go out of scope
    mp.new_k = k;
    // owners pack their new hot rows into the staging
    MultiArgs m = picasso_multi_args(ctx);
    for (int p = 0; p < P; ++p)
        if (mp.hot_pslot[p + 1] > mp.hot_pslot[p])
            launch_pack_owned(ctx->pack_dim[p], m, p, mp.hot_keys, mp.stage_idx, ctx->w[p], ctx->s1[p], ctx->s2[p],
                              nst, mp.stage, ctx->rank, ctx->num_sms, s);
    return PICASSO_OK;
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

int64_t kc_for(picasso_ctx *ctx, size_t capacity) {
    int minD = 1 << 30;
    for (int p = 0; p < ctx->P; ++p) minD = std::min(minD, ctx->pack_dim[p]);
    return std::min<int64_t>(ctx->mp.k_max, (int64_t)(capacity / ((size_t)4 * minD * (1 + nst_of(ctx)))));
}

}  // namespace

// ---- NCCL: one rank per process -----------------------------------------------------------
picasso_status ct_refresh(picasso_ctx *ctx, size_t capacity, cudaStream_t s, picasso_cache_stats *stats);  // coldtier.cu
picasso_status ct_hot_keys(picasso_ctx *ctx, int32_t *pack, int64_t *key, int64_t cap, int64_t *n);

extern "C" picasso_status picasso_hot_cache_refresh(picasso_ctx *ctx, size_t capacity_bytes, void *stream,
                                                    picasso_cache_stats *stats) {
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
    const auto t0 = clk::now();
    auto t1 = t0, t2 = t0;
    if (mp.hot_k > 0)
        HNK(ncclAllReduce(mp.hot_cnt, mp.cnt_sum, mp.hot_k, ncclUint32, ncclSum, mp.comm, s));
    if ((st = refresh_writeback(ctx, s))) return st;
    if (capacity_bytes > 0) {
        const int64_t kc = kc_for(ctx, capacity_bytes);
        std::vector<Cand> mine;
        if ((st = refresh_propose(ctx, kc, mine, s))) return st;
        t1 = clk::now();
        // gather the proposals: fixed kc records per rank (count 0 = padding)
        const int W = ctx->world;
        std::vector<unsigned long long> kk(kc, 0ull);
        std::vector<uint32_t> cc(kc, 0u);
        for (size_t i = 0; i < mine.size(); ++i) {
            kk[i] = mine[i].key;
            cc[i] = mine[i].cnt;
        }
        // in-place AllGather: this rank's records at slot `rank` of the [W, kc] arrays
        HCK(cudaMemcpy(mp.cand_key + (size_t)ctx->rank * kc, kk.data(), sizeof(unsigned long long) * kc,
                       cudaMemcpyHostToDevice));
        HCK(cudaMemcpy(mp.cand_cnt + (size_t)ctx->rank * kc, cc.data(), sizeof(uint32_t) * kc, cudaMemcpyHostToDevice));
        HNK(ncclGroupStart());
        HNK(ncclAllGather(mp.cand_key + (size_t)ctx->rank * kc, mp.cand_key, kc, ncclUint64, mp.comm, s));
        HNK(ncclAllGather(mp.cand_cnt + (size_t)ctx->rank * kc, mp.cand_cnt, kc, ncclUint32, mp.comm, s));
        HNK(ncclGroupEnd());
        std::vector<unsigned long long> ak((size_t)kc * W);
        std::vector<uint32_t> ac((size_t)kc * W);
        HCK(cudaMemcpyAsync(ak.data(), mp.cand_key, sizeof(unsigned long long) * kc * W, cudaMemcpyDeviceToHost, s));
        HCK(cudaMemcpyAsync(ac.data(), mp.cand_cnt, sizeof(uint32_t) * kc * W, cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        std::vector<Cand> all;
        for (size_t i = 0; i < ak.size(); ++i)
            if (ac[i] > 0) all.push_back({ac[i], ak[i]});
        if ((st = refresh_select(ctx, all, capacity_bytes, s))) return st;
        t2 = clk::now();
        HNK(ncclGroupStart());
        for (int o = 0; o < W; ++o) {
            const int64_t n = mp.stage_blk[o + 1] - mp.stage_blk[o];
            if (n > 0)
                HNK(ncclBroadcast(mp.stage + mp.stage_blk[o], mp.stage + mp.stage_blk[o], n, ncclFloat32, o, mp.comm, s));
        }
        HNK(ncclGroupEnd());
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
        std::vector<Cand> all;
        for (auto *c : g->ctx) {
            std::vector<Cand> mine;
            if ((st = refresh_propose(c, kc_for(c, capacity_bytes), mine, s))) return st;
            all.insert(all.end(), mine.begin(), mine.end());
        }
        for (auto *c : g->ctx)
            if ((st = refresh_select(c, all, capacity_bytes, s))) return st;
        for (int o = 0; o < W; ++o) {  // owner o's block to every other rank
            picasso_ctx *src = g->ctx[o];
            const int64_t off = src->mp.stage_blk[o], n = src->mp.stage_blk[o + 1] - off;
            for (int r = 0; r < W; ++r)
                if (r != o && n > 0)
                    HCK(cudaMemcpyAsync(g->ctx[r]->mp.stage + off, src->mp.stage + off, sizeof(float) * n,
                                        cudaMemcpyDeviceToDevice, s));
        }
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
