// ctx.h — the context object behind the C ABI (internal).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a tool is attached

#include "kernels.h"
#include "multi.h"
#include "p2p.h"
#include "picasso.h"

using namespace picasso;

namespace ctxutil {

constexpr size_t kAlign = 256;

struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(size_t n) {
        off = (off + kAlign - 1) / kAlign * kAlign;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += n * sizeof(T);
        return p;
    }
};

inline uint64_t pow2_at_least(uint64_t x) {
    uint64_t p = 1024;
    while (p < x) p <<= 1;
    return p;
}

inline int bits_for(int64_t maxval) {
    int b = 1;
    while (b < 31 && ((int64_t)1 << b) <= maxval) ++b;
    return b;
}

}  // namespace ctxutil
using namespace ctxutil;

// NVTX range over one ABI call (Nsight timelines: picasso_fwd / picasso_bwd_update / picasso_refresh)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct picasso_group;

// Per-rank state of the row-sharded step (world > 1), host side.
struct MultiState {
    bool reset_forked = false;  // p2p: this forward's dtab reset runs on side2 (joined in p2p_c)
    ncclComm_t comm = nullptr;       // NCCL mode
    picasso_group *group = nullptr;  // loopback mode (all ranks in one process)
    int64_t max_recv = 0;
    // device
    int32_t *bkey = nullptr, *bval = nullptr, *bsorted = nullptr, *send_uid = nullptr, *bhist = nullptr,
            *bcount = nullptr;
    int64_t *bstart = nullptr, *sroff = nullptr;
    int32_t *send_pos = nullptr, *send_keys = nullptr;
    int64_t *row_off = nullptr;
    int32_t *cnt_recv_d = nullptr;   // [W*P] counts this rank receives, (source, pack)
    int32_t *recv_keys = nullptr, *opos_map = nullptr, *oslot = nullptr, *oinv = nullptr;
    unsigned long long *ouid_key = nullptr;
    int32_t *opack_gstart = nullptr, *opack_ustart = nullptr, *od_total = nullptr, *oblk_cnt = nullptr,
            *oblk_off = nullptr;
    int64_t *opack_ostart_d = nullptr, *ogbase_scratch = nullptr;
    OwnerBlock *oblk_d = nullptr;
    int32_t *contrib = nullptr;
    int64_t *rsend_off = nullptr;
    float *rows_send = nullptr;
    // host (pinned staging for the counts / block tables)
    int32_t *cnt_send_h = nullptr, *cnt_recv_h = nullptr;
    OwnerBlock *oblk_h = nullptr;
    int32_t *og_h = nullptr;
    uint8_t uid[128] = {0};
    bool has_uid = false;
    int64_t *ostart_h = nullptr;
    std::vector<int64_t> skoff, sk, rkoff, rk, srow_off, srow_n, rrow_off, rrow_n;  // per peer
    int64_t R = 0, U_send = 0;
    std::vector<int64_t> opack_ostart;  // [P+1]
    // ---- HybridHash (cache.cu / cache_host.cu)
    int64_t k_max = 0;                  // hot rows the workspace can hold
    int32_t hot_k = 0;                  // current hot rows (0 = off)
    uint32_t hot_mask = 0;
    Slot *hot_index = nullptr;
    int32_t *hslot = nullptr;
    unsigned long long *hot_keys = nullptr;
    float *hot_arena = nullptr, *hot_g = nullptr, *hot_gsum = nullptr, *hot_touch = nullptr, *stage = nullptr;
    uint32_t *hot_cnt = nullptr, *cnt_sum = nullptr, *fcnt = nullptr;
    int32_t *hot_pslot_d = nullptr;
    int64_t *hot_off_d = nullptr;       // [4P]: w, s1, s2, g offsets
    int64_t *fcnt_off_d = nullptr;
    // refresh selection (cache_host.cu refresh_select_all)
    uint32_t *phist = nullptr;          // [P, 65536] per-pack count histograms of the owned rows
    uint32_t *khist = nullptr;          // [65536 + 2] tie bytes by global-key bin
    unsigned long long *tie_keys = nullptr;  // [W, tcap] tie keys in the cut bin (+ [W] counts)
    int32_t *tie_n = nullptr;           // [1]
    uint32_t *sel_bits = nullptr;       // [key space / 32 + 1] the selection bitmap
    int32_t *bits_blk = nullptr;        // [words / 1024 + 3] compaction scratch (+ total)
    int64_t *stage_idx = nullptr;       // [k_max] float offset of each slot in the staging
    int64_t *stage_off_d = nullptr;     // [P] staging offset of each pack's slots
    int64_t stage_floats = 0;
    int64_t rows_total = 0;
    std::vector<int64_t> fcnt_off;      // [P+1]
    std::vector<int32_t> hot_pslot;     // [P+1]
    std::vector<int64_t> hot_off;       // [4P]
    int64_t hot_g_floats = 0;
    int64_t last_hot_uniques = 0, last_uniques = 0;
    int32_t new_k = 0;
    // ---- NVLink peer-memory exchange (p2p.cu / p2p_host.cu)
    bool p2p = false;                   // exchanges go through the peers' windows (no NCCL a2av)
    bool p2p_loop = false;              // loopback group: the host sequences the phases, no barriers
    char *win = nullptr;                // this rank's IPC window (cudaMalloc)
    size_t win_bytes = 0, win_bcount = 0, win_keys = 0, win_gbuf = 0;
    P2PPeers peers{};
    void *peer_base[kP2PMaxW] = {};     // opened IPC mappings (closed at destroy)
    uint32_t *epoch_d = nullptr;        // [2 * kP2PFlags] signal / wait counts per barrier slot
    int32_t *R_d = nullptr;             // [1] received keys (device)
    int64_t *gsrc = nullptr;            // [max_recv * W] G-row offsets per (owner-unique, source)
    int64_t *pack_fbase_d = nullptr, *dbase_d = nullptr, *dst_off = nullptr, *row_base_d = nullptr;
    std::vector<int64_t> row_base;      // [P+1] owned rows per pack, prefix
    int32_t *dtab = nullptr;            // [rows_total * W] owner position of (owned row, source), or -1
    int32_t *dst_rank = nullptr;
    size_t win_ogbuf = 0;
    // ---- NVLS multicast of the hot-row gradients (nvls.cu)
    bool nvls = false;
    unsigned long long nvls_mc = 0, nvls_uc = 0, nvls_uva = 0, nvls_mva = 0;  // driver handles / VAs
    size_t nvls_bytes = 0, nvls_touch_off = 0;
};

struct picasso_ctx {
    int32_t rank = 0, world = 1;
    MultiState mp;
    picasso_ctx_opts opts{};
    int32_t F = 0, T = 0, P = 0;
    std::vector<int32_t> f2t, t2p, tdim, pack_dim;
    std::vector<int64_t> tbase, trows, fcol, pack_rows, pack_key_off;
    std::vector<uint64_t> tsalt;
    int64_t out_width = 0;
    std::vector<int32_t> pm_fields, pack_first_k;
    std::vector<int32_t> pack_slot;  // [P] K-Interleaving barrier slot (excluded packs, then groups)
    int32_t n_slots = 0;
    // workspace layout
    size_t ws_bytes = 0;
    uint32_t cap = 0;
    bool bound = false;
    FieldInfo *finfo = nullptr;
    int32_t *pm_fields_d = nullptr, *pack_first_k_d = nullptr;
    int32_t *field_k_d = nullptr;  // [F] index of each field within its pack
    bool pipe_pool = true;         // PICASSO_POOL=legacy selects the register-staged pool for every D
    int pool_kind = 1;             // PICASSO_POOL=flat (2: k_pool_flat for every D) | default (1: the
                                   // cp.async ring for D >= 64, k_pool_flat below) | legacy (k_pool)
    int64_t *pack_key_off_d = nullptr;
    int32_t *id_start = nullptr, *gstart_pm = nullptr, *field_gstart = nullptr, *pack_gstart = nullptr;
    int32_t *pack_ustart = nullptr;
    Slot *table = nullptr;
    int32_t *slot_of = nullptr, *seg_of = nullptr, *inverse = nullptr;
    uint8_t *fmask = nullptr;  // first-occurrence flags (k_flag_count -> k_assign)
    int64_t *region_base = nullptr;  // per-table dedup hash regions (k_field_prep)
    int region_shift = 1;
    bool use_regions = false;        // max_ids > 2M: one global table would not stay in L2
    uint32_t *region_mask = nullptr;
    int32_t *tocc = nullptr;
    int32_t *empty_pack = nullptr;  // [P] the pack has an empty segment this step
    int32_t *blk_cnt = nullptr, *blk_off = nullptr, *d_total = nullptr, *long_cnt = nullptr;
    int *err = nullptr;
    int32_t *seg_limit = nullptr;  // [1] k_field_prep -> k_seg_of (0 after an offsets error)
    unsigned long long *unique_gkey = nullptr;
    int32_t *k_a = nullptr, *v_a = nullptr, *k_b = nullptr, *v_b = nullptr, *hist = nullptr, *scratch = nullptr;
    int32_t *hist0 = nullptr, *hist1 = nullptr, *rowtot = nullptr;
    SortPlan splan{};
    int32_t *ustart = nullptr, *long_list = nullptr, *chunk_off = nullptr, *chunk_row = nullptr;
    dbl4 *partial = nullptr;
    float *gbuf = nullptr;
    int64_t *pack_gbase = nullptr;
    int32_t *pack_dim_d = nullptr;
    bool bulk_segsum = true;  // PICASSO_SEGSUM=legacy selects the register-staged segsum + hot-row path
    bool flat_small = true;   // D <= 8 segsum: k_segsum_flat (PICASSO_SEGSUM_SMALL=legacy: k_segsum)
    int seg_cfg = 0;          // PICASSO_SEGSUM_CFG (warps x stages of the pipelined segsum)
    int32_t seg_nt = 0;       // its tiles per pack
    int32_t *tile_start = nullptr;
    int4 *split = nullptr;
    bool split_bwd = true;  // the backward keeps a G buffer (k_segsum* -> k_update_rows, the long rows, D-Interleaving)
    int fuse_rw = 3;        // fused backward: tile cost of a row in occurrences (PICASSO_FUSE_RW; C2 sweep)
    bool fuse_pipe = true;   // W = 1, tiled packs of D = 64 / 128: k_segsum_upd, the pipelined segment-sum
                             // with each row's weight / state prefetched into a shared-memory ring and
                             // the optimizer applied at its flush (C2: 116 us vs 74 + 71 us split);
                             // PICASSO_BWD=split: segment-sum + k_update_rows
    bool overlap = true;    // PICASSO_OVERLAP=0: the transpose runs on the caller's stream
    int overlap_env = -1;   // PICASSO_OVERLAP (0 / 1) if set; else chosen per world == 1 forward
    int pool_reserve = 0, pool_sms = 148;  // pipelined pool grid = SMs minus the transpose's share
    bool early_pool = false;  // W = 1: this forward pools concurrently with the dedup + transpose chain
    int early_env = -1;       // PICASSO_EARLY_POOL (0 / 1) if set; else on below kOverlapMinIds IDs
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fp = nullptr, ev_seg = nullptr;
    cudaStream_t side2 = nullptr;  // K-Interleaving: the pools / owner updates beside the exchange
    cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
    int kinterleave = 1;           // PICASSO_KINTERLEAVE=0 turns the per-pack pipelining off
    int32_t *su = nullptr, *sseg = nullptr;  // the last forward's transpose (uid-sorted occurrences)
    // world == 1, several packs: dY regrouped pack by pack before the backward (k_dy_pack), so a
    // pack's per-occurrence dY row reads hit L2 (PICASSO_DY_STAGE=0 reads dY in place)
    bool dy_stage = false;
    float *dyp = nullptr;                 // [max_batch * out_width]
    int32_t *col4_field_d = nullptr;      // [out_width / 4] field of each 16-B column chunk
    int64_t *dyp_base_d = nullptr;        // [F] float offset of field f's block in its pack's rows
    int32_t *dyp_stride_d = nullptr;      // [F] row stride of field f's pack (F_p * D_p)
    int32_t *dyp_col_d = nullptr;         // [F] column of field f inside its pack's rows
    std::vector<int64_t> dyp_off;         // [P] float offset of each pack's [max_batch, F_p * D_p] block
    // sort-based index (k_sortidx.cu): world == 1, pack keys < 2^32, the tiled backward; used from
    // sort_min_ids IDs on (PICASSO_INDEX=hash / sort forces either; PICASSO_SORT_MIN_IDS).  A sorted step numbers the
    // backward's rows in run order and keeps their keys in run_keys() (the dedup table's memory).
    bool sort_idx = false;
    bool sort_step = false;       // the last forward indexed by sort
    bool views_ready = false;     // its reading-O1 views (inverse, Unique) materialised
    const uint64_t *sorted_items = nullptr;  // its sorted (key << 32 | position) items
    bool sort_overlap = true;     // PICASSO_SORT_OVERLAP=0: index chain and pool on the caller's stream
    int sort_key_bits = 32;
    int64_t sort_min_ids = 0;     // (every world == 1 step: C2 0.2411 -> 0.2202 ms, C3 25.3 -> 18.3 ms)
    int sort_reserve = 52;        // SMs the pool leaves to the sort chain beside it (PICASSO_SORT_RESERVE;
                                  // C2 sweep 24 / 32 / 40 / 48 / 56 / 64: 0.2286 / 0.2223 / 0.2185 / 0.2178 / 0.2172 / 0.2185 ms)
    unsigned long long *run_keys() const { return reinterpret_cast<unsigned long long *>(table); }
    // the row-sharded step indexed by sort (world > 1, from sort_min_ids_w IDs on): Unique / inverse
    // from the sort's views (the exchange's uid order), the backward in run order with its per-row
    // arrays gathered through run_uid — no uid transpose (PICASSO_INDEX=hash: off)
    bool sort_w = false;
    bool w_runorder = false;      // the last row-sharded forward indexed by sort
    // ... and exchanged in run order (peer-memory exchange: the order inside a bucket is free, so
    // uid = run index, the inverse comes from k_si_final, no views / run_uid / run gather; the
    // reading-O1 views only on request).  The NCCL exchange keeps first-occurrence order (O2).
    bool w_runx = false;
    int64_t sort_min_ids_w = (int64_t)1 << 20;
    int32_t *run_uid = nullptr, *hs_run = nullptr, *dr_run = nullptr;  // [N]
    int64_t *ro_run = nullptr, *do_run = nullptr;                        // [N]
    unsigned long long *row_keys() const { return sort_step ? run_keys() : unique_gkey; }
    std::vector<float *> w, s1, s2;
    // step state
    bool fwd_done = false;
    int32_t B = 0;
    int64_t N = 0;
    const int32_t *offsets = nullptr;
    cudaStream_t last_stream = nullptr;
    int num_sms = 148;
    int64_t launches_fwd = 0, launches_bwd = 0;
    std::string last_msg;
    // phase profiling (events on the caller's stream)
    // 0 unique(+partition) 1 pool 2 transpose 3 segsum(+update at W=1) 4 owner dedup+gather 5 owner update
    // then per pack (first kPackPhases packs): kPhases + p its pool, kPhases + kPackPhases + p its backward
    static constexpr int kPhases = 6, kPackPhases = 64, kAllPhases = kPhases + 2 * kPackPhases;
    bool prof = false;
    bool prof_graph = false;  // events were captured into a CUDA graph: reads do not reset them
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kAllPhases];
    size_t ev_used[kAllPhases] = {};
    int64_t prof_calls = 0;

    // inside a capture, an external record becomes a graph node that re-records on every replay
    void record(cudaEvent_t e, cudaStream_t s) const {
        if (prof_graph) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
        else cudaEventRecord(e, s);
    }
    void mark_pack(int which, int p, bool begin, cudaStream_t s) {  // which: 0 pool, 1 backward
        if (p < kPackPhases) mark(kPhases + which * kPackPhases + p, begin, s);
    }
    void mark(int ph, bool begin, cudaStream_t s) {
        if (!prof || ph >= kAllPhases) return;
        auto &v = ev[ph];
        if (begin) {
            if (ev_used[ph] == v.size()) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                v.emplace_back(a, b);
            }
            record(v[ev_used[ph]].first, s);
        } else {
            record(v[ev_used[ph]].second, s);
            ++ev_used[ph];
        }
    }
    ~picasso_ctx() {
        for (auto &v : ev)
            for (auto &p : v) {
                cudaEventDestroy(p.first);
                cudaEventDestroy(p.second);
            }
    }

    // D-Interleaving (dinterleave.cu): step accumulator over the micro-batches
    Slot *di_table = nullptr;              // key -> arena offset (dbl4 units, in the uid field)
    uint64_t di_cap = 0;                   // index slots (pow2)
    double *di_acc = nullptr;              // fp64 arena
    int64_t di_acc_cap4 = 0;               // arena capacity, dbl4 units
    int64_t *di_off = nullptr;             // [max_ids] arena offset of each uid of the micro-batch
    int32_t *di_list = nullptr;            // [max_step_unique] index slot of every accumulated row
    unsigned long long *di_counters = nullptr;  // [2] rows, arena used
    float **di_w = nullptr, **di_s1 = nullptr, **di_s2 = nullptr;  // [P] device copies of the pack pointers
                                                                    // (D-Interleaving and the cold tier)
    // HybridHash with a host-DRAM cold tier (coldtier.cu), world == 1
    uint32_t *ct_fcnt = nullptr;           // [ct_rows_total] FCounter by global key
    Slot *ct_index = nullptr;              // HStore index: key -> slot
    uint32_t ct_mask = 0;
    unsigned long long *ct_keys = nullptr; // [ct_kmax] global key of each hot slot (pack-major)
    float *ct_arena = nullptr;             // HStore rows: w of every pack, then s1, then s2
    int32_t *ct_pslot_d = nullptr;         // [P+1]
    int64_t *ct_arena_off_d = nullptr;     // [3P]
    int32_t *ct_hslot = nullptr;           // [max_ids]
    int64_t *ct_row_off = nullptr;         // [max_ids]
    unsigned long long *ct_hits = nullptr, *ct_hist = nullptr, *ct_bsum = nullptr, *ct_bcnt = nullptr,
                       *ct_nsel = nullptr;
    // double-buffered HStore (current = index ct_buf; the refresh builds the other one)
    int ct_buf = 0;
    Slot *ct_index_b[2] = {nullptr, nullptr};
    unsigned long long *ct_keys_b[2] = {nullptr, nullptr};
    float *ct_arena_b[2] = {nullptr, nullptr};
    int32_t *ct_pslot_b[2] = {nullptr, nullptr};
    int64_t *ct_aoff_b[2] = {nullptr, nullptr};
    int64_t ct_kmax = 0, ct_rows_total = 0;
    int32_t ct_k = 0;
    std::vector<int32_t> ct_pslot;
    bool di_active = false;
    int64_t di_micro = 0;

    int32_t *osort_hist = nullptr;  // k_inverse's pass-0 histogram output when run on the owner stream

    size_t carve(char *base) {
        Carver c{base};
        const int64_t N = std::max<int64_t>(opts.max_ids, 1);
        const int64_t NR = std::max<int64_t>(N, mp.max_recv);  // index work of both stream kinds
        const int64_t nblk = (NR + kTile - 1) / kTile + 1;
        finfo = c.take<FieldInfo>(F);
        pm_fields_d = c.take<int32_t>(F);
        field_k_d = c.take<int32_t>(F);
        pack_first_k_d = c.take<int32_t>(P + 1);
        pack_key_off_d = c.take<int64_t>(P + 1);
        id_start = c.take<int32_t>(F);
        gstart_pm = c.take<int32_t>(F + 1);
        field_gstart = c.take<int32_t>(F);
        pack_gstart = c.take<int32_t>(P + 1);
        pack_ustart = c.take<int32_t>(P + 1);
        table = c.take<Slot>(cap);
        region_base = c.take<int64_t>(T + 1);
        region_mask = c.take<uint32_t>(T);
        tocc = c.take<int32_t>(T);
        empty_pack = c.take<int32_t>(P);
        slot_of = c.take<int32_t>(N);
        fmask = c.take<uint8_t>(4 * (size_t)(NR / 32 + 2));  // (also the sort index's 32-bit bitmap words)
        seg_of = c.take<int32_t>(N);
        inverse = c.take<int32_t>(N);
        blk_cnt = c.take<int32_t>(nblk);
        blk_off = c.take<int32_t>(nblk);
        d_total = c.take<int32_t>(1);
        long_cnt = c.take<int32_t>(P + 1);  // (+ the k_si_heads ticket)
        err = c.take<int>(1);
        seg_limit = c.take<int32_t>(1);
        unique_gkey = c.take<unsigned long long>(N);
        k_a = c.take<int32_t>(2 * (size_t)N);  // (k_a, v_a) / (k_b, v_b) adjacent: the sort-based
        v_a = k_a ? k_a + N : nullptr;          //  index's 8-byte items use each pair as one buffer
        k_b = c.take<int32_t>(2 * (size_t)N);
        v_b = k_b ? k_b + N : nullptr;
        hist0 = c.take<int32_t>(radix_hist2_ints(N));
        hist1 = c.take<int32_t>(radix_hist2_ints(N));
        rowtot = c.take<int32_t>(kMaxRadix);
        ustart = c.take<int32_t>(N + 1);
        long_list = c.take<int32_t>(N / (kLongRow + 1) + 2);
        chunk_off = c.take<int32_t>(N / (kLongRow + 1) + 3);
        int maxD = 4;
        for (int32_t d : pack_dim) maxD = std::max(maxD, d);
        partial = reinterpret_cast<dbl4 *>(
            c.take<double>(std::max(long_partial_doubles(N, maxD), segsum_bulk_partial_doubles(maxD, num_sms))));
        tile_start = c.take<int32_t>(segsum_tile_ints(P, num_sms));
        split = c.take<int4>(segsum_split_entries(num_sms));
        chunk_row = c.take<int32_t>(long_partial_doubles(N, 1));
        pack_gbase = c.take<int64_t>(P + 1);
        pack_dim_d = c.take<int32_t>(P);
        if (dy_stage) {
            dyp = c.take<float>((size_t)opts.max_batch * (size_t)out_width);
            col4_field_d = c.take<int32_t>(out_width / 4 + 1);
            dyp_base_d = c.take<int64_t>(F);
            dyp_stride_d = c.take<int32_t>(F);
            dyp_col_d = c.take<int32_t>(F);
        }
        if (world == 1 && opts.max_step_unique > 0) {  // D-Interleaving step accumulator
            di_cap = pow2_at_least((uint64_t)opts.max_step_unique * 2);
            di_table = c.take<Slot>(di_cap);
            di_acc_cap4 = opts.max_step_floats > 0 ? (opts.max_step_floats + 3) / 4 : opts.max_step_unique * (maxD / 4);
            di_acc = c.take<double>((size_t)di_acc_cap4 * 4);
            di_off = c.take<int64_t>(N);
            di_list = c.take<int32_t>(opts.max_step_unique);
            di_counters = c.take<unsigned long long>(2);
        }
        if (world == 1 && (opts.max_step_unique > 0 || opts.cold_tier)) {
            di_w = c.take<float *>(P);
            di_s1 = c.take<float *>(P);
            di_s2 = c.take<float *>(P);
        }
        if (world == 1 && opts.cold_tier) {  // HStore + FCounter of the host-DRAM cold tier
            int minD = 1 << 30;
            for (int32_t d : pack_dim) minD = std::min(minD, d);
            const int nst = opts.opt == PICASSO_OPT_ADAM_LAZY ? 2 : 1;
            ct_kmax = std::max<int64_t>(opts.cache_max_bytes / ((int64_t)4 * minD * (1 + nst)), 1);
            ct_rows_total = pack_key_off.empty() ? 0 : pack_key_off[P];
            ct_mask = (uint32_t)(pow2_at_least((uint64_t)ct_kmax * 2) - 1);
            ct_fcnt = c.take<uint32_t>(std::max<int64_t>(ct_rows_total, 1));
            for (int b = 0; b < 2; ++b) {
                ct_index_b[b] = c.take<Slot>((size_t)ct_mask + 1);
                ct_keys_b[b] = c.take<unsigned long long>(ct_kmax);
                ct_arena_b[b] = c.take<float>(opts.cache_max_bytes / 4 + 4 * P);
                ct_pslot_b[b] = c.take<int32_t>(P + 1);
                ct_aoff_b[b] = c.take<int64_t>(3 * P);
            }
            ct_index = ct_index_b[ct_buf];
            ct_keys = ct_keys_b[ct_buf];
            ct_arena = ct_arena_b[ct_buf];
            ct_pslot_d = ct_pslot_b[ct_buf];
            ct_arena_off_d = ct_aoff_b[ct_buf];
            ct_hslot = c.take<int32_t>(N);
            ct_row_off = c.take<int64_t>(N);
            ct_hits = c.take<unsigned long long>(1);
            ct_hist = c.take<unsigned long long>(1 << 16);
            ct_bsum = c.take<unsigned long long>((ct_rows_total + 1023) / 1024 + 1);
            ct_bcnt = c.take<unsigned long long>((ct_rows_total + 1023) / 1024 + 2);
            ct_nsel = c.take<unsigned long long>(1);
        }
        // rows / G buffer: the IPC window holds it with the peer-memory exchange
        const bool p2p_ex = world > 1 && opts.exchange == 0;
        gbuf = ((split_bwd && world == 1) || (world > 1 && !p2p_ex)) ? c.take<float>((size_t)N * maxD) : nullptr;
        if (world > 1 && sort_w) {
            run_uid = c.take<int32_t>(N);
            hs_run = c.take<int32_t>(N);
            dr_run = c.take<int32_t>(N);
            ro_run = c.take<int64_t>(N);
            do_run = c.take<int64_t>(N);
        }
        if (world > 1) {
            const int64_t RM = std::max<int64_t>(mp.max_recv, 1);
            const int WP = world * P;
            int bb = 1;
            while ((1 << bb) < WP + 1) ++bb;  // + the hot bucket (multi_args' bucket_bits)
            mp.bkey = c.take<int32_t>(N);
            mp.bval = c.take<int32_t>(N);
            mp.bsorted = c.take<int32_t>(N);
            mp.send_uid = c.take<int32_t>(N);
            mp.bhist = c.take<int32_t>((size_t)(1 << bb) * ((N + kTile - 1) / kTile) + 1);
            mp.bcount = c.take<int32_t>(kMaxRadix);
            mp.bstart = c.take<int64_t>(WP + 1);
            mp.sroff = c.take<int64_t>(WP + 1);
            mp.send_pos = c.take<int32_t>(N);
            mp.send_keys = c.take<int32_t>(N);
            mp.row_off = c.take<int64_t>(N);
            mp.cnt_recv_d = c.take<int32_t>(WP);
            mp.recv_keys = c.take<int32_t>(RM);
            mp.opos_map = c.take<int32_t>(RM);
            mp.oslot = c.take<int32_t>(RM);
            mp.oinv = c.take<int32_t>(RM);
            mp.ouid_key = c.take<unsigned long long>(RM);
            mp.opack_gstart = c.take<int32_t>(P + 1);
            mp.opack_ustart = c.take<int32_t>(P + 1);
            mp.od_total = c.take<int32_t>(P + 1);  // NCCL driver: owner unique count; p2p: per-pack row counts
            mp.opack_ostart_d = c.take<int64_t>(P + 1);
            mp.ogbase_scratch = c.take<int64_t>(P + 1);
            mp.oblk_d = c.take<OwnerBlock>(WP);
            mp.contrib = c.take<int32_t>((size_t)RM * world);
            mp.gsrc = c.take<int64_t>((size_t)RM * world);
            mp.pack_fbase_d = c.take<int64_t>(P + 1);
            mp.row_base_d = c.take<int64_t>(P + 1);
            mp.dbase_d = c.take<int64_t>(WP);
            mp.dst_rank = c.take<int32_t>(N);
            mp.dst_off = c.take<int64_t>(N);
            mp.rsend_off = c.take<int64_t>(RM);
            mp.rows_send = p2p_ex ? nullptr : c.take<float>((size_t)RM * maxD);  // NCCL staging only
            osort_hist = c.take<int32_t>(2 * ((RM + kTile - 1) / kTile) + 2);
            mp.epoch_d = c.take<uint32_t>(2 * kP2PFlags);
            mp.R_d = c.take<int32_t>(1);
            if (opts.cache_max_bytes > 0) {  // HybridHash
                const int64_t K = std::max<int64_t>(mp.k_max, 1);
                const int64_t arena = opts.cache_max_bytes / 4 + 4 * P;
                mp.hot_index = c.take<Slot>((size_t)mp.hot_mask + 1);
                mp.hslot = c.take<int32_t>(N);
                mp.hot_keys = c.take<unsigned long long>(K);
                mp.hot_arena = c.take<float>(arena);
                mp.hot_g = c.take<float>(arena / 2 + 4);
                mp.hot_gsum = c.take<float>(arena / 2 + 4);
                mp.hot_touch = c.take<float>(2 * K);
                mp.stage = c.take<float>(arena);
                mp.hot_cnt = c.take<uint32_t>(K);
                mp.cnt_sum = c.take<uint32_t>(2 * K);
                mp.fcnt = c.take<uint32_t>(std::max<int64_t>(mp.rows_total, 1));
                mp.hot_pslot_d = c.take<int32_t>(P + 1);
                mp.hot_off_d = c.take<int64_t>(4 * P);
                mp.fcnt_off_d = c.take<int64_t>(P + 1);
                const int64_t KT = pack_key_off.empty() ? 0 : pack_key_off[P], nw = KT / 32 + 1;
                mp.phist = c.take<uint32_t>((size_t)P << 16);
                mp.khist = c.take<uint32_t>((1 << 16) + 2);
                mp.tie_keys = c.take<unsigned long long>((size_t)world * ((1 << 16) / world + 2) + world + 2);
                mp.tie_n = c.take<int32_t>(1);
                mp.sel_bits = c.take<uint32_t>(nw);
                mp.bits_blk = c.take<int32_t>(nw / 1024 + 3);
                mp.stage_idx = c.take<int64_t>(K);
                mp.stage_off_d = c.take<int64_t>(P);
            }
        }
        return c.off + kAlign;
    }
};

// Loopback group: all ranks of a row-sharded step in one process (multi_host.cu, cache_host.cu).
struct picasso_group {
    std::vector<picasso_ctx *> ctx;
};

