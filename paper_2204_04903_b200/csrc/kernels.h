// kernels.h — host-side launchers of the sm_100a kernels (internal; not part of the C ABI).
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

#include "common.cuh"

namespace picasso {

// Opt a kernel in to `bytes` of dynamic shared memory on the current device (the attribute is
// per device: a process driving several GPUs sets it once per (kernel, device)).
inline cudaError_t ensure_dyn_smem(const void *fn, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    std::lock_guard<std::mutex> g(mu);
    size_t &v = done[{fn, dev}];
    if (v >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) v = bytes;
    return e;
}

#ifndef PICASSO_KTILE
#define PICASSO_KTILE 2048
#endif
constexpr int kTile = PICASSO_KTILE;  // keys per block in the index / scan / sort kernels
constexpr int kTileThreads = 256;
constexpr int64_t kOverlapMinIds = (int64_t)1 << 22;  // world == 1: transpose beside the pool from here on
constexpr int kLongRow = 256;   // rows with more occurrences take the chunked backward path

struct IndexArgs {
    const int64_t *ids;
    const int32_t *offsets;
    int32_t B;
    int64_t N;
    int32_t F, P;
    int32_t id_mode;
    const FieldInfo *finfo;        // [F]
    const int32_t *pm_fields;      // [F] fields in pack-major order (pack asc, field asc)
    const int32_t *pack_first_k;   // [P+1] first pm index of each pack
    const int64_t *pack_key_off;   // [P+1] global key offset of each pack
    int32_t *id_start;             // [F]  out: offsets[f*B]
    int32_t *gstart_pm;            // [F+1] out: packed-stream start of the k-th pm field
    int32_t *field_gstart;         // [F]  out
    int32_t *pack_gstart;          // [P+1] out
    Slot *table;
    uint32_t cap_mask;
    int32_t *slot_of;              // [N]
    int32_t *seg_of;               // [N]
    int32_t *inverse;              // [N] global uid per packed position
    int32_t *blk_cnt;              // [nblk]
    int32_t *blk_off;              // [nblk]
    int32_t *d_total;              // [1] U (all packs)
    unsigned long long *unique_gkey; // [N]
    int32_t *pack_ustart;          // [P+1]
    const int32_t *pack_dim;       // [P]
    int64_t *pack_gbase;           // [P+1] out: float offset of each pack's G rows (sum U_p * D_p)
    const int32_t *n_dev;          // if set: the position count lives on the device (N = capacity)
    uint8_t *fmask;                // [N/8+1] first-occurrence flags, 8 positions per byte
    int32_t T;                     // tables
    int64_t *region_base;          // [T+1] per-table hash region start (slots); [T] = total (nullptr:
                                   //   one global table masked by cap_mask)
    uint32_t *region_mask;         // [T] region size - 1
    int32_t region_shift;          // region >= occurrences << shift (load factor <= 1/2 or 1/4)
    int32_t *tocc;                 // [T] scratch: occurrences per table
    int32_t *empty_pack;           // [P] zeroed here, set by k_seg_of
    int32_t *seg_limit;            // [1] out: positions k_seg_of may place (n_ids; 0 after an offsets error)
    uint32_t *keys;                // [N] sort-based index: k_field_prep's substitute layout also keys every
                                   //   position (row 0 of the first field's table) after an offsets error
    int32_t sort_bits0;            // digit width of the backward's first radix pass
    int32_t *sort_hist0;           // [radix0, nblk] out: digit-major histogram of that pass
    int *err;
};

// Radix sort plan of the backward's transpose: keys (uids) < 2^bits, passes of <= 10 bits.
constexpr int kMaxRadixBits = 10;
constexpr int kMaxRadix = 1 << kMaxRadixBits;
struct SortPlan {
    int passes;
    int bits[4];
    int shift[4];
};
SortPlan make_sort_plan(int64_t n);
// Stable LSD radix sort of (key, val) int32 pairs; hist0 = digit-major histogram of pass 0
// (from k_inverse).  hist1: scratch of the same size; rowtot: [kMaxRadix].
void radix_sort_pairs2(const int32_t *k_in, const int32_t *v_in, int32_t *k_a, int32_t *v_a, int32_t *k_b,
                       int32_t *v_b, int32_t **k_out, int32_t **v_out, int64_t n, const SortPlan &plan,
                       int32_t *hist0, int32_t *hist1, int32_t *rowtot, cudaStream_t s, int64_t *launches);
size_t radix_hist2_ints(int64_t n);
// per-digit exclusive scan of a digit-major [radix, nblk] histogram (+ digit totals); zero_next:
// also zeroes the [next_radix, nblk] rows of that buffer (the next pass's counts)
void bucket_scan(int32_t *hist, int64_t nblk, int32_t *rowtot, int radix, cudaStream_t s, int32_t *zero_next = nullptr,
                 int next_radix = 0);
void bucket_sort_pass(const int32_t *k_in, const int32_t *v_in, int32_t *k_out, int32_t *v_out, int64_t n_max,
                      const int32_t *n_dev, int bits, int32_t *bhist, int32_t *rowtot, cudaStream_t s);

// k_sortidx.cu: the index phase of a large world == 1 step as one stable LSD sort of
// (pack key << 32 | position); rows come out in run (ascending key) order
struct SortIdxArgs {
    const int64_t *ids;            // first up-sweep: keys from the IDs
    const int32_t *seg_of;         //   [N] segment f * B + b of each packed position
    int32_t B;
    int64_t N;
    int32_t id_mode;
    const FieldInfo *finfo;
    const int32_t *id_start, *field_gstart;
    const int64_t *pack_key_off;
    int *err;
    uint32_t *keys;                // [N] pack key of each position (first pass)
    const int32_t *vals;           // [N] first pass's item values (nullptr: the position itself)
    int32_t *hist, *rowtot;        // LSD passes: [radix, nc] chunk counts, [radix] digit totals
    int32_t nc;
    int64_t chunk;
    int32_t *tile_heads, *tile_last, *run_base, *carry;  // [nblk] each
    int32_t *pack_hb;              // [P+1] heads before each pack's first item, in its tile
    int32_t *d_total;              // [1] U
    int32_t *su, *sseg;            // [N] row (run index) and segment of each sorted occurrence
    int32_t *ustart;               // [U+1] first sorted occurrence of each row (run order)
    unsigned long long *run_key;   // [U] pack key of each row (run order: the backward's rows)
    int32_t P;
    const int32_t *pack_gstart;
    int32_t *pack_ustart;
    int64_t *pack_gbase;
    const int32_t *pack_dim;
    int32_t nt, rw;                // equal-cost tiles of the backward (k_csr_tiles partition)
    int32_t *tile_start;           //   [P, nt+1] (nullptr: none)
    int32_t *long_cnt;             // [P] zeroed
    // reading-O1 views (launch_sort_views)
    uint32_t *bm;                  // [N/32] first-occurrence bitmap over positions
    int32_t *wpref;                // [N/32] first occurrences before each bitmap word
    int32_t *view_scratch;         // [2 nblk]
    int32_t *inverse;              // [N] uid of each position
    unsigned long long *unique_gkey;  // [U] key of each uid (first-occurrence order)
    int32_t *run_uid;              // [U] (optional) uid of each row in run order
    int32_t *inv_run;              // [N] (optional) k_si_final: row (run index) of each position
};
struct SortIdxPlan {
    int passes;
    int bits[4];
    int shift[4];
    int64_t chunk;  // items per CTA (a multiple of kTile)
    int32_t nc;     // CTAs
};
SortIdxPlan make_sortidx_plan(int64_t n, int key_bits, int num_sms);
size_t sortidx_scratch_ints(int64_t n, int32_t P);  // tile arrays + views scratch + word ranks
// returns #launches; *sorted: the sorted items, *other: the buffer holding su / sseg
int launch_sort_index(SortIdxArgs a, const SortIdxPlan &plan, uint64_t *buf_a, uint64_t *buf_b, uint64_t **sorted,
                      uint64_t **other, cudaStream_t s);
int launch_sort_views(SortIdxArgs a, const uint64_t *sorted, cudaStream_t s);  // inverse + Unique (reading O1)
// row-sharded step indexed by sort: the backward's per-row arrays in run order (row r = uid run_uid[r]);
// any source may be nullptr (its destination is then left alone)
void launch_run_gather(const int32_t *run_uid, const int32_t *d_total, int64_t n_max, const int32_t *hslot,
                       int32_t *hs_run, const int64_t *row_off, int64_t *ro_run, const int32_t *dst_rank,
                       int32_t *dr_run, const int64_t *dst_off, int64_t *do_run, int num_sms, cudaStream_t s);
// stable sort of int32 (key, val) pairs by key < 2^key_bits through the chunked passes; the sorted
// pairs land in the buffer the last pass did not write (*k_out, *v_out = *k_out + n); #launches
int sort_pairs_chunked(const int32_t *k_in, const int32_t *v_in, uint64_t *buf_a, uint64_t *buf_b, int32_t **k_out,
                       int32_t **v_out, int64_t n, int key_bits, int32_t *hist, int32_t *rowtot, int num_sms,
                       cudaStream_t s);

// k_index.cu
void launch_field_prep(const IndexArgs &a, cudaStream_t s);
void launch_dedup_insert(const IndexArgs &a, cudaStream_t s);
void launch_dedup_assign(const IndexArgs &a, cudaStream_t s);  // flag, scan, uid, unique, pack_ustart, inverse

// k_scan.cu / k_sort.cu
void launch_scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *scratch, int32_t *total,
                           cudaStream_t s);
size_t scan_scratch_ints(int64_t n);


// k_pool.cu
struct PoolArgs {
    const int64_t *ids;
    const int32_t *offsets;
    int32_t B;
    int32_t Fp;                 // fields in this pack
    const int32_t *pack_fields; // [Fp] field indices (ascending)
    const FieldInfo *finfo;
    const int32_t *field_gstart; // [F] packed-stream start of each field
    const int32_t *id_start;     // [F] offsets[f*B]
    int32_t *seg_of;             // [N] out: global segment f*B+b of each packed position
    const int64_t *row_off;      // W > 1: [U] float offset of each unique row in `weight` (the
    const int32_t *inverse;      //        received rows); inverse [N] maps positions to uids
    int32_t id_mode, pool_mean;
    const float *weight;        // [rows, D]
    float *out;
    int64_t out_stride;
    int *err;
    int32_t pack;                // pipelined pool: this pack,
    const int32_t *pack_gstart;  //   [P+1] its packed positions,
    const int32_t *field_k;      //   [F] index of each field within its pack
    const int32_t *empty_pack;   //   [P] 1 if the pack has an empty segment this step (k_seg_of)
    int64_t n_ids;               // IDs of the step: per-segment ranges are clamped to [0, n_ids)
    int32_t vec8;                // k_pool_flat: 32-B chunks allowed (rows, output columns 32-B aligned)
};
void launch_pool(int D, const PoolArgs &a, int num_sms, cudaStream_t s);
// k_pool_pipe.cu: pipelined pool for D >= 64 (needs seg_of from launch_seg_of); returns #launches
bool pool_pipe_supported(int D, const PoolArgs &a);
int launch_pool_pipe(int D, const PoolArgs &a, int num_sms, cudaStream_t s);
// gtotal: [1] positions k_seg_of may place (k_field_prep: n_ids, 0 after an offsets error); err: latch;
// ka (optional): also the pack key of every position (the sort-based index's first pass)
struct SegKeyArgs {
    const int64_t *ids;
    const int64_t *pack_key_off;
    int32_t id_mode;
    uint32_t *keys;  // [N] out (nullptr: seg_of only)
};
void launch_seg_of(const int32_t *offsets, int32_t B, int32_t F, const int32_t *field_gstart, const int32_t *id_start,
                   int32_t *seg_of, cudaStream_t s, const FieldInfo *finfo, int32_t *empty_pack, const int32_t *gtotal,
                   int *err, const SegKeyArgs *ka = nullptr);
// k_pool_flat.cu: one thread per 16-B output chunk (every D); returns #launches
int launch_pool_flat(int D, const PoolArgs &a, int num_sms, cudaStream_t s);

// k_update.cu
struct UpdateArgs {
    const int32_t *sorted_u;     // [N] (unused by kernels; boundaries)
    const int32_t *sorted_seg;   // [N]
    const int32_t *ustart;       // [U+1]
    const int32_t *pack_ustart;  // [P+1]
    int32_t pack;
    const unsigned long long *unique_gkey;
    int64_t pack_key_off;
    const int32_t *offsets;
    int32_t B;
    const FieldInfo *finfo;
    const float *dy;
    int64_t dy_stride;
    const int32_t *dy_col;       // [F] column of each field in dy (nullptr: finfo[f].col)
    int32_t pool_mean;
    int32_t opt;                 // 0 adagrad, 1 adam
    float lr, eps, beta1, beta2, adam_ss;
    float *weight, *state1, *state2;
    int32_t *long_list;          // [cap] rows deferred to the chunked path (this pack)
    int32_t *long_cnt;           // [1]   this pack's counter
    int32_t *chunk_off;          // [cap+1]
    int32_t *chunk_row;          // [chunks] deferred-row index of each chunk
    dbl4 *partial;               // [chunks, D/4] fp64 chunk partial sums
    float *gbuf;                 // split backward: G rows of all packs (nullptr: fused)
    const int64_t *row_off;      // W > 1: [U] float offset of each unique row's G in gbuf
    const int64_t *pack_gbase;   // [P+1] float offset of each pack's G rows in gbuf
    const int32_t *hslot;        // HybridHash: [U] hot slot or -1 (nullptr: no hot rows)
    float *hot_g;                // hot-slot gradient rows (pack p at hot_g_off[p])
    const int64_t *hot_g_off;    // [P]
    const int32_t *hot_pslot;    // [P+1]
    float *hot_touch;            // [k] occurrences of the hot slot this step
    const int32_t *tile_start;   // pipelined segsum: [P, nt+1] equal-cost tile starts (nullptr: legacy)
    int32_t nt;                  //   tiles per pack (= SMs x warps per CTA)
    int4 *split;                 //   [nt] rows cut by tile edges: {first tile, uid, start, end}
    // W > 1 over peer memory: G rows go straight to their owner's receive buffer
    const int32_t *dst_rank;     //   [U] owner of each unique row (nullptr: G stays local)
    const int64_t *dst_off;      //   [U] float offset of its G row in the owner's receive buffer
    float *dst_buf[8];           //   the ranks' receive buffers (NVLink peer pointers)
};
#ifdef __CUDACC__
__device__ __forceinline__ int64_t dy_col(const UpdateArgs &a, int32_t f) {
    return a.dy_col ? (int64_t)__ldg(a.dy_col + f) : a.finfo[f].col;
}
#endif
// dY of a multi-pack step regrouped pack by pack ([pack][b][F_p * D_p], so one pack's gradient is
// contiguous and its random per-occurrence row reads stay in L2); one thread per 16-B chunk
void launch_dy_pack(const float *dy, int32_t B, int64_t out_width, const int32_t *col4_field, const FieldInfo *finfo,
                    const int64_t *dst_base, const int32_t *fstride, float *dyp, cudaStream_t s);
void launch_segsum(int D, const UpdateArgs &a, int num_sms, cudaStream_t s, bool flat_small = true);
void launch_update_rows(int D, const UpdateArgs &a, int num_sms, cudaStream_t s);
void launch_csr_bounds(const int32_t *sorted_u, int64_t N, int32_t *ustart, int32_t *long_cnt, int32_t n_cnt,
                       cudaStream_t s);
int launch_long_update(int D, const UpdateArgs &a, int num_sms, cudaStream_t s);  // returns #launches
size_t long_partial_doubles(int64_t N, int maxD);
// k_segsum_bulk.cu: bulk-copy pipelined segsum (+ split-row fix-up); returns #launches
int segsum_pipe_cfg();            // PICASSO_SEGSUM_CFG
int segsum_pipe_warps(int cfg);    // warps per CTA of that configuration
bool segsum_bulk_supported(int D, const UpdateArgs &a);
int launch_segsum_bulk(int cfg, int D, const UpdateArgs &a, int num_sms, cudaStream_t s);
void launch_csr_tiles(const int32_t *sorted_u, int64_t N, int32_t *ustart, int32_t *long_cnt,
                      const int32_t *pack_gstart, const int32_t *pack_ustart, int32_t P, int32_t nt,
                      int32_t *tile_start, cudaStream_t s, int32_t row_weight = 1);
size_t segsum_bulk_partial_doubles(int maxD, int num_sms);
int launch_segsum_fused(int D, const UpdateArgs &a, int num_sms, cudaStream_t s);  // 0: not applicable
int segsum_upd_warps(int opt);  // warps per CTA (= tiles per SM) of the fused segment-sum + update
size_t segsum_tile_ints(int P, int num_sms);
size_t segsum_split_entries(int num_sms);

}  // namespace picasso
