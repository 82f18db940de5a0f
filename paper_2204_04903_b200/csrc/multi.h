// multi.h — device-side arguments of the row-sharded multi-GPU path (internal).
#pragma once
#include "kernels.h"

namespace picasso {

constexpr int kMaxOwnerBlocks = 1024;  // W * P blocks of the owner stream (W <= 8, P <= 128)

struct RankPtrs {  // the W ranks' buffers of a loopback group, passed to a kernel by value
    const void *p[8];
};

// One (pack, source) block of the owner stream (pack-major: pack, then source rank).
struct OwnerBlock {
    int64_t ostart;  // first owner-stream position of the block
    int64_t rstart;  // first receive index (receive buffer is source-major, then pack)
    int64_t rroff;   // float offset of the block's first row in the owner's rows-send buffer
    int32_t pack, src;
};

struct MultiArgs {
    int32_t W, P;
    int64_t nblk;                    // tiles of the bucket pass (ceil(max U / kTile))
    int32_t bucket_bits;             // digit width of the bucket pass (W*P <= 2^bits)
    const int32_t *pack_dim;         // [P]
    const int64_t *pack_key_off;     // [P+1]
    // requester side (this rank's uniques)
    const int32_t *d_total;          // [1] U
    const int32_t *pack_ustart;      // [P+1]
    const unsigned long long *unique_gkey;  // [U]
    int32_t *bkey, *bval;            // [U] bucket, uid (pass input)
    int32_t *bhist;                  // [2^bits, nblk] bucket histogram (digit-major)
    int32_t *bcount;                 // [W*P+1] bucket counts (radix row totals; hot bucket last)
    int64_t *bstart;                 // [W*P+1] first send slot of each bucket
    int64_t *sroff;                  // [W*P+1] float offset of each bucket in the rows buffer
    const int32_t *send_uid;         // [U] uid of each send slot (bucket-sorted)
    int32_t *send_pos;               // [U] send slot of each uid
    int32_t *send_keys;              // [U] requested local row (key div W)
    int64_t *row_off;                // [U] float offset of the uid's row in the rows/G buffer
    // owner side
    int64_t R;                       // received keys (host-known after the counts exchange)
    const OwnerBlock *oblk;          // [W*P] pack-major blocks
    const int64_t *pack_ostart;      // [P+1] owner-stream start of each pack (host & device)
    const int32_t *recv_keys;        // [R] local rows requested (source-major, pack, order)
    int32_t *opos_map;               // [R] owner-stream position -> receive index
    int32_t *oslot;                  // [R] hash slot per owner position
    const int32_t *oinv;             // [R] owner-unique index per owner position
    const unsigned long long *ouid_key;  // [U_o] pack_key_off + local row
    const int32_t *opack_ustart;     // [P+1]
    int32_t *contrib;                // [U_o, W] receive index of each source's request, or -1
    int64_t *rsend_off;              // [R] float offset of receive index i's row in rows_send
    float *rows_send;                // owner rows out (fwd) / gradient rows in (bwd)
    // HybridHash hot storage: replicated top-k rows on every rank
    int32_t hot_k;                   // hot rows (all packs); 0 = cache off
    const Slot *hot_index;           // key -> slot (minpos field holds the slot), replicated
    uint32_t hot_mask;               // hot index capacity - 1
    int32_t *hslot;                  // [U] hot slot of each unique, or -1
    const int32_t *hot_pslot;        // [P+1] slot range of each pack (slots grouped by pack)
    const int64_t *hot_w_off;        // [P] float offset of pack p's replica rows in the arena
    float *hot_arena;                // replicas: per pack [k_p, D] weights, then states
    const int64_t *hot_s1_off, *hot_s2_off;  // [P] offsets of the replicated optimizer state
    float *hot_g;                    // [k rows of D_p] gradient rows of the hot slots (summed over ranks)
    float *hot_touch;                // [k] occurrences of each hot slot this step (summed over ranks)
    uint32_t *hot_cnt;               // [k] FCounter of hot keys (this rank's post-unique hits)
    const int64_t *hot_g_off;        // [P] float offset of pack p's hot G rows in hot_g
    const float *gbuf_base;          // rows/G buffer base (row_off of a hot unique is relative to it)
    uint32_t *fcnt;                  // FCounter of owned rows: [sum_p local_rows_p]
    const int64_t *fcnt_off;         // [P] offset of pack p's counters
};

void launch_bucket(const MultiArgs &m, cudaStream_t s);
void launch_bucket_prefix(const MultiArgs &m, cudaStream_t s);
void launch_send_prep(const MultiArgs &m, int num_sms, cudaStream_t s);
// Partition of the peer-memory exchange: stable (uid order inside a bucket), placed without a sort
void launch_partition_p2p(const MultiArgs &m, int num_sms, cudaStream_t s);
void launch_owner_insert(const MultiArgs &m, Slot *table, uint32_t cap_mask, int *err, cudaStream_t s);
void launch_contrib(const MultiArgs &m, cudaStream_t s);
void launch_gather(int D, const MultiArgs &m, const float *weight, int pack, int num_sms, cudaStream_t s);
void launch_owner_update(int D, const MultiArgs &m, int pack, float *w, float *s1, float *s2, int opt, float lr,
                         float eps, float b1, float b2, float ss, int num_sms, cudaStream_t s);

}  // namespace picasso
