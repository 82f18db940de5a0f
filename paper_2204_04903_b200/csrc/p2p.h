// p2p.h — device-side arguments of the NVLink peer-memory exchange (internal; p2p.cu).
#pragma once
#include "kernels.h"
#include "multi.h"

namespace picasso {

constexpr int kP2PMaxW = 8;                                 // ranks per node at most
constexpr int kP2PPhases = 4;                               // barrier phases per step
constexpr int kP2PMaxGroups = 16;                           // K-Interleaving groups (packs) with own barriers
constexpr int kP2PFlags = kP2PPhases * kP2PMaxGroups;       // barrier slots: (phase, group)
constexpr unsigned long long kP2PTimeoutNs = 20000000000ull;  // a peer missing for 20 s latches an error
enum P2PErrBits : int { ERR_PEER_TIMEOUT = 4 };

// One rank's IPC window, seen by everyone (index = rank; own pointers at [rank]).
struct P2PPeers {
    uint32_t *flags[kP2PMaxW];     // [kP2PFlags][kP2PMaxW] epoch written by each source rank
    int32_t *bcount[kP2PMaxW];     // [W*P+1] bucket counts (owner-major, pack), hot bucket last
    int32_t *send_keys[kP2PMaxW];  // [max_ids] requested local rows, owner-major send layout
    float *gbuf[kP2PMaxW];         // [max_ids * maxD] rows received (fwd), send layout
    float *ogbuf[kP2PMaxW];        // [max_recv * maxD] G rows received by the owner (bwd), owner-
                                   //   stream layout: pack p's rows from pack_fbase[p], D_p floats each
};

struct P2PArgs {
    int32_t W, P, rank;
    int64_t max_recv;
    P2PPeers peer;
    uint32_t *epoch;               // [2 * kP2PFlags] this rank's signal, then wait counts per slot
    int *err;
    const int32_t *pack_dim;       // [P]
    const int64_t *pack_key_off;   // [P+1]
    OwnerBlock *oblk;              // [W*P] pack-major (p, src): ostart, rstart = key index in src's
                                   //   send list, rroff = float offset of the row slot in src's gbuf
    int64_t *pack_ostart;          // [P+1] owner-stream start of each pack
    int32_t *opack_gstart;         // [P+1] same, int32, for the index kernels
    int32_t *R;                    // [1] received keys
    int32_t *cnt_recv;             // [W*P] received counts (source, pack), introspection
    int32_t *lrow;                 // [max_recv] local row per owner position
    int32_t *osrc;                 // [max_recv] source rank per owner position
    int64_t *roff;                 // [max_recv] float offset of the row slot in the source's gbuf
    int32_t *dtab;                 // [rows_total * W] owner position of (owned row, source), or -1
    int32_t *olist;                // [max_recv] (W > 2) rows requested this step, once each, per pack block
    int32_t *ocount;               // [P] (W > 2) rows listed per pack
    const int64_t *row_base;       // [P+1] owned rows per pack, prefix
    int64_t *pack_fbase;           // [P+1] float offset of pack p's G rows in this rank's ogbuf
    // requester side (push destinations of its G rows)
    const int32_t *d_total;        // [1] U
    const int32_t *bkey;           // [U] bucket (owner * P + pack; W * P = hot) of each unique
    const int32_t *send_pos;       // [U] send slot of each unique
    const int64_t *bstart;         // [W*P+1] first send slot of each bucket
    int64_t *dbase;                // [W*P] float offset of my block of bucket (r, p) in r's ogbuf
    int32_t *dst_rank;             // [U]
    int64_t *dst_off;              // [U]
    uint32_t *fcnt;                // HybridHash FCounter of owned rows (nullptr: off)
    const int64_t *fcnt_off;
};

// barrier slot = phase * kP2PMaxGroups + group
void launch_p2p_signal(const P2PArgs &a, int slot, cudaStream_t s);
void launch_p2p_wait(const P2PArgs &a, int slot, cudaStream_t s);
void launch_p2p_tables(const P2PArgs &a, cudaStream_t s);
void launch_p2p_dst_insert(const P2PArgs &a, int num_sms, cudaStream_t s);
void launch_p2p_leaders(const P2PArgs &a, int num_sms, cudaStream_t s);
void launch_p2p_reset(const P2PArgs &a, int num_sms, cudaStream_t s);
void launch_p2p_gather(int D, const P2PArgs &a, const float *weight, int pack, int num_sms, cudaStream_t s,
                       bool vec8 = false);
void launch_p2p_update(int D, const P2PArgs &a, int pack, float *w, float *s1, float *s2, int opt, float lr, float eps,
                       float b1, float b2, float ss, int num_sms, cudaStream_t s, bool vec8 = false,
                       bool list = false);

}  // namespace picasso
