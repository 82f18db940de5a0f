// k_sortidx.cu — the index phase of a large step as ONE stable sort (world == 1).
//
// Unique ("Unique&Partition") and the backward's transpose (each
// row's occurrences, ascending position: L219) both follow from sorting the packed key stream.
// Above a few million IDs the hash path's table (2-4 slots per ID) no longer stays in L2: at C3
// (83.5 M IDs) its clear / insert / flag / assign / inverse passes each stream the 3.3 GB table
// from HBM and the uid sort of the transpose runs on top (11.3 of a 26.5 ms step).  Here the
// item (key << 32 | position g) is sorted by key, least significant digit first, so equal keys
// keep ascending g; every later output is one streaming pass:
//
//   k_si_up / bucket_scan / k_si_down : one LSD pass of <= 8 bits.  Each CTA owns a contiguous
//        chunk of the input (~70 tiles of 2048 at C3): the up-sweep counts the chunk's digits
//        (digit-major [radix, nc], scanned per digit row by bucket_scan), the down-sweep walks the
//        chunk tile by tile with a running base per digit, ranks each tile stably (warp
//        __match_any_sync), stages it in digit order in shared memory and stores it so
//        consecutive threads write consecutive slots of a digit's run (~8 items per run at 8 bits),
//        while the next tile's items are already being loaded.  The first pass reads the keys
//        k_seg_of derived from the IDs (position -> field -> table row -> pack key).
//   k_si_heads   : run heads (first item of each key): per tile head count, last head, and the
//                  heads before each pack's first item
//   (scan)       : in k_si_heads' last CTA: run index base per tile, last head before each tile
//                  (runs that cross tiles), U, per-pack row ranges, the split backward's G layout
//   k_si_final   : per sorted item: its row (run index) and segment, row starts and keys, and the
//                  backward's equal-cost tiles (the k_csr_tiles partition)
//
// Rows are numbered in RUN order (ascending key) instead of uid order: a pack's keys are
// contiguous, so pack ranges (pack_ustart) are the same; each row's occurrences are in the same
// ascending-position order, so every update equals the one the uid-ordered transpose gives;
// the backward reads row keys from run_key.  Nothing in a world == 1 step consumes the uid
// numbering (the pool maps raw IDs to rows itself), so the reading-O1 views — Unique in
// first-occurrence order and the inverse index — are materialised from the sorted items on
// request (launch_sort_views: first-occurrence bitmap over positions, word ranks, one pass).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace picasso {
namespace {

constexpr int kSiThreads = 256;
constexpr int kSiItems = kTile / kSiThreads;  // 8 items per thread per tile
constexpr int kSiWarps = kSiThreads / 32;
constexpr int kSiBits = 8;                    // digit width of an LSD pass
constexpr int kSiRadix = 1 << kSiBits;
static_assert(kSiItems == 8 && kSiRadix == kSiThreads, "one digit per thread; 8 consecutive items = 4 x 16 B");

__device__ __forceinline__ uint64_t ld_item(const uint64_t *p, int64_t i) {
    return __ldg(reinterpret_cast<const unsigned long long *>(p) + i);
}

// 8 consecutive sorted items from i0 (vector loads when all are in range)
__device__ __forceinline__ void load8(const uint64_t *s, int64_t i0, int64_t N, uint64_t *x) {
    if (i0 + kSiItems <= N) {
        const uint4 *p = reinterpret_cast<const uint4 *>(s + i0);
#pragma unroll
        for (int q = 0; q < kSiItems / 2; ++q) {
            const uint4 v = __ldg(p + q);
            x[2 * q] = ((uint64_t)v.y << 32) | v.x;
            x[2 * q + 1] = ((uint64_t)v.w << 32) | v.z;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSiItems; ++k) x[k] = i0 + k < N ? ld_item(s, i0 + k) : 0ull;
    }
}

// head flags of 8 consecutive sorted items (bit k: item i0 + k starts a run)
__device__ __forceinline__ unsigned heads8(const uint64_t *s, int64_t i0, int64_t N, const uint64_t *x) {
    uint32_t kprev = i0 > 0 && i0 < N ? (uint32_t)(ld_item(s, i0 - 1) >> 32) : 0u;
    unsigned hm = 0;
#pragma unroll
    for (int k = 0; k < kSiItems; ++k) {
        const uint32_t key = (uint32_t)(x[k] >> 32);
        if (i0 + k < N && (i0 + k == 0 || key != kprev)) hm |= 1u << k;
        kprev = key;
    }
    return hm;
}

// FIRST: the keys k_seg_of derived from the IDs (position -> field -> table row -> pack key)
template <bool FIRST>
__global__ void __launch_bounds__(kSiThreads) k_si_up(SortIdxArgs a, const uint64_t *in, int shift, int bits) {
    __shared__ int32_t h[kSiRadix];
    const uint32_t dm = (1u << bits) - 1u;
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t c0 = (int64_t)blockIdx.x * a.chunk;
    const int64_t c1 = c0 + a.chunk < a.N ? c0 + a.chunk : a.N;
    for (int64_t b = c0; b < c1; b += kSiItems * kSiThreads) {
        uint32_t k[kSiItems];
#pragma unroll
        for (int r = 0; r < kSiItems; ++r) {  // eight independent load chains in flight per thread
            const int64_t g = b + r * kSiThreads + threadIdx.x;
            if (FIRST) k[r] = g < c1 ? __ldg(a.keys + g) : 0u;
            else k[r] = g < c1 ? (uint32_t)(ld_item(in, g) >> 32) : 0u;
        }
#pragma unroll
        for (int r = 0; r < kSiItems; ++r)
            if (b + r * kSiThreads + threadIdx.x < c1) atomicAdd(&h[(k[r] >> shift) & dm], 1);
    }
    __syncthreads();
    if (threadIdx.x < (1 << bits)) a.hist[(int64_t)threadIdx.x * a.nc + blockIdx.x] = h[threadIdx.x];
}

template <bool FIRST>
__device__ __forceinline__ void si_load_tile(const SortIdxArgs &a, const uint64_t *in, int64_t t0, int nt, int wb,
                                             int lane, uint64_t *it) {
#pragma unroll
    for (int r = 0; r < kSiItems; ++r) {
        const int li = wb + r * 32 + lane;
        if (li < nt) {
            const int64_t g = t0 + li;
            if (FIRST) it[r] = ((uint64_t)__ldg(a.keys + g) << 32) | (a.vals ? (uint32_t)__ldg(a.vals + g) : (uint32_t)g);
            else it[r] = ld_item(in, g);
        } else {
            it[r] = 0ull;
        }
    }
}

template <bool FIRST>
__global__ void __launch_bounds__(kSiThreads, 3) k_si_down(SortIdxArgs a, const uint64_t *in, uint64_t *out,
                                                           int shift, int bits) {
    __shared__ __align__(16) uint64_t stage[kTile];   // the tile in digit order
    __shared__ int32_t wc[kSiWarps][kSiRadix];         // per-warp digit counts, then warp offsets
    __shared__ int32_t rbase[kSiRadix];                // output slot of each digit's next item
    __shared__ int32_t tstart[kSiRadix + 1];           // tile-local digit starts
    using BlockScan = cub::BlockScan<int32_t, kSiThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    const int radix = 1 << bits;
    const uint32_t dm = (uint32_t)radix - 1u;
    const int dshift = 32 + shift;
    const int d0 = threadIdx.x;  // this thread's digit
    {   // the chunk's first slot per digit: all smaller digits + this digit in earlier chunks
        const int32_t v = d0 < radix ? a.rowtot[d0] : 0;
        int32_t e;
        BlockScan(tmp).ExclusiveSum(v, e);
        if (d0 < radix) rbase[d0] = e + a.hist[(int64_t)d0 * a.nc + blockIdx.x];
    }
#pragma unroll
    for (int w = 0; w < kSiWarps; ++w) wc[w][d0] = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int wb = w * 32 * kSiItems;  // the warp's 256 consecutive items of a tile
    const int64_t c0 = (int64_t)blockIdx.x * a.chunk;
    const int64_t c1 = c0 + a.chunk < a.N ? c0 + a.chunk : a.N;
    uint64_t it[kSiItems];
    if (c0 < c1) si_load_tile<FIRST>(a, in, c0, (int)(c1 - c0 < kTile ? c1 - c0 : kTile), wb, lane, it);
    __syncthreads();
    for (int64_t t0 = c0; t0 < c1; t0 += kTile) {
        const int nt = (int)(c1 - t0 < kTile ? c1 - t0 : kTile);
        int dg[kSiItems], rk[kSiItems];
#pragma unroll
        for (int r = 0; r < kSiItems; ++r) {  // stable rank inside the warp's run of each digit
            const bool valid = wb + r * 32 + lane < nt;
            dg[r] = valid ? (int)((uint32_t)(it[r] >> dshift) & dm) : 0;
            // lanes holding the same digit: MATCH.ANY for half the rounds, one ballot per digit bit
            // for the other half — MATCH alone kept the ADU pipe 88 % busy, the ballots alone the
            // ALU pipe 65 % (C3 ncu); alternating splits the work between the two pipes
            unsigned peers;
            if (r & 1) {
                peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
                for (int b = 0; b < kSiBits; ++b) {
                    const bool bit = (dg[r] >> b) & 1;
                    const unsigned m = __ballot_sync(0xffffffffu, bit);
                    peers &= bit ? m : ~m;
                }
            } else {
                peers = __match_any_sync(0xffffffffu, valid ? dg[r] : kSiRadix + lane);
            }
            const int before = valid ? wc[w][dg[r]] : 0;
            rk[r] = before + __popc(peers & lt);
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) wc[w][dg[r]] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {   // warp offsets per digit (in place) and the tile's digit starts
            int32_t run = 0;
#pragma unroll
            for (int ww = 0; ww < kSiWarps; ++ww) {
                const int32_t t = wc[ww][d0];
                wc[ww][d0] = run;
                run += t;
            }
            int32_t e;
            BlockScan(tmp).ExclusiveSum(run, e);
            tstart[d0] = e;
            if (d0 == kSiThreads - 1) tstart[kSiRadix] = e + run;  // = nt
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kSiItems; ++r)
            if (wb + r * 32 + lane < nt) stage[tstart[dg[r]] + wc[w][dg[r]] + rk[r]] = it[r];
        __syncthreads();
#pragma unroll
        for (int ww = 0; ww < kSiWarps; ++ww) wc[ww][d0] = 0;  // (read above; next tile's counts)
        const int64_t t1 = t0 + kTile;
        if (t1 < c1) si_load_tile<FIRST>(a, in, t1, (int)(c1 - t1 < kTile ? c1 - t1 : kTile), wb, lane, it);
        for (int i = threadIdx.x; i < nt; i += kSiThreads) {  // consecutive threads, consecutive slots
            const uint64_t x = stage[i];
            const int d = (int)((uint32_t)(x >> dshift) & dm);
            out[rbase[d] + (i - tstart[d])] = x;
        }
        __syncthreads();
        rbase[d0] += tstart[d0 + 1] - tstart[d0];
    }
}

// one block of NT threads: run bases, carries, U, pack row ranges, G layout (the tile arrays are
// read through L2: the last k_si_heads CTA runs this on the other CTAs' stores)
template <int NT>
__device__ __forceinline__ void si_scan_body(const SortIdxArgs &a, int64_t nblk,
                                             typename cub::BlockScan<int32_t, NT>::TempStorage &tmp) {
    using BS = cub::BlockScan<int32_t, NT>;
    __shared__ int32_t c_run, c_last;
    if (threadIdx.x == 0) {
        c_run = 0;
        c_last = -1;
    }
    __syncthreads();
    for (int64_t base = 0; base < nblk; base += NT) {
        const int64_t i = base + threadIdx.x;
        const bool v = i < nblk;
        int32_t e, agg;
        BS(tmp).ExclusiveSum(v ? __ldcg(a.tile_heads + i) : 0, e, agg);
        if (v) a.run_base[i] = c_run + e;
        __syncthreads();
        if (threadIdx.x == 0) c_run += agg;
        // last head before each tile (head indices rise with the tile: a running max)
        BS(tmp).ExclusiveScan(v ? __ldcg(a.tile_last + i) : -1, e, cub::Max(), agg);
        if (v) a.carry[i] = threadIdx.x == 0 ? c_last : max(c_last, e);
        __syncthreads();
        if (threadIdx.x == 0) c_last = max(c_last, agg);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int32_t U = c_run;
        *a.d_total = U;
        int64_t gb = 0;
        int32_t prev = 0;
        for (int p = 0; p <= a.P; ++p) {  // a pack's first row: run base of its first item's tile + heads before it
            const int32_t G0 = a.pack_gstart[p];
            const int32_t u = G0 < a.N ? a.run_base[G0 / kTile] + __ldcg(a.pack_hb + p) : U;
            a.pack_ustart[p] = u;
            if (p > 0) {
                a.pack_gbase[p - 1] = gb;
                gb += (int64_t)(u - prev) * a.pack_dim[p - 1];
            }
            prev = u;
        }
        a.pack_gbase[a.P] = gb;
        a.ustart[U] = (int32_t)a.N;
    }
}

// run heads per sorted tile: head count, last head, heads before each pack's first item; the
// last CTA to finish (ticket a.long_cnt[P], zeroed with the step's counters) then scans the tile
// arrays (si_scan_body) — no separate single-block launch on the chain
__global__ void __launch_bounds__(kSiThreads) k_si_heads(SortIdxArgs a, const uint64_t *s) {
    using BS = cub::BlockScan<int32_t, kSiThreads>;
    using BR = cub::BlockReduce<int32_t, kSiThreads>;
    __shared__ union {
        typename BS::TempStorage scan;
        typename BR::TempStorage red;
    } tmp;
    __shared__ bool s_last;
    const int64_t i0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kSiItems;
    uint64_t x[kSiItems];
    load8(s, i0, a.N, x);
    const unsigned hm = heads8(s, i0, a.N, x);
    const int32_t cnt = __popc(hm);
    const int32_t my_last = hm ? (int32_t)(i0 + 31 - __clz(hm)) : -1;
    int32_t hb, tot;
    BS(tmp.scan).ExclusiveSum(cnt, hb, tot);
    __syncthreads();
    const int32_t last = BR(tmp.red).Reduce(my_last, cub::Max());
    if (threadIdx.x == 0) {
        a.tile_heads[blockIdx.x] = tot;
        a.tile_last[blockIdx.x] = last;
    }
    if (i0 < a.N) {
        // packs whose first item falls in [i0, i0 + 8): their first row = heads before it
        int lo = 0, hi = a.P + 1;  // first p with pack_gstart[p] >= i0
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(a.pack_gstart + mid) < i0) lo = mid + 1; else hi = mid;
        }
        for (int p = lo; p <= a.P; ++p) {
            const int64_t G0 = __ldg(a.pack_gstart + p);
            if (G0 >= i0 + kSiItems || G0 >= a.N) break;
            a.pack_hb[p] = hb + __popc(hm & ((1u << (int)(G0 - i0)) - 1u));
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.long_cnt + a.P, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    si_scan_body<kSiThreads>(a, gridDim.x, tmp.scan);
}

// one block: the same scan for an empty step (no k_si_heads)
__global__ void __launch_bounds__(1024) k_si_scan(SortIdxArgs a, int64_t nblk) {
    __shared__ typename cub::BlockScan<int32_t, 1024>::TempStorage tmp;
    si_scan_body<1024>(a, nblk, tmp);
}

// tile of cost c in [0, C): floor(c * nte / C) in double (monotone in c; nte <= C, so consecutive
// costs never skip a tile; the k_csr_tiles partition up to rounding at the cuts)
__device__ __forceinline__ int64_t si_tile_of(int64_t c, double scale, int64_t nte) {
    const int64_t k = (int64_t)((double)c * scale);
    return k < nte ? k : nte - 1;
}

__global__ void __launch_bounds__(kSiThreads, 3) k_si_final(SortIdxArgs a, const uint64_t *s) {
    using BS = cub::BlockScan<int32_t, kSiThreads>;
    __shared__ typename BS::TempStorage tmp;
    // the tile's outputs staged in shared memory, then stored with consecutive threads on
    // consecutive addresses (per-thread scattered stores of the row starts / keys and half-used
    // 32-B sectors of su / sseg made k_si_final L2-store bound: 247 M sectors per launch at C3)
    __shared__ __align__(16) int32_t s_su[kTile], s_seg[kTile], s_us[kTile];
    __shared__ __align__(16) unsigned long long s_key[kTile];
    __shared__ int32_t s_nh;
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    const int64_t i0 = t0 + (int64_t)threadIdx.x * kSiItems;
    uint64_t x[kSiItems];
    load8(s, i0, a.N, x);
    const unsigned hm = heads8(s, i0, a.N, x);
    int32_t hb, nh;
    BS(tmp).ExclusiveSum(__popc(hm), hb, nh);
    if (threadIdx.x == 0) s_nh = nh;
    int32_t out_r[kSiItems], out_s[kSiItems];
#pragma unroll
    for (int k = 0; k < kSiItems; ++k)  // segments first: eight independent gathers in flight
        out_s[k] = i0 + k < a.N ? __ldg(a.seg_of + (uint32_t)x[k]) : 0;
    const int32_t rb = __ldg(a.run_base + blockIdx.x);
    int32_t r = rb + hb - 1;  // the row the thread's first items continue
    int hl = hb;              // tile-local index of the thread's next head
#pragma unroll
    for (int k = 0; k < kSiItems; ++k) {
        if (i0 + k < a.N && ((hm >> k) & 1u)) {
            ++r;
            s_us[hl] = (int32_t)(i0 + k);
            s_key[hl] = x[k] >> 32;
            ++hl;
        }
        out_r[k] = r;
    }
    if (a.inv_run) {  // the run-order inverse (row-sharded peer-memory steps): position -> row
#pragma unroll
        for (int k = 0; k < kSiItems; ++k)
            if (i0 + k < a.N) a.inv_run[(uint32_t)x[k]] = out_r[k];
    }
    const int lt = threadIdx.x * kSiItems;
#pragma unroll
    for (int k = 0; k < kSiItems; ++k) {
        s_su[lt + k] = out_r[k];
        s_seg[lt + k] = out_s[k];
    }
    if (a.tile_start && i0 < a.N) {  // the backward's equal-cost tiles (k_csr_tiles): tile of each item's cost
        const int64_t rw = a.rw;
        int64_t G0 = 0, G1 = -1, U0 = 0, nte = 1, kp = -1;
        double scale = 0.0;
        int32_t *ts = nullptr;
#pragma unroll
        for (int k = 0; k < kSiItems; ++k) {
            const int64_t i = i0 + k;
            if (i >= a.N) continue;
            const bool head = (hm >> k) & 1u;
            if (i >= G1) {  // (re)locate: the last pack starting at or before i (skips empty packs)
                int l = 0, h = a.P;
                while (h - l > 1) {
                    const int mid = (l + h) >> 1;
                    if (__ldg(a.pack_gstart + mid) <= i) l = mid; else h = mid;
                }
                G0 = __ldg(a.pack_gstart + l);
                G1 = __ldg(a.pack_gstart + l + 1);
                U0 = __ldg(a.pack_ustart + l);
                const int64_t C = (G1 - G0) + rw * (__ldg(a.pack_ustart + l + 1) - U0);
                nte = a.nt < C ? a.nt : C;
                scale = (double)nte / (double)C;
                ts = a.tile_start + (int64_t)l * (a.nt + 1);
                const int64_t c0 = (i - G0) + rw * (out_r[k] - U0);  // the previous item's tile
                kp = i > G0 ? si_tile_of(c0 - (head ? 1 + rw : 1), scale, nte) : -1;
            }
            const int64_t kt = si_tile_of((i - G0) + rw * (out_r[k] - U0), scale, nte);
            for (int64_t kk = kp + 1; kk <= kt; ++kk) ts[kk] = (int32_t)i;
            if (i == G1 - 1)
                for (int64_t kk = kt + 1; kk <= a.nt; ++kk) ts[kk] = (int32_t)G1;
            kp = kt;
        }
    }
    __syncthreads();
    const int nt = (int)(a.N - t0 < kTile ? a.N - t0 : kTile);
    nh = s_nh;
    if (nt == kTile && ((uintptr_t)(a.su + t0) & 15) == 0 && ((uintptr_t)(a.sseg + t0) & 15) == 0) {
        for (int q = threadIdx.x; q < kTile / 4; q += kSiThreads) {
            reinterpret_cast<int4 *>(a.su + t0)[q] = reinterpret_cast<const int4 *>(s_su)[q];
            reinterpret_cast<int4 *>(a.sseg + t0)[q] = reinterpret_cast<const int4 *>(s_seg)[q];
        }
    } else {
        for (int q = threadIdx.x; q < nt; q += kSiThreads) {
            a.su[t0 + q] = s_su[q];
            a.sseg[t0 + q] = s_seg[q];
        }
    }
    for (int q = threadIdx.x; q < nh; q += kSiThreads) {  // rows starting in this tile: rb .. rb + nh
        a.ustart[rb + q] = s_us[q];
        a.run_key[rb + q] = s_key[q];
    }
}

// ---- the reading-O1 views (on request) ------------------------------------------------------
__global__ void __launch_bounds__(kSiThreads) k_sv_heads(SortIdxArgs a, const uint64_t *s) {
    const int64_t i0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kSiItems;
    if (i0 >= a.N) return;
    uint64_t x[kSiItems];
    load8(s, i0, a.N, x);
    const unsigned hm = heads8(s, i0, a.N, x);
#pragma unroll
    for (int k = 0; k < kSiItems; ++k)
        if ((hm >> k) & 1u) {
            const uint32_t g = (uint32_t)x[k];
            atomicOr(a.bm + (g >> 5), 1u << (g & 31));
        }
}

// first occurrences per 2048-position tile (64 bitmap words, one warp per tile)
__global__ void __launch_bounds__(256) k_bm_count(const uint32_t *bm, int64_t nwords, int32_t *cnt, int64_t nblk) {
    const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t >= nblk) return;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = t * 64 + lane * 2;
    int32_t c = (w0 < nwords ? __popc(bm[w0]) : 0) + (w0 + 1 < nwords ? __popc(bm[w0 + 1]) : 0);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[t] = c;
}

__global__ void __launch_bounds__(1024) k_bm_scan(const int32_t *cnt, int32_t *pref, int64_t nblk) {
    using BS = cub::BlockScan<int32_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nblk; base += 1024) {
        const int64_t i = base + threadIdx.x;
        int32_t e, agg;
        BS(tmp).ExclusiveSum(i < nblk ? cnt[i] : 0, e, agg);
        if (i < nblk) pref[i] = carry + e;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
}

// rank of every bitmap word: first occurrences before it
__global__ void __launch_bounds__(256) k_bm_prefix(const uint32_t *bm, int64_t nwords, const int32_t *bm_pref,
                                                   int32_t *wpref, int64_t nblk) {
    const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t >= nblk) return;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = t * 64 + lane * 2;
    const int32_t c0 = w0 < nwords ? __popc(bm[w0]) : 0;
    const int32_t c1 = w0 + 1 < nwords ? __popc(bm[w0 + 1]) : 0;
    int32_t x = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const int32_t e = bm_pref[t] + x - (c0 + c1);
    if (w0 < nwords) wpref[w0] = e;
    if (w0 + 1 < nwords) wpref[w0 + 1] = e + c0;
}

// uid of first occurrence g: first occurrences before g
__device__ __forceinline__ int32_t sv_rank(const SortIdxArgs &a, uint32_t g) {
    const uint32_t w = g >> 5;
    return __ldg(a.wpref + w) + __popc(__ldg(a.bm + w) & ((1u << (g & 31)) - 1u));
}

// inverse[g] = uid of g's run; Unique in first-occurrence order
__global__ void __launch_bounds__(kSiThreads) k_sv_final(SortIdxArgs a, const uint64_t *s) {
    using BS = cub::BlockScan<int32_t, kSiThreads>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t i0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kSiItems;
    uint64_t x[kSiItems];
    load8(s, i0, a.N, x);
    const unsigned hm = heads8(s, i0, a.N, x);
    const int32_t my_last = hm ? (int32_t)(i0 + 31 - __clz(hm)) : -1;
    int32_t lastb;
    BS(tmp).ExclusiveScan(my_last, lastb, cub::Max());
    if (threadIdx.x == 0) lastb = -1;
    if (i0 >= a.N) return;
    int32_t uid = 0;
    if (!(hm & 1u)) {  // the run the thread's first items continue: its head's first position
        const int64_t h = lastb >= 0 ? lastb : __ldg(a.carry + blockIdx.x);
        uid = sv_rank(a, (uint32_t)ld_item(s, h));
    }
#pragma unroll
    for (int k = 0; k < kSiItems; ++k) {
        if (i0 + k >= a.N) continue;
        const uint32_t g = (uint32_t)x[k];
        if ((hm >> k) & 1u) {
            uid = sv_rank(a, g);
            a.unique_gkey[uid] = x[k] >> 32;
        }
        a.inverse[g] = uid;
    }
}

// uid of each row (run order): the rank of its head's first position
__global__ void k_sv_run_uid(SortIdxArgs a, const uint64_t *s) {
    const int32_t U = *a.d_total;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < U; r += (int64_t)gridDim.x * blockDim.x)
        a.run_uid[r] = sv_rank(a, (uint32_t)ld_item(s, __ldg(a.ustart + r)));
}

__global__ void k_run_gather(const int32_t *run_uid, const int32_t *d_total, const int32_t *hslot, int32_t *hs_run,
                             const int64_t *row_off, int64_t *ro_run, const int32_t *dst_rank, int32_t *dr_run,
                             const int64_t *dst_off, int64_t *do_run) {
    const int32_t U = *d_total;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < U; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = __ldg(run_uid + r);
        if (hslot) hs_run[r] = hslot[u];
        if (row_off) ro_run[r] = row_off[u];
        if (dst_rank) dr_run[r] = dst_rank[u];
        if (dst_off) do_run[r] = dst_off[u];
    }
}

__global__ void k_unpack_pairs(const uint64_t *items, int64_t n, int32_t *k_out, int32_t *v_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = ld_item(items, i);
        k_out[i] = (int32_t)(x >> 32);
        v_out[i] = (int32_t)(uint32_t)x;
    }
}

}  // namespace

// The hash index's transpose (stable sort of (uid, segment) pairs by uid) through the same chunked
// LSD passes: for large sorts they beat the per-tile-histogram passes of k_sort2.cu, whose digit-
// major [1024, N / 2048] histograms and their scans are re-read every pass.
int sort_pairs_chunked(const int32_t *k_in, const int32_t *v_in, uint64_t *buf_a, uint64_t *buf_b, int32_t **k_out,
                       int32_t **v_out, int64_t n, int key_bits, int32_t *hist, int32_t *rowtot, int num_sms,
                       cudaStream_t s) {
    SortIdxArgs a{};
    a.N = n;
    a.keys = reinterpret_cast<uint32_t *>(const_cast<int32_t *>(k_in));
    a.vals = v_in;
    a.hist = hist;
    a.rowtot = rowtot;
    const SortIdxPlan plan = make_sortidx_plan(n, key_bits, num_sms);
    a.chunk = plan.chunk;
    a.nc = plan.nc;
    uint64_t *bufs[2] = {buf_a, buf_b};
    const uint64_t *cur = nullptr;
    int launches = 0;
    for (int p = 0; p < plan.passes; ++p) {
        uint64_t *out = bufs[p & 1];
        if (p == 0) k_si_up<true><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, nullptr, plan.shift[p], plan.bits[p]);
        else k_si_up<false><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, cur, plan.shift[p], plan.bits[p]);
        bucket_scan(a.hist, a.nc, a.rowtot, 1 << plan.bits[p], s);
        if (p == 0) k_si_down<true><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, nullptr, out, plan.shift[p], plan.bits[p]);
        else k_si_down<false><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, cur, out, plan.shift[p], plan.bits[p]);
        cur = out;
        launches += 3;
    }
    int32_t *ko = reinterpret_cast<int32_t *>(cur == buf_a ? buf_b : buf_a);
    *k_out = ko;
    *v_out = ko + n;
    k_unpack_pairs<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 16), 256, 0, s>>>(cur, n, ko, ko + n);
    return launches + 1;
}

SortIdxPlan make_sortidx_plan(int64_t n, int key_bits, int num_sms) {
    SortIdxPlan p{};
    p.passes = std::max(1, (key_bits + kSiBits - 1) / kSiBits);
    int shift = 0;
    for (int i = 0; i < p.passes; ++i) {  // even digit widths
        const int b = (key_bits - shift + (p.passes - i) - 1) / (p.passes - i);
        p.bits[i] = std::max(b, 1);
        p.shift[i] = shift;
        shift += b;
    }
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const int64_t target = std::max<int64_t>(1, (int64_t)num_sms * 3);  // k_si_down: 3 CTAs per SM
    const int64_t tpc = std::max<int64_t>(1, (ntiles + target - 1) / target);
    p.chunk = tpc * kTile;
    p.nc = (int32_t)std::max<int64_t>(1, (n + p.chunk - 1) / p.chunk);
    return p;
}

size_t sortidx_scratch_ints(int64_t n, int32_t P) {
    const int64_t nblk = (n + kTile - 1) / kTile + 1;
    return (size_t)(5 * nblk + (P + 1) + 64 + (n + 31) / 32 + 2);
}

int launch_sort_index(SortIdxArgs a, const SortIdxPlan &plan, uint64_t *buf_a, uint64_t *buf_b, uint64_t **sorted,
                      uint64_t **other, cudaStream_t s) {
    int launches = 0;
    a.chunk = plan.chunk;
    a.nc = plan.nc;
    const int64_t nblk = (a.N + kTile - 1) / kTile;
    uint64_t *bufs[2] = {buf_a, buf_b};
    const uint64_t *cur = nullptr;
    cudaMemsetAsync(a.long_cnt, 0, sizeof(int32_t) * (a.P + 1), s);  // (+ the k_si_heads ticket)
    if (a.N > 0) {
        for (int p = 0; p < plan.passes; ++p) {
            uint64_t *out = bufs[p & 1];
            if (p == 0) k_si_up<true><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, nullptr, plan.shift[p], plan.bits[p]);
            else k_si_up<false><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, cur, plan.shift[p], plan.bits[p]);
            bucket_scan(a.hist, a.nc, a.rowtot, 1 << plan.bits[p], s);
            if (p == 0) k_si_down<true><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, nullptr, out, plan.shift[p], plan.bits[p]);
            else k_si_down<false><<<(unsigned)a.nc, kSiThreads, 0, s>>>(a, cur, out, plan.shift[p], plan.bits[p]);
            cur = out;
            launches += 3;
        }
        int32_t *su = reinterpret_cast<int32_t *>(cur == buf_a ? buf_b : buf_a);
        a.su = su;
        a.sseg = su + a.N;
        k_si_heads<<<(unsigned)nblk, kSiThreads, 0, s>>>(a, cur);  // (+ the scan, in its last CTA)
        k_si_final<<<(unsigned)nblk, kSiThreads, 0, s>>>(a, cur);
        launches += 2;
    } else {
        cudaMemsetAsync(a.d_total, 0, sizeof(int32_t), s);
        k_si_scan<<<1, 1024, 0, s>>>(a, 0);  // empty packs, ustart[0] = 0
        launches += 1;
    }
    *sorted = const_cast<uint64_t *>(cur);
    *other = cur == buf_a ? buf_b : buf_a;
    return launches;
}

int launch_sort_views(SortIdxArgs a, const uint64_t *sorted, cudaStream_t s) {
    if (a.N <= 0 || !sorted) return 0;
    const int64_t nblk = (a.N + kTile - 1) / kTile;
    const int64_t nwords = (a.N + 31) / 32;
    cudaMemsetAsync(a.bm, 0, sizeof(uint32_t) * nwords, s);
    int32_t *bm_cnt = a.view_scratch, *bm_pref = a.view_scratch + nblk;
    k_sv_heads<<<(unsigned)nblk, kSiThreads, 0, s>>>(a, sorted);
    k_bm_count<<<(unsigned)((nblk + 7) / 8), 256, 0, s>>>(a.bm, nwords, bm_cnt, nblk);
    k_bm_scan<<<1, 1024, 0, s>>>(bm_cnt, bm_pref, nblk);
    k_bm_prefix<<<(unsigned)((nblk + 7) / 8), 256, 0, s>>>(a.bm, nwords, bm_pref, a.wpref, nblk);
    k_sv_final<<<(unsigned)nblk, kSiThreads, 0, s>>>(a, sorted);
    if (a.run_uid) k_sv_run_uid<<<(unsigned)std::min<int64_t>((a.N + 255) / 256, 4096), 256, 0, s>>>(a, sorted);
    return a.run_uid ? 7 : 6;
}

void launch_run_gather(const int32_t *run_uid, const int32_t *d_total, int64_t n_max, const int32_t *hslot,
                       int32_t *hs_run, const int64_t *row_off, int64_t *ro_run, const int32_t *dst_rank,
                       int32_t *dr_run, const int64_t *dst_off, int64_t *do_run, int num_sms, cudaStream_t s) {
    if (n_max <= 0) return;
    k_run_gather<<<(unsigned)std::min<int64_t>((n_max + 255) / 256, (int64_t)num_sms * 8), 256, 0, s>>>(
        run_uid, d_total, hslot, hs_run, row_off, ro_run, dst_rank, dr_run, dst_off, do_run);
}

}  // namespace picasso
