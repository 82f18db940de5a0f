// k_sort2.cu — the backward's transpose: stable LSD radix sort of (uid, segment) pairs with
// passes of up to 10 bits and two launches per pass.
//
// The backward needs, per unique row, its occurrences in ascending packed
// position: a stable sort of the forward's inverse index by uid.  Per pass:
//   k_scan_rows    : one block per digit scans its row of the digit-major per-tile histogram
//                    (exclusive, in place), writes the digit total, and zeroes the same row of
//                    the other histogram buffer for the next pass;
//   k_scatter2     : every block scans the digit totals (<= 1024) in shared memory, ranks its
//                    2048 keys stably (each warp takes 256 contiguous keys in 8 rounds of
//                    __match_any_sync), scatters them, and — when another pass follows — adds
//                    each key's next digit to the next pass's histogram of the tile it lands in.
// The first pass's histogram comes from k_inverse, so a 2-pass sort is 4 launches.
#include <cub/block/block_scan.cuh>

#include <cstdlib>
#include <string>

#include "kernels.h"

namespace picasso {

SortPlan make_sort_plan(int64_t n) {
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < n) ++bits;  // keys (uids) < U <= n
    SortPlan p{};
    p.passes = (bits + kMaxRadixBits - 1) / kMaxRadixBits;
    int shift = 0;
    for (int i = 0; i < p.passes; ++i) {
        const int b = (bits - shift + (p.passes - i) - 1) / (p.passes - i);
        p.bits[i] = b;
        p.shift[i] = shift;
        shift += b;
    }
    return p;
}

size_t radix_hist2_ints(int64_t n) { return (size_t)kMaxRadix * (size_t)((n + kTile - 1) / kTile) + 1; }

// one warp per digit row: rows are short (nblk = N / 2048 tiles), so a warp-level scan with a
// running carry keeps 8 rows per 256-thread block busy instead of idling 1024 threads per row
__global__ void __launch_bounds__(256) k_scan_rows(int32_t *hist, int64_t nblk, int32_t *rowtot, int32_t *zero_next,
                                                   int radix, int next_radix) {
    const int lane = threadIdx.x & 31;
    const int d = blockIdx.x * 8 + (threadIdx.x >> 5);
    constexpr int kRegRow = 16;  // rows up to 32 x 16 entries: every load issued at once
    if (d < radix && nblk <= 32 * kRegRow) {
        int32_t *row = hist + (int64_t)d * nblk;
        const int64_t k0 = (int64_t)lane * kRegRow;  // this lane's consecutive entries
        int32_t v[kRegRow], sum = 0;
#pragma unroll
        for (int j = 0; j < kRegRow; ++j) {
            v[j] = k0 + j < nblk ? row[k0 + j] : 0;
            sum += v[j];
        }
        int32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int32_t run = x - sum;
#pragma unroll
        for (int j = 0; j < kRegRow; ++j)
            if (k0 + j < nblk) {
                row[k0 + j] = run;
                run += v[j];
            }
        if (lane == 31) rowtot[d] = x;
    } else if (d < radix) {
        int32_t *row = hist + (int64_t)d * nblk;
        int32_t carry = 0;
        for (int64_t base = 0; base < nblk; base += 32) {
            const int64_t i = base + lane;
            const int32_t v = i < nblk ? row[i] : 0;
            int32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (i < nblk) row[i] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) rowtot[d] = carry;
    }
    if (zero_next && d < next_radix)  // the next pass's histogram row of the same index
        for (int64_t i = lane; i < nblk; i += 32) zero_next[(int64_t)d * nblk + i] = 0;
}

__global__ void __launch_bounds__(kTileThreads) k_scatter2(const int32_t *kin, const int32_t *vin, int32_t *kout,
                                                           int32_t *vout, int64_t n, int shift, int bits,
                                                           const int32_t *hist_off, const int32_t *rowtot,
                                                           int64_t nblk, int32_t *hist_next, int next_shift,
                                                           int next_bits, const int32_t *n_dev) {
    if (n_dev) n = *n_dev;  // device-side element count (tiles past it are empty)
    constexpr int kWarps = kTileThreads / 32;
    constexpr int kRounds = kTile / kTileThreads;  // 8 rounds of 32 keys per warp
    __shared__ int32_t wc[kWarps][kMaxRadix];
    __shared__ int32_t dbase[kMaxRadix];
    using BlockScan = cub::BlockScan<int32_t, kTileThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    const int radix = 1 << bits;
    const unsigned dmask = (unsigned)radix - 1u;
    for (int i = threadIdx.x; i < kWarps * kMaxRadix; i += kTileThreads) (&wc[0][0])[i] = 0;
    {   // digit bases: exclusive scan of the digit totals (radix <= 1024 = 4 per thread)
        constexpr int PER = kMaxRadix / kTileThreads;
        int32_t v[PER], s = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int d = threadIdx.x * PER + i;
            v[i] = d < radix ? rowtot[d] : 0;
            s += v[i];
        }
        int32_t e;
        BlockScan(tmp).ExclusiveSum(s, e);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            dbase[threadIdx.x * PER + i] = e;
            e += v[i];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * (32 * kRounds);
    int32_t key[kRounds], val[kRounds], rk[kRounds];
    int dg[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // all loads first: 16 independent requests in flight
        const int64_t g = base + r * 32 + lane;
        key[r] = g < n ? __ldg(kin + g) : 0;
        val[r] = g < n ? __ldg(vin + g) : 0;
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t g = base + r * 32 + lane;
        const bool valid = g < n;
        dg[r] = valid ? (int)(((unsigned)key[r] >> shift) & dmask) : (kMaxRadix + lane);
        const unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
        int32_t before = 0;
        if (valid) before = wc[w][dg[r]];
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wc[w][dg[r]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kTileThreads) {  // prefix across warps + global offset
        int32_t run = dbase[d] + hist_off[(int64_t)d * nblk + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
            const int32_t t = wc[ww][d];
            wc[ww][d] = run;
            run += t;
        }
    }
    __syncthreads();
    const unsigned nmask = (1u << next_bits) - 1u;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t g = base + r * 32 + lane;
        const bool valid = g < n;
        int32_t pos = 0;
        if (valid) {
            pos = wc[w][dg[r]] + rk[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
        if (hist_next) {  // next pass: digit of this key in the tile it lands in
            const unsigned vm = __ballot_sync(0xffffffffu, valid);
            if (valid) {
                const int64_t slot = (int64_t)(((unsigned)key[r] >> next_shift) & nmask) * nblk + pos / kTile;
                const unsigned peers = __match_any_sync(vm, (unsigned long long)slot);
                if (lane == __ffs(peers) - 1) atomicAdd(hist_next + slot, (int32_t)__popc(peers));
            }
        }
    }
}

// Same pass with coalesced writes: the tile is first sorted by digit in shared memory (stable),
// then written out in that order, so consecutive threads store consecutive positions of a digit's
// run instead of scattering one key per digit run per warp.
__global__ void __launch_bounds__(kTileThreads) k_scatter3(const int32_t *kin, const int32_t *vin, int32_t *kout,
                                                           int32_t *vout, int64_t n, int shift, int bits,
                                                           const int32_t *hist_off, const int32_t *rowtot,
                                                           int64_t nblk, int32_t *hist_next, int next_shift,
                                                           int next_bits, const int32_t *n_dev) {
    if (n_dev) n = *n_dev;
    constexpr int kWarps = kTileThreads / 32;
    constexpr int kRounds = kTile / kTileThreads;
    constexpr int PER = kMaxRadix / kTileThreads;
    extern __shared__ int32_t sm3[];
    const int radix = 1 << bits;
    int32_t *wc = sm3;                           // [kWarps][radix]
    int32_t *gbase = wc + kWarps * radix;        // [radix] global start of this tile's digit run
    int32_t *tstart = gbase + radix;             // [radix] tile-local start of the digit run
    int32_t *sk = tstart + radix;                // [kTile] staged keys
    int32_t *sv = sk + kTile;                    // [kTile] staged values
    using BlockScan = cub::BlockScan<int32_t, kTileThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    const unsigned dmask = (unsigned)radix - 1u;
    for (int i = threadIdx.x; i < kWarps * radix; i += kTileThreads) wc[i] = 0;
    {   // global digit starts: exclusive scan of the digit totals + this tile's offset
        int32_t v[PER], s = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int d = threadIdx.x * PER + i;
            v[i] = d < radix ? rowtot[d] : 0;
            s += v[i];
        }
        int32_t e;
        BlockScan(tmp).ExclusiveSum(s, e);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int d = threadIdx.x * PER + i;
            if (d < radix) gbase[d] = e + hist_off[(int64_t)d * nblk + blockIdx.x];
            e += v[i];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t tile0 = (int64_t)blockIdx.x * kTile;
    const int64_t base = tile0 + (int64_t)w * (32 * kRounds);
    int32_t key[kRounds], val[kRounds], rk[kRounds];
    int dg[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t g = base + r * 32 + lane;
        key[r] = g < n ? __ldg(kin + g) : 0;
        val[r] = g < n ? __ldg(vin + g) : 0;
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // stable rank within the warp's digit run
        const int64_t g = base + r * 32 + lane;
        const bool valid = g < n;
        dg[r] = valid ? (int)(((unsigned)key[r] >> shift) & dmask) : (kMaxRadix + lane);
        const unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
        int32_t before = 0;
        if (valid) before = wc[w * radix + dg[r]];
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wc[w * radix + dg[r]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // per digit: warp prefixes (in place) and the tile total; then tile-local digit starts
        int32_t tot[PER], s = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int d = threadIdx.x * PER + i;
            int32_t run = 0;
            if (d < radix)
#pragma unroll
                for (int ww = 0; ww < kWarps; ++ww) {
                    const int32_t t = wc[ww * radix + d];
                    wc[ww * radix + d] = run;
                    run += t;
                }
            tot[i] = run;
            s += run;
        }
        int32_t e;
        BlockScan(tmp).ExclusiveSum(s, e);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int d = threadIdx.x * PER + i;
            if (d < radix) tstart[d] = e;
            e += tot[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // stage in digit order (stable)
        const int64_t g = base + r * 32 + lane;
        if (g < n) {
            const int lp = tstart[dg[r]] + wc[w * radix + dg[r]] + rk[r];
            sk[lp] = key[r];
            sv[lp] = val[r];
        }
    }
    __syncthreads();
    const int nt = (int)(n - tile0 < kTile ? n - tile0 : kTile);
    const unsigned nmask = (1u << next_bits) - 1u;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // consecutive threads -> consecutive positions of a run
        const int i = r * kTileThreads + threadIdx.x;
        const bool valid = i < nt;
        int32_t pos = 0, k = 0;
        if (valid) {
            k = sk[i];
            const int d = (int)(((unsigned)k >> shift) & dmask);
            pos = gbase[d] + (i - tstart[d]);
            kout[pos] = k;
            vout[pos] = sv[i];
        }
        if (hist_next) {
            const unsigned vm = __ballot_sync(0xffffffffu, valid);
            if (valid) {
                const int64_t slot = (int64_t)(((unsigned)k >> next_shift) & nmask) * nblk + pos / kTile;
                const unsigned peers = __match_any_sync(vm, (unsigned long long)slot);
                if (lane == __ffs(peers) - 1) atomicAdd(hist_next + slot, (int32_t)__popc(peers));
            }
        }
    }
}

size_t scatter3_smem(int bits) { return sizeof(int32_t) * ((size_t)(kTileThreads / 32 + 2) * (1u << bits) + 2 * kTile); }

// Next pass's digit histogram of every 2048-key tile of a pass's output (large sorts: cheaper
// than the scatter's per-key global atomics once the key count is in the millions).
__global__ void __launch_bounds__(kTileThreads) k_hist_tiles(const int32_t *keys, int64_t n, int shift, int bits,
                                                             int32_t *hist, int64_t nblk) {
    __shared__ int32_t h[kMaxRadix];
    const int radix = 1 << bits;
    for (int d = threadIdx.x; d < radix; d += kTileThreads) h[d] = 0;
    __syncthreads();
    const unsigned dmask = (unsigned)radix - 1u;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kTile; i += kTileThreads) {
        const int64_t g = (int64_t)blockIdx.x * kTile + i;
        const bool valid = g < n;
        const int d = valid ? (int)(((unsigned)__ldg(keys + g) >> shift) & dmask) : 0;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(vm, d);
            if (lane == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kTileThreads) hist[(int64_t)d * nblk + blockIdx.x] = h[d];
}

constexpr int64_t kBigSort = (int64_t)1 << 22;  // from here on the next histogram is its own pass
constexpr int64_t kChunkedSort = (int64_t)1 << 20;  // from here on: the chunked passes (k_sortidx.cu)

void radix_sort_pairs2(const int32_t *k_in, const int32_t *v_in, int32_t *k_a, int32_t *v_a, int32_t *k_b,
                       int32_t *v_b, int32_t **k_out, int32_t **v_out, int64_t n, const SortPlan &plan,
                       int32_t *hist0, int32_t *hist1, int32_t *rowtot, cudaStream_t s, int64_t *launches) {
    const int64_t nblk = (n + kTile - 1) / kTile;
    // large sorts: the chunked LSD passes of k_sortidx.cu ((k_a, v_a) and (k_b, v_b) are adjacent:
    // 8-byte item buffers); PICASSO_SORT=2 / 3 keep these passes
    static const char *sort_env0 = std::getenv("PICASSO_SORT");
    if (n >= kChunkedSort && !sort_env0 && v_a == k_a + n && v_b == k_b + n) {
        static int num_sms = [] {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            return sms;
        }();
        int bits = 0;
        for (int i = 0; i < plan.passes; ++i) bits += plan.bits[i];
        *launches += sort_pairs_chunked(k_in, v_in, reinterpret_cast<uint64_t *>(k_a), reinterpret_cast<uint64_t *>(k_b),
                                        k_out, v_out, n, bits, hist0, rowtot, num_sms, s);
        return;
    }
    const int32_t *ck = k_in, *cv = v_in;
    int32_t *bufk[2] = {k_a, k_b}, *bufv[2] = {v_a, v_b};
    int32_t *hist[2] = {hist0, hist1};
    if (nblk == 0) {
        *k_out = const_cast<int32_t *>(ck);
        *v_out = const_cast<int32_t *>(cv);
        return;
    }
    for (int p = 0; p < plan.passes; ++p) {
        const bool more = p + 1 < plan.passes;
        const int radix = 1 << plan.bits[p];
        const int next_radix = more ? 1 << plan.bits[p + 1] : 0;
        const int rows = radix > next_radix ? radix : next_radix;
        k_scan_rows<<<(rows + 7) / 8, 256, 0, s>>>(hist[p & 1], nblk, rowtot, more ? hist[(p + 1) & 1] : nullptr,
                                                   radix, next_radix);
        const bool fused_hist = more && n < kBigSort;
        // staged (coalesced) scatter for large sorts; below kBigSort the direct scatter is faster
        // (C2: 13.5 vs 14.7 us per pass).  PICASSO_SORT=2 / 3 forces one.
        static const char *sort_env = std::getenv("PICASSO_SORT");
        const bool v3 = sort_env ? std::string(sort_env) == "3" : n >= kBigSort;
        if (v3) {
            const size_t sm = scatter3_smem(plan.bits[p]);
            ensure_dyn_smem((const void *)k_scatter3, scatter3_smem(kMaxRadixBits));
            k_scatter3<<<(unsigned)nblk, kTileThreads, sm, s>>>(ck, cv, bufk[p & 1], bufv[p & 1], n, plan.shift[p],
                                                                plan.bits[p], hist[p & 1], rowtot, nblk,
                                                                fused_hist ? hist[(p + 1) & 1] : nullptr,
                                                                more ? plan.shift[p + 1] : 0,
                                                                more ? plan.bits[p + 1] : 0, nullptr);
        } else {
            k_scatter2<<<(unsigned)nblk, kTileThreads, 0, s>>>(ck, cv, bufk[p & 1], bufv[p & 1], n, plan.shift[p],
                                                              plan.bits[p], hist[p & 1], rowtot, nblk,
                                                              fused_hist ? hist[(p + 1) & 1] : nullptr,
                                                              more ? plan.shift[p + 1] : 0,
                                                              more ? plan.bits[p + 1] : 0, nullptr);
        }
        *launches += 2;
        if (more && !fused_hist) {
            k_hist_tiles<<<(unsigned)nblk, kTileThreads, 0, s>>>(bufk[p & 1], n, plan.shift[p + 1], plan.bits[p + 1],
                                                                 hist[(p + 1) & 1], nblk);
            *launches += 1;
        }
        ck = bufk[p & 1];
        cv = bufv[p & 1];
    }
    *k_out = const_cast<int32_t *>(ck);
    *v_out = const_cast<int32_t *>(cv);
}

// Per-tile bucket offsets (exclusive, in place) and bucket totals of a digit-major histogram
// (the peer-memory partition's k_bucket output).
void bucket_scan(int32_t *hist, int64_t nblk, int32_t *rowtot, int radix, cudaStream_t s, int32_t *zero_next,
                 int next_radix) {
    const int rows = radix > next_radix ? radix : next_radix;
    if (nblk > 0) k_scan_rows<<<(rows + 7) / 8, 256, 0, s>>>(hist, nblk, rowtot, zero_next, radix, next_radix);
}

// One stable pass by a small key (the multi-GPU partition by (owner, pack)); bhist was filled
// by k_bucket; rowtot receives the bucket counts.
void bucket_sort_pass(const int32_t *k_in, const int32_t *v_in, int32_t *k_out, int32_t *v_out, int64_t n_max,
                      const int32_t *n_dev, int bits, int32_t *bhist, int32_t *rowtot, cudaStream_t s) {
    const int64_t nblk = (n_max + kTile - 1) / kTile;
    if (nblk == 0) return;
    const int radix = 1 << bits;
    k_scan_rows<<<(radix + 7) / 8, 256, 0, s>>>(bhist, nblk, rowtot, nullptr, radix, 0);
    k_scatter2<<<(unsigned)nblk, kTileThreads, 0, s>>>(k_in, v_in, k_out, v_out, n_max, 0, bits, bhist, rowtot, nblk,
                                                      nullptr, 0, 0, n_dev);
}

}  // namespace picasso
