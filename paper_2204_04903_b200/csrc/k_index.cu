// k_index.cu — ID hashing + fused Unique ("Unique&Partition").
//
// All packs are processed by one launch over the *packed ID stream*: the concatenation, pack
// by pack (ascending pack, then ascending field, then sample b, then j), of every ID of the
// batch (D-Packing's "packed ID tensor", L319-323; kept virtual — position g maps back to
// its field-major index j by a binary search, no copy).
//
//   k_field_prep   : per-field ID ranges and the packed-stream layout (one small block)
//   k_dedup_insert : row mapping, pack key; warp pre-dedup (__match_any_sync) and
//                    one open-addressing insert per distinct key per warp; atomicMin keeps the
//                    first position of every key
//   k_flag_count   : first-occurrence flags, counted per 2048-position tile
//   k_assign       : tile-ordered exclusive scan -> global uid in first-occurrence order;
//                    unique keys; per-pack uid ranges
//   k_inverse      : inverse index (global uid per packed position)
// Unique order is the first-occurrence order of each pack's key stream (reading O1), and
// because packs occupy contiguous position ranges the per-pack uid of a key is its global
// uid minus pack_ustart[p].
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "kernels.h"

namespace picasso {

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_field_prep(IndexArgs a) {
    __shared__ int32_t warp_sums[32];
    __shared__ int32_t carry;
    const int tid = threadIdx.x;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < a.F; base += 1024) {
        const int k = base + tid;
        int32_t len = 0;
        if (k < a.F) {
            const int f = a.pm_fields[k];
            const int32_t s0 = a.offsets[(int64_t)f * a.B];
            const int32_t s1 = a.offsets[(int64_t)(f + 1) * a.B];
            a.id_start[f] = s0;
            len = s1 - s0;
        }
        // block exclusive scan of len
        int32_t x = len;
        const int lane = tid & 31, w = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;  // inclusive
        }
        __syncthreads();
        const int32_t excl = carry + (w ? warp_sums[w - 1] : 0) + x - len;
        if (k < a.F) {
            a.gstart_pm[k] = excl;
            a.field_gstart[a.pm_fields[k]] = excl;
        }
        __syncthreads();
        if (tid == 0) carry += warp_sums[31];
        __syncthreads();
    }
    // offsets must be a CSR over the n_ids IDs (offsets[0] = 0, non-decreasing, offsets[F*B] =
    // n_ids).  Checked at the field boundaries, the layout's only inputs; on a violation the
    // error latches (PICASSO_ERR_INVALID_ARG) and the step runs on a substitute layout whose
    // every position and segment is in range, so no later kernel indexes past the ID, position,
    // output or dY buffers (per-segment kernels also clamp their ranges to [0, n_ids)).  The
    // step's results are then meaningless: the caller must check picasso_last_error.
    __shared__ int bad;
    if (tid == 0) bad = (carry != a.N) || (a.F > 0 && a.offsets[0] != 0);
    __syncthreads();
    for (int f = tid; f < a.F; f += 1024)
        if (a.offsets[(int64_t)(f + 1) * a.B] < a.offsets[(int64_t)f * a.B]) bad = 1;
    __syncthreads();
    if (bad) {  // substitute layout: the first field of the first pack holds all n_ids IDs in one bag
        if (tid == 0) atomicOr(a.err, ERR_OFFSETS);
        for (int k = tid; k < a.F; k += 1024) {
            const int32_t gs = k == 0 ? 0 : (int32_t)a.N;
            a.gstart_pm[k] = gs;
            a.field_gstart[a.pm_fields[k]] = gs;
            a.id_start[a.pm_fields[k]] = 0;
        }
        if (a.F > 0) {
            const int32_t sg0 = a.pm_fields[0] * a.B;
            for (int64_t g = tid; g < a.N; g += 1024) a.seg_of[g] = sg0;
            if (a.keys) {  // every position keys row 0 of that field's table: in range, meaningless
                const FieldInfo fi = a.finfo[a.pm_fields[0]];
                const uint32_t k0 = (uint32_t)(a.pack_key_off[fi.pack] + fi.base);
                for (int64_t g = tid; g < a.N; g += 1024) a.keys[g] = k0;
            }
        }
        if (tid == 0) carry = (int32_t)a.N;
        __syncthreads();
    }
    if (tid == 0 && a.seg_limit) *a.seg_limit = bad ? 0 : (int32_t)a.N;  // k_seg_of: nothing to place
    if (tid == 0) a.gstart_pm[a.F] = carry;
    __syncthreads();
    for (int p = tid; p <= a.P; p += 1024) a.pack_gstart[p] = a.gstart_pm[a.pack_first_k[p]];
    if (a.empty_pack)
        for (int p = tid; p < a.P; p += 1024) a.empty_pack[p] = 0;
    if (!a.region_base) return;
    // per-table hash regions: pow2 >= 2^region_shift x (occurrences of the table's fields), >= 64
    // slots, laid out in table order — the positions of one table are contiguous in the packed
    // stream, so the inserts / flag / assign / inverse passes over a range of positions touch one
    // region at a time, which stays in L2 even when the whole table is gigabytes
    for (int t = tid; t < a.T; t += 1024) a.tocc[t] = 0;
    __syncthreads();
    if (!bad)
        for (int f = tid; f < a.F; f += 1024)
            atomicAdd(a.tocc + a.finfo[f].table,
                      a.offsets[(int64_t)(f + 1) * a.B] - a.offsets[(int64_t)f * a.B]);
    __syncthreads();
    __shared__ int64_t s_carry, wsum64[32];
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base0 = 0; base0 < a.T; base0 += 1024) {  // block scan of the region sizes
        const int t = base0 + tid;
        uint64_t sz = 0;
        if (t < a.T) {
            const int32_t occ = __ldcg(a.tocc + t);
            sz = 64;
            while (sz < ((uint64_t)occ << a.region_shift)) sz <<= 1;
            a.region_mask[t] = (uint32_t)(sz - 1);
        }
        const int lane = tid & 31, w = tid >> 5;
        int64_t x = (int64_t)sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum64[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t y = wsum64[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            wsum64[lane] = y;
        }
        __syncthreads();
        if (t < a.T) a.region_base[t] = s_carry + (w ? wsum64[w - 1] : 0) + x - (int64_t)sz;
        __syncthreads();
        if (tid == 0) s_carry += wsum64[31];
        __syncthreads();
    }
    if (tid == 0) a.region_base[a.T] = s_carry;
}

// the dedup table's used part (the regions) back to empty (0xFF), size from the device
__global__ void k_table_clear(ulonglong2 *table, const int64_t *total) {
    const int64_t n = *total;
    const ulonglong2 e = make_ulonglong2(~0ull, ~0ull);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        table[i] = e;
}

void launch_field_prep(const IndexArgs &a, cudaStream_t s) {
    k_field_prep<<<1, 1024, 0, s>>>(a);
    if (a.region_base)
        k_table_clear<<<1184, 256, 0, s>>>(reinterpret_cast<ulonglong2 *>(a.table), a.region_base + a.T);
}

// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dedup_insert(IndexArgs a) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = g < a.N;
    unsigned long long gkey = 0;
    int32_t tbl = 0;
    bool ok = false;
    if (valid) {
        // packed position -> pm field -> field-major index j (k == F only after an offsets error:
        // k_field_prep then laid every field out empty)
        const int64_t k = upper_bound_dev(a.gstart_pm, 0, a.F + 1, (int32_t)g) - 1;
        if (k < a.F) {
            const int f = __ldg(a.pm_fields + k);
            const int64_t j = (int64_t)__ldg(a.id_start + f) + (g - __ldg(a.gstart_pm + k));
            const FieldInfo fi = a.finfo[f];
            const int64_t row = row_of(a.id_mode, __ldg(a.ids + j), fi, a.err);
            gkey = (unsigned long long)(__ldg(a.pack_key_off + fi.pack) + fi.base + row);
            tbl = fi.table;
            ok = true;
        } else {
            a.slot_of[g] = 0;
        }
    }
    // warp pre-dedup: lanes holding the same key elect the lowest lane (= smallest g)
    const unsigned vmask = __ballot_sync(0xffffffffu, ok);
    if (!ok) return;
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(vmask, gkey);
    const int leader = __ffs(peers) - 1;
    uint32_t slot = 0;
    if (lane == leader) {
        uint32_t rbase = 0, mask = a.cap_mask;
        if (a.region_base) {  // the table's own region (k_field_prep); equal keys: same table
            rbase = (uint32_t)__ldg(a.region_base + tbl);
            mask = __ldg(a.region_mask + tbl);
        }
        uint32_t h = slot_hash(gkey) & mask;
        slot = rbase + h;
        for (uint32_t probe = 0;; ++probe) {
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(&a.table[slot].key);
            if (cur == kEmptyKey) cur = atomicCAS(&a.table[slot].key, kEmptyKey, gkey);
            if (cur == kEmptyKey || cur == gkey) break;
            h = (h + 1) & mask;
            slot = rbase + h;
            if (probe > mask) {  // region full: cannot happen with 2x occurrences
                atomicOr(a.err, ERR_CAPACITY);
                break;
            }
        }
        atomicMin(&a.table[slot].minpos, (unsigned int)g);
    }
    slot = __shfl_sync(vmask, slot, leader);
    a.slot_of[g] = (int32_t)slot;
}

void launch_dedup_insert(const IndexArgs &a, cudaStream_t s) {
    const int64_t nb = (a.N + 255) / 256;
    if (nb) k_dedup_insert<<<(unsigned)nb, 256, 0, s>>>(a);
}

// ------------------------------------------------------------------------------------------
// 1024 threads x 2 positions per 2048-position tile: at C2 there are only ~208 tiles, and the
// passes are latency-bound table lookups, so parallelism comes from threads, not from items
constexpr int kIdxThreads = 1024;
constexpr int kItems = kTile / kIdxThreads;  // consecutive positions per thread
constexpr int kTpb = 8 / kItems;             // threads whose flags share one fmask byte
static_assert(8 % kItems == 0 && 32 % kTpb == 0, "fmask packing");

__global__ void __launch_bounds__(kIdxThreads) k_flag_count(IndexArgs a) {
    using BlockReduce = cub::BlockReduce<int32_t, kIdxThreads>;
    __shared__ typename BlockReduce::TempStorage tmp;
    const int64_t N = a.n_dev ? *a.n_dev : a.N;
    const int64_t g0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    int32_t slot[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) slot[i] = g0 + i < N ? __ldg(a.slot_of + g0 + i) : 0;
    int32_t c = 0;
    uint32_t m = 0;  // first-occurrence flags of this thread's positions (k_assign reads them)
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int64_t g = g0 + i;
        if (g < N && a.table[slot[i]].minpos == (unsigned int)g) {
            ++c;
            m |= 1u << i;
        }
    }
    uint32_t m8 = m;  // 8 positions per byte: kTpb consecutive threads
#pragma unroll
    for (int t = 1; t < kTpb; ++t) m8 |= __shfl_down_sync(0xffffffffu, m, t) << (t * kItems);
    if (threadIdx.x % kTpb == 0 && g0 < N) a.fmask[g0 / 8] = (uint8_t)m8;
    const int32_t tot = BlockReduce(tmp).Sum(c);
    if (threadIdx.x == 0) a.blk_cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kIdxThreads) k_assign(IndexArgs a) {
    using BlockScan = cub::BlockScan<int32_t, kIdxThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    const int64_t N = a.n_dev ? *a.n_dev : a.N;
    const int64_t g0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    int32_t slot[kItems];
    bool first[kItems];
    unsigned long long key[kItems];
    const uint32_t m = g0 < N ? (a.fmask[g0 / 8] >> (g0 % 8)) & ((1u << kItems) - 1u) : 0u;  // k_flag_count's
    const int32_t c = __popc(m);
    // table reads (first occurrences only) before any table write: stores to table[] would
    // otherwise order every later load behind them (possible aliasing)
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        first[i] = (m >> i) & 1u;
        slot[i] = first[i] ? __ldg(a.slot_of + g0 + i) : 0;
        key[i] = first[i] ? a.table[slot[i]].key : 0ull;
    }
    int32_t excl;
    BlockScan(tmp).ExclusiveSum(c, excl);
    int32_t uid = a.blk_off[blockIdx.x] + excl;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if (first[i]) {
            a.table[slot[i]].uid = uid;
            a.unique_gkey[uid] = key[i];
            // the first position of a non-empty pack is always a first occurrence
            const int64_t g = g0 + i;
            const int64_t p = upper_bound_dev(a.pack_gstart, 0, a.P + 1, (int32_t)g) - 1;
            if (p < a.P && __ldg(a.pack_gstart + p) == (int32_t)g) a.pack_ustart[p] = uid;
            ++uid;
        }
    }
}

// inverse[g] = uid; also the digit histogram of the backward's first radix pass over this
// 2048-position tile (digit-major, so the sort starts with its scan: one pass over N saved)
__global__ void __launch_bounds__(kIdxThreads) k_inverse(IndexArgs a) {
    __shared__ int32_t h[kMaxRadix];
    const int radix = 1 << a.sort_bits0;
    for (int d = threadIdx.x; d < radix; d += kIdxThreads) h[d] = 0;
    __syncthreads();
    const int64_t N = a.n_dev ? *a.n_dev : a.N;
    const int64_t g0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    const int lane = threadIdx.x & 31;
    int32_t uids[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) uids[i] = g0 + i < N ? __ldg(a.slot_of + g0 + i) : 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) uids[i] = g0 + i < N ? a.table[uids[i]].uid : 0;  // all lookups in flight
    // a position left out of the dedup (only after an offsets error: k_field_prep) has no uid;
    // 0 keeps the transpose's digits and row starts in range
    const uint32_t U = (uint32_t)*a.d_total;
#pragma unroll
    for (int i = 0; i < kItems; ++i)
        if ((uint32_t)uids[i] >= U) uids[i] = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int64_t g = g0 + i;
        const bool valid = g < N;
        const int32_t uid = uids[i];
        if (valid) a.inverse[g] = uid;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int d = uid & (radix - 1);
            const unsigned peers = __match_any_sync(vm, d);
            if (lane == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    const int64_t nblk = (N + kTile - 1) / kTile;
    if (N > 0 && blockIdx.x < nblk)
        for (int d = threadIdx.x; d < radix; d += kIdxThreads) a.sort_hist0[(int64_t)d * nblk + blockIdx.x] = h[d];
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // uid ranges of empty packs (and the end)
        int32_t next = *a.d_total;
        a.pack_ustart[a.P] = next;
        for (int p = a.P - 1; p >= 0; --p) {
            if (a.pack_gstart[p] == a.pack_gstart[p + 1]) a.pack_ustart[p] = next;
            next = a.pack_ustart[p];
        }
        int64_t gb = 0;  // G-buffer layout of the split backward
        for (int p = 0; p < a.P; ++p) {
            a.pack_gbase[p] = gb;
            gb += (int64_t)(a.pack_ustart[p + 1] - a.pack_ustart[p]) * a.pack_dim[p];
        }
        a.pack_gbase[a.P] = gb;
    }
}

__global__ void k_scan_blocks(const int32_t *cnt, int32_t *off, int32_t n, int32_t *total, const int32_t *n_dev) {
    // single block, n small (N / 2048): chunked sequential scan with block carry
    if (n_dev) n = (*n_dev + kTile - 1) / kTile;
    __shared__ int32_t s_carry;
    using BlockScan = cub::BlockScan<int32_t, 1024>;
    __shared__ typename BlockScan::TempStorage tmp;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + threadIdx.x;
        int32_t v = i < n ? cnt[i] : 0, e, agg;
        BlockScan(tmp).ExclusiveSum(v, e, agg);
        if (i < n) off[i] = s_carry + e;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

void launch_dedup_assign(const IndexArgs &a, cudaStream_t s) {
    const int64_t nb = (a.N + kTile - 1) / kTile;
    if (nb) {
        k_flag_count<<<(unsigned)nb, kIdxThreads, 0, s>>>(a);
        k_scan_blocks<<<1, 1024, 0, s>>>(a.blk_cnt, a.blk_off, (int32_t)nb, a.d_total, a.n_dev);
        k_assign<<<(unsigned)nb, kIdxThreads, 0, s>>>(a);
    } else {
        cudaMemsetAsync(a.d_total, 0, sizeof(int32_t), s);
    }
    k_inverse<<<(unsigned)std::max<int64_t>(1, nb), kIdxThreads, 0, s>>>(a);
}

}  // namespace picasso
