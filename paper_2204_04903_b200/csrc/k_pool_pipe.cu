// k_pool_pipe.cu — fused Gather + Stitch + SegmentReduction as a
// copy pipeline, for row widths D >= 64 (k_pool.cu serves the narrow packs).
//
//   out[b, col(f) + d] = sum_{j in seg(f,b)} W[key_j][d]   (ascending j from +0.0f; mean: / len;
//                                                          empty segment: 0)
//
//   k_seg_of      : segment of every packed-stream position (one thread per segment; the
//                   backward's transpose sorts by it as well)
//   k_pool_pipe   : one warp per tile of packed positions (equal sizes, moved forward to segment
//                   starts so a segment is summed by one warp in ascending j).  Lanes resolve 32
//                   positions at a time (segment -> field, raw ID -> row (HASH / ROWS) or the
//                   received row at W > 1), one round ahead; per ring stage (~4 KB) every lane
//                   issues the LDGSTS copies of its slice of each row into a per-warp
//                   shared-memory ring.  Landed rows are added in order in fp32; a finished
//                   segment is written into its column block of the [B, out_width] output
//                   with streaming stores.  Empty segments (no position to visit) are zeroed
//                   after the tiles, by a grid-stride pass over the segments' offsets in packs
//                   k_seg_of flagged: a warp here would walk them one by one inside its ring
//                   (C4's sparse positional fields: 13 ms).
#include "kernels.h"

namespace picasso {
namespace {

__device__ __forceinline__ void ldgsts16(void *smem, const void *gmem) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void ldgsts_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ldgsts_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kNW = 16, kS = 3, kStageBytes = 4096;
#ifndef PICASSO_CONSUME_ROWS
#define PICASSO_CONSUME_ROWS 4
#endif
constexpr int kConsumeRows = PICASSO_CONSUME_ROWS;  // rows per unrolled consume step

template <int D>
struct PG {
    static constexpr int ROWB = D * 4;
    static constexpr int RS = ROWB >= kStageBytes ? 1 : kStageBytes / ROWB;
    static constexpr int SB = RS * ROWB;
    static constexpr int EPL = D / 32;
    static constexpr int META = kNW * kS * RS * 16;  // per staged row: out offset (8) + segment (4) + pad
    static constexpr int RING_OFF = (META + 127) / 128 * 128;
    static constexpr int SMEM = RING_OFF + kNW * kS * SB;
    static_assert(32 % RS == 0 && (EPL == 2 || EPL % 4 == 0), "lane layout");
};

template <int D>
__device__ __forceinline__ void lane_load(const float *row, int lane, float *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        const float2 x = reinterpret_cast<const float2 *>(row)[lane];
        v[0] = x.x;
        v[1] = x.y;
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q) {
            const float4 x = reinterpret_cast<const float4 *>(row)[q * 32 + lane];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    }
}
template <int D>
__device__ __forceinline__ void lane_store_cs(float *row, int lane, const float *v) {
    constexpr int EPL = D / 32;
    if constexpr (EPL == 2) {
        __stcs(reinterpret_cast<float2 *>(row) + lane, make_float2(v[0], v[1]));
    } else {
#pragma unroll
        for (int q = 0; q < EPL / 4; ++q)
            __stcs(reinterpret_cast<float4 *>(row) + q * 32 + lane,
                   make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    }
}

// (also flags the packs that have an empty segment: k_pool_pipe zeroes them only there)
// One warp per 32 consecutive segments: the lanes read the 33 offsets, then walk the warp's
// positions j (consecutive lanes, consecutive j: coalesced ID reads and seg_of / key writes), each
// finding its segment by a 5-step search over the lanes' starts.  Offsets that decrease inside
// the warp (an invalid CSR: latched) fall back to one lane per segment.  ka (sort-based index):
// also the pack key of every position.
__global__ void __launch_bounds__(256) k_seg_of(const int32_t *offsets, int32_t B, int32_t F,
                                                const int32_t *field_gstart, const int32_t *id_start, int32_t *seg_of,
                                                const FieldInfo *finfo, int32_t *empty_pack, const int32_t *gtotal,
                                                int *err, SegKeyArgs ka) {
    const int64_t S = (int64_t)F * B;
    const int64_t sg0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * 32;
    if (sg0 >= S) return;
    const int lane = threadIdx.x & 31;
    const int64_t sg = sg0 + lane;
    const bool valid = sg < S;
    const int32_t f = valid ? (int32_t)(sg / B) : 0;
    const int32_t o0 = valid ? __ldg(offsets + sg) : INT32_MAX;
    const int32_t o1 = valid ? __ldg(offsets + sg + 1) : INT32_MAX;
    const int32_t gb = valid ? __ldg(field_gstart + f) - __ldg(id_start + f) : 0;
    // positions stay inside [0, total) whatever the offsets hold (total = 0 after an offsets
    // error: k_field_prep filled seg_of itself)
    const int64_t total = __ldg(gtotal);
    const bool bad = valid && o1 < o0;
    if (bad && err) atomicOr(err, ERR_OFFSETS);
    if (valid && o1 == o0 && empty_pack) empty_pack[finfo[f].pack] = 1;
    auto put = [&](int64_t j, int32_t s, int32_t ff, int32_t gbo) {
        const int64_t g = j + gbo;
        if (g < 0 || g >= total) return;
        seg_of[g] = s;
        if (ka.keys) {
            const FieldInfo fi = finfo[ff];
            const int64_t row = row_of(ka.id_mode, __ldg(ka.ids + j), fi, err);
            ka.keys[g] = (uint32_t)(__ldg(ka.pack_key_off + fi.pack) + fi.base + row);
        }
    };
    if (__any_sync(0xffffffffu, bad)) {  // not a CSR here: one lane per segment, ranges clamped
        if (valid) {
            const int64_t lo = max((int64_t)o0, -(int64_t)gb), hi = min((int64_t)o1, total - gb);
            for (int64_t j = lo; j < hi; ++j) put(j, (int32_t)sg, f, gb);
        }
        return;
    }
    const int nv = S - sg0 < 32 ? (int)(S - sg0) : 32;
    const int32_t J0 = __shfl_sync(0xffffffffu, o0, 0), J1 = __shfl_sync(0xffffffffu, o1, nv - 1);
    for (int64_t jb = J0; jb < J1; jb += 32) {
        const int64_t j = jb + lane;
        int o = 0;  // the last lane whose segment starts at or before j (non-empty when j < J1)
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const int32_t v = __shfl_sync(0xffffffffu, o0, o + step);
            if (v <= j) o += step;
        }
        const int32_t fo = __shfl_sync(0xffffffffu, f, o), gbo = __shfl_sync(0xffffffffu, gb, o);
        if (j < J1) put(j, (int32_t)(sg0 + o), fo, gbo);
    }
}

template <int D>
__global__ void __launch_bounds__(kNW * 32, 1) k_pool_pipe(PoolArgs a) {
    using G = PG<D>;
    constexpr int RS = G::RS, SB = G::SB, ROWB = G::ROWB, EPL = G::EPL;
    constexpr int CH = RS < kConsumeRows ? RS : kConsumeRows;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t P0 = __ldg(a.pack_gstart + a.pack), P1 = __ldg(a.pack_gstart + a.pack + 1);
    const int64_t nwarps = (int64_t)gridDim.x * kNW;
    const int64_t t = (int64_t)blockIdx.x * kNW + w;
    const int32_t tile = (int32_t)((P1 - P0 + nwarps - 1) / nwarps);
    // segment (pack order) of packed position p
    auto pseg = [&](int32_t p) {
        const int32_t sg = __ldg(a.seg_of + p);
        const int32_t f = sg / a.B;
        return __ldg(a.field_k + f) * a.B + (sg - f * a.B);
    };
    // first segment start at or after p (warp-uniform: 32 positions checked per round)
    auto seg_start_from = [&](int32_t p) {
        if (p <= P0 || p >= P1) return p;
        const int32_t s = pseg(p - 1);
        for (;; p += 32) {
            const int32_t q = p + lane;
            const unsigned m = __ballot_sync(0xffffffffu, q >= P1 || pseg(q) != s);
            if (m) return p + __ffs(m) - 1;
        }
    };
    // tile [pa, pb): nominal bounds moved forward to segment starts
    const int64_t n = P1 - P0, na = t * tile, nb = (t + 1) * tile;
    const int32_t pa = seg_start_from(P0 + (int32_t)(na < n ? na : n));
    const int32_t pb = seg_start_from(P0 + (int32_t)(nb < n ? nb : n));
    const int32_t seg_before = pa > P0 && pa < P1 ? pseg(pa - 1) : -1;  // segment of position pa - 1
    auto tiles = [&]() {  // this warp's tile (empty segments: the zero pass below)
    int64_t *s_out = reinterpret_cast<int64_t *>(smem) + (size_t)w * kS * RS;
    int32_t *s_seg = reinterpret_cast<int32_t *>(smem + (size_t)kNW * kS * RS * 8) + (size_t)w * kS * RS;
    unsigned char *wr = smem + G::RING_OFF + (size_t)w * kS * SB;
    const int32_t nst = (pb - pa + RS - 1) / RS;

    // lane l holds position base + l of a 32-position round: row offset (floats), pack segment,
    // output offset
    int64_t row_c, row_n, out_c, out_n;
    int32_t seg_c, seg_n;
    auto resolve = [&](int32_t base, int64_t &row, int32_t &seg, int64_t &out) {
        const int32_t p = base + lane;
        row = 0;
        seg = -1;
        out = 0;
        if (p < pb) {
            const int32_t sg = __ldg(a.seg_of + p);
            const int32_t f = sg / a.B, b = sg - f * a.B;
            const FieldInfo &fi = a.finfo[f];
            seg = __ldg(a.field_k + f) * a.B + b;
            out = (int64_t)b * a.out_stride + fi.col;
            if (a.row_off) {
                row = a.row_off[__ldg(a.inverse + p)];
            } else {
                const int32_t j = p - (__ldg(a.field_gstart + f) - __ldg(a.id_start + f));
                row = (fi.base + row_of(a.id_mode, __ldg(a.ids + j), fi, a.err)) * D;
            }
        }
    };
    resolve(pa, row_c, seg_c, out_c);
    resolve(pa + 32, row_n, seg_n, out_n);
    int32_t round_c = 0;
    auto issue = [&](int32_t k) {
        const int slot = k % kS;
        const int32_t r = (k * RS) >> 5;
        if (r != round_c) {
            row_c = row_n;
            seg_c = seg_n;
            out_c = out_n;
            round_c = r;
            resolve(pa + (r + 1) * 32, row_n, seg_n, out_n);
        }
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const int l0 = (k * RS) & 31;
        unsigned char *dst = wr + slot * SB;
        if constexpr (EPL == 2) {  // D = 64: two rows per instruction, a half-warp of 16-B copies each
            const int h = lane >> 4, c = lane & 15;
#pragma unroll
            for (int i = 0; i < RS; i += 2) {
                const int64_t row = __shfl_sync(0xffffffffu, row_c, l0 + i + h);
                if (i + h < nrows) ldgsts16(dst + (i + h) * ROWB + c * 16, a.weight + row + c * 4);
            }
        } else {
#pragma unroll
            for (int i = 0; i < RS; ++i) {
                const int64_t row = __shfl_sync(0xffffffffu, row_c, l0 + i);
                if (i < nrows) {
                    const float *src = a.weight + row;
#pragma unroll
                    for (int q = 0; q < EPL / 4; ++q) ldgsts16(dst + i * ROWB + q * 512 + lane * 16, src + q * 128 + lane * 4);
                }
            }
        }
        const int i = lane - l0;
        if (i >= 0 && i < nrows) {
            s_out[slot * RS + i] = out_c;
            s_seg[slot * RS + i] = seg_c;
        }
    };

    float acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
    int32_t cur = seg_before, ncur = 0;  // current segment (pack order) and its length so far
    int64_t cur_out = 0;
    auto flush = [&]() {
        if (a.pool_mean) {
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[e] = __fdiv_rn(acc[e], (float)ncur);
        }
        lane_store_cs<D>(a.out + cur_out, lane, acc);
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
    };

    for (int32_t k = 0; k < kS; ++k) {
        if (k < nst) issue(k);
        ldgsts_commit();
    }
#pragma unroll 1
    for (int32_t k = 0; k < nst; ++k) {
        const int slot = k % kS;
        ldgsts_wait<kS - 1>();
        __syncwarp();
        const int32_t p0 = pa + k * RS;
        const int nrows = pb - p0 < RS ? pb - p0 : RS;
        const float *rows = reinterpret_cast<const float *>(wr + slot * SB);
        // CH rows at a time (a fully unrolled stage with its inlined flushes overflows the
        // instruction cache at D = 64)
#pragma unroll 1
        for (int i0 = 0; i0 < nrows; i0 += CH) {
            float v[CH][EPL];
#pragma unroll
            for (int c = 0; c < CH; ++c)
                if (i0 + c < nrows) lane_load<D>(rows + (i0 + c) * D, lane, v[c]);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = i0 + c;
                if (i < nrows) {
                    const int32_t sg = s_seg[slot * RS + i];
                    if (sg != cur) {
                        if (ncur > 0) flush();
                        cur = sg;
                        cur_out = s_out[slot * RS + i];
                        ncur = 0;
                    }
                    ++ncur;
#pragma unroll
                    for (int e = 0; e < EPL; ++e) acc[e] = __fadd_rn(acc[e], v[c][e]);
                }
            }
        }
        __syncwarp();
        if (k + kS < nst) issue(k + kS);
        ldgsts_commit();
    }
    flush();
    };
    if (pa < pb) tiles();

    // empty segments (no position, so no tile writes them): zeros, only in packs k_seg_of
    // flagged (a sparse scan inside the ring would stall every warp on them)
    if (!a.empty_pack || a.empty_pack[a.pack]) {
        const int64_t S = (int64_t)a.Fp * a.B;
        for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
            const int32_t k = (int32_t)(s / a.B);
            const int32_t b = (int32_t)(s - (int64_t)k * a.B);
            const int32_t f = __ldg(a.pack_fields + k);
            const int64_t sg = (int64_t)f * a.B + b;
            if (__ldg(a.offsets + sg + 1) > __ldg(a.offsets + sg)) continue;
            float4 *o = reinterpret_cast<float4 *>(a.out + (int64_t)b * a.out_stride + a.finfo[f].col);
#pragma unroll
            for (int c = 0; c < D / 4; ++c) __stcs(o + c, make_float4(0.f, 0.f, 0.f, 0.f));
        }
    }
}

template <int D>
void launch_pipe(const PoolArgs &a, int num_sms, cudaStream_t s) {
    ensure_dyn_smem((const void *)k_pool_pipe<D>, PG<D>::SMEM);
    k_pool_pipe<D><<<(unsigned)num_sms, kNW * 32, PG<D>::SMEM, s>>>(a);
}

}  // namespace

bool pool_pipe_supported(int D, const PoolArgs &a) {
    const bool dim_ok = D == 64 || D == 128 || D == 256 || D == 384 || D == 512;
    return dim_ok && a.field_k && a.pack_gstart && ((uintptr_t)a.weight & 15) == 0 && ((uintptr_t)a.out & 15) == 0 &&
           (a.out_stride & 3) == 0;
}

void launch_seg_of(const int32_t *offsets, int32_t B, int32_t F, const int32_t *field_gstart, const int32_t *id_start,
                   int32_t *seg_of, cudaStream_t s, const FieldInfo *finfo, int32_t *empty_pack, const int32_t *gtotal,
                   int *err, const SegKeyArgs *ka) {
    const int64_t n = (int64_t)F * B;
    if (n > 0)
        k_seg_of<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(offsets, B, F, field_gstart, id_start, seg_of, finfo,
                                                            empty_pack, gtotal, err, ka ? *ka : SegKeyArgs{});
}

int launch_pool_pipe(int D, const PoolArgs &a, int num_sms, cudaStream_t s) {
    if ((int64_t)a.Fp * a.B == 0) return 0;
    switch (D) {
        case 64: launch_pipe<64>(a, num_sms, s); break;
        case 128: launch_pipe<128>(a, num_sms, s); break;
        case 256: launch_pipe<256>(a, num_sms, s); break;
        case 384: launch_pipe<384>(a, num_sms, s); break;
        case 512: launch_pipe<512>(a, num_sms, s); break;
        default: return 0;
    }
    return 1;
}

}  // namespace picasso
