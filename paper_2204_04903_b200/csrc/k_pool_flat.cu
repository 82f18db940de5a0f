// k_pool_flat.cu — fused Gather + Stitch + SegmentReduction, one
// thread per 16-B chunk of an output row (segment s, chunk c), grid-stride.
//
//   out[b, col(f) + 4c .. 4c+3] = sum_{j in seg(f,b)} W[row(j)][4c .. 4c+3]   (ascending j from +0.0f;
//                                                                            mean: / len; empty: 0)
// The threads of one segment (D/4 of them: a warp at D = 128) read one 4·D-byte row per
// occurrence together — a coalesced request — and write the pooled row with streaming stores.
// No shared memory and few registers, so every SM keeps ~64 warps, i.e. as many independent
// row requests in flight as the access pattern can use (tools/gather_bench.cu: one 16-B
// load per thread is the fastest way to gather random rows on this GPU).  The row index is
// resolved by every thread of the segment (same address: one broadcast load; the hash is ALU).
#include "kernels.h"

namespace picasso {
namespace {

// D % 8 == 0: one thread per 32-B chunk, 256-bit loads / stores (LDG.E.ENL2.256): half the
// instructions per byte of the 16-B version
template <int D>
__global__ void __launch_bounds__(256) k_pool_flat8(PoolArgs a) {
    constexpr int V8 = D / 8;
    const int64_t n = (int64_t)a.Fp * a.B * V8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / V8;
        const int c = (int)(e - s * V8);
        const int32_t k = (int32_t)(s / a.B);
        const int32_t b = (int32_t)(s - (int64_t)k * a.B);
        const int32_t f = __ldg(a.pack_fields + k);
        const int64_t sg = (int64_t)f * a.B + b;
        const int32_t j0 = __ldg(a.offsets + sg), j1 = __ldg(a.offsets + sg + 1);
        const FieldInfo fi = a.finfo[f];
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int32_t gb = __ldg(a.field_gstart + f) - __ldg(a.id_start + f);
        const int64_t lo = max(max((int64_t)j0, (int64_t)0), -(int64_t)gb);
        const int64_t hi = min(min((int64_t)j1, a.n_ids), a.n_ids - gb);
#pragma unroll 4
        for (int64_t j = lo; j < hi; ++j) {
            const float *src = a.row_off ? a.weight + a.row_off[__ldg(a.inverse + j + gb)]
                                         : a.weight + (fi.base + row_of(a.id_mode, __ldg(a.ids + j), fi, a.err)) * D;
            const f8 v = ldg_f8(src + c * 8);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], v.v[q]);
        }
        f8 o;
#pragma unroll
        for (int q = 0; q < 8; ++q) o.v[q] = (a.pool_mean && j1 > j0) ? __fdiv_rn(acc[q], (float)(j1 - j0)) : acc[q];
        stcs_f8(a.out + (int64_t)b * a.out_stride + fi.col + c * 8, o);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_pool_flat(PoolArgs a) {
    constexpr int V4 = D / 4;
    const int64_t n = (int64_t)a.Fp * a.B * V4;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / V4;
        const int c = (int)(e - s * V4);
        const int32_t k = (int32_t)(s / a.B);
        const int32_t b = (int32_t)(s - (int64_t)k * a.B);
        const int32_t f = __ldg(a.pack_fields + k);
        const int64_t sg = (int64_t)f * a.B + b;
        const int32_t j0 = __ldg(a.offsets + sg), j1 = __ldg(a.offsets + sg + 1);
        const FieldInfo fi = a.finfo[f];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int32_t gb = __ldg(a.field_gstart + f) - __ldg(a.id_start + f);
        // IDs [lo, hi): the segment's range clamped so that j and its packed position j + gb stay
        // inside [0, n_ids) whatever the offsets hold (an offsets error latches in k_field_prep)
        const int64_t lo = max(max((int64_t)j0, (int64_t)0), -(int64_t)gb);
        const int64_t hi = min(min((int64_t)j1, a.n_ids), a.n_ids - gb);
        if (a.row_off) {  // W > 1: the rows received for the position's unique key
#pragma unroll 4
            for (int64_t j = lo; j < hi; ++j)
                acc = add4(acc, ldg_f4(a.weight + a.row_off[__ldg(a.inverse + j + gb)] + c * 4));
        } else {
#pragma unroll 4
            for (int64_t j = lo; j < hi; ++j) {
                const int64_t row = fi.base + row_of(a.id_mode, __ldg(a.ids + j), fi, a.err);
                acc = add4(acc, ldg_f4(a.weight + row * D + c * 4));
            }
        }
        if (a.pool_mean && j1 > j0) acc = div4(acc, (float)(j1 - j0));
        stcs_f4(a.out + (int64_t)b * a.out_stride + fi.col + c * 4, acc);
    }
}

}  // namespace

// One thread per segment: reads its two offsets (coalesced), writes a zero row only if the segment is
// empty — a cheap pass when there are none (one-hot packs), and no per-segment walk when most are
// (sparse positional fields).
int launch_pool_flat(int D, const PoolArgs &a, int num_sms, cudaStream_t s) {
    if ((int64_t)a.Fp * a.B == 0) return 0;
    const unsigned blocks = (unsigned)num_sms * 8;
    switch (D) {
        case 4: k_pool_flat<4><<<blocks, 256, 0, s>>>(a); break;
        case 8: a.vec8 ? k_pool_flat8<8><<<blocks, 256, 0, s>>>(a) : k_pool_flat<8><<<blocks, 256, 0, s>>>(a); break;
        case 16: a.vec8 ? k_pool_flat8<16><<<blocks, 256, 0, s>>>(a) : k_pool_flat<16><<<blocks, 256, 0, s>>>(a); break;
        case 32: k_pool_flat<32><<<blocks, 256, 0, s>>>(a); break;  // (32-B chunks measured slower here)
        case 64: k_pool_flat<64><<<blocks, 256, 0, s>>>(a); break;
        case 128: k_pool_flat<128><<<blocks, 256, 0, s>>>(a); break;
        case 256: k_pool_flat<256><<<blocks, 256, 0, s>>>(a); break;
        case 384: k_pool_flat<384><<<blocks, 256, 0, s>>>(a); break;
        case 512: k_pool_flat<512><<<blocks, 256, 0, s>>>(a); break;
        default: return 0;
    }
    return 1;
}

}  // namespace picasso
