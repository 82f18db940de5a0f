// dinterleave.cu — D-Interleaving (Eq. 2): a step's batch sliced into
// micro-batches that flow through the layer one after another, so the batch-proportional
// buffers (pooled output, dY, the per-ID index scratch, the per-unique G rows) are sized for a
// micro-batch instead of the whole batch (the paper's motivation: "large batch size is likely
// to cause an out-of-memory (OOM) issue", L398-403), with the result of the whole batch.
//
// Per micro-batch i the usual forward runs (its own Unique, pooling of its samples — the
// embedding of a sample depends only on its own IDs, so the concatenated outputs equal the
// whole batch's), then picasso_packed_lookup_bwd_accumulate: the usual segment-sum writes the
// micro-batch's G rows (one per unique key, rounded once from fp64), and
//   k_di_slot : per unique key, its row in the step accumulator — found, or inserted (open
//               addressing on the global pack key, arena offset from a bump counter); keys are
//               unique within a micro-batch and micro-batches are sequential, so no two threads
//               ever race on one key
//   k_di_add  : acc[slot] += G (fp64), one thread per 4-float chunk of the micro-batch's G
// and at the end picasso_dinterleave_apply:
//   k_di_apply: per accumulated row, G = fp32(acc) and the optimizer step (optim.cuh) — once per
//               step, on the pre-step weights every micro-batch's forward also read.
// The touched set is the union of the micro-batches' uniques = the whole batch's (reading O9).
// Rounding: a micro-batch's partial G is rounded to fp32 once, the partials are summed in fp64
// in micro-batch order and rounded again — reading O6' (the same as the W > 1 owner's sum over
// source ranks): exact under dyadic dY, within 1 ulp of the single rounding otherwise.
#include <cmath>
#include <cstring>

#include "ctx.h"
#include "optim.cuh"

namespace picasso {
namespace {

struct DiArgs {
    int32_t P;
    const int32_t *pack_ustart;            // [P+1] this micro-batch's uid ranges
    const unsigned long long *unique_gkey; // [U] global pack keys
    const int64_t *pack_key_off;           // [P+1]
    const int32_t *pack_dim;               // [P]
    const int64_t *pack_gbase;             // [P+1] float offset of each pack's G rows
    const float *gbuf;                     // the micro-batch's G rows (pack layout)
    Slot *table;                           // step accumulator index: key -> arena offset (uid field, in dbl4)
    uint32_t mask;
    double *acc;                           // arena
    int64_t acc_cap4;                      // arena capacity in dbl4 units
    int64_t *off;                          // [U] this micro-batch: arena offset (doubles) per uid, -1 overflow
    int32_t *list;                         // [max_step_unique] table slot of every accumulated row
    int64_t list_cap;
    unsigned long long *counters;          // [0] rows accumulated, [1] arena used (dbl4 units)
    int *err;
};

__device__ __forceinline__ int pack_of_key(const int64_t *pack_key_off, int P, unsigned long long k) {
    int lo = 0, hi = P;  // last p with pack_key_off[p] <= k
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((unsigned long long)__ldg(pack_key_off + mid) <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_di_slot(DiArgs a) {
    const int32_t U = __ldg(a.pack_ustart + a.P) - __ldg(a.pack_ustart);
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = a.unique_gkey[u];
        const int p = pack_of_key(a.pack_key_off, a.P, key);
        const int D = __ldg(a.pack_dim + p);
        uint32_t h = slot_hash(key) & a.mask;
        int64_t off = -1;
        for (uint32_t probe = 0; probe <= a.mask; ++probe) {
            Slot *s = a.table + h;
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(&s->key);
            if (cur == kEmptyKey) cur = atomicCAS(&s->key, kEmptyKey, key);
            if (cur == kEmptyKey) {  // new row of this step: arena space + list entry
                const unsigned long long o4 = atomicAdd(a.counters + 1, (unsigned long long)(D / 4));
                const unsigned long long li = atomicAdd(a.counters, 1ull);
                if ((int64_t)li < a.list_cap) a.list[li] = (int32_t)h;
                if ((int64_t)(o4 + D / 4) > a.acc_cap4 || (int64_t)li >= a.list_cap) {
                    s->uid = -1;  // no room: the row is dropped (CAPACITY latched below)
                    break;
                }
                s->uid = (int)o4;
                double *r = a.acc + (int64_t)o4 * 4;
                for (int d = 0; d < D; ++d) r[d] = 0.0;
                off = (int64_t)o4 * 4;
                break;
            }
            if (cur == key) {  // accumulated by an earlier micro-batch of this step
                off = s->uid < 0 ? -1 : (int64_t)s->uid * 4;
                break;
            }
            h = (h + 1) & a.mask;
        }
        if (off < 0) atomicOr(a.err, ERR_CAPACITY);  // arena, list or index full: the step is lost
        a.off[u] = off;
    }
}

__global__ void __launch_bounds__(256) k_di_add(DiArgs a) {
    const int64_t n4 = __ldg(a.pack_gbase + a.P) / 4;  // 4-float chunks of the micro-batch's G
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = e * 4;
        int lo = 0, hi = a.P;  // pack of G float f
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(a.pack_gbase + mid) <= f) lo = mid; else hi = mid;
        }
        const int D = __ldg(a.pack_dim + lo);
        const int64_t rel = f - __ldg(a.pack_gbase + lo);
        const int64_t u = __ldg(a.pack_ustart + lo) + rel / D;
        const int c = (int)(rel % D);
        const int64_t off = a.off[u];
        if (off < 0) continue;
        const float4 g = ldg_f4(a.gbuf + f);
        double2 *r = reinterpret_cast<double2 *>(a.acc + off + c);
        double2 x = r[0], y = r[1];
        x.x = __dadd_rn(x.x, (double)g.x);
        x.y = __dadd_rn(x.y, (double)g.y);
        y.x = __dadd_rn(y.x, (double)g.z);
        y.y = __dadd_rn(y.y, (double)g.w);
        r[0] = x;
        r[1] = y;
    }
}

struct DiApply {
    int32_t P;
    const Slot *table;
    const double *acc;
    const int32_t *list;
    const unsigned long long *counters;
    int64_t list_cap;
    const int64_t *pack_key_off;
    const int32_t *pack_dim;
    float *const *w;   // [P] device array of the packs' weight / state pointers
    float *const *s1;
    float *const *s2;
    OptParams o;
};

// one warp-group of D/4 threads per accumulated row (4 floats per thread), grid-stride
__global__ void __launch_bounds__(256) k_di_apply(DiApply a, int maxD) {
    const int64_t nrow = min((int64_t)a.counters[0], a.list_cap);
    const int V4 = maxD / 4;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nrow * V4; e += nth) {
        const int64_t i = e / V4;
        const int c = (int)(e % V4) * 4;
        const Slot s = a.table[a.list[i]];
        if (s.uid < 0) continue;
        const int p = pack_of_key(a.pack_key_off, a.P, s.key);
        const int D = __ldg(a.pack_dim + p);
        if (c >= D) continue;
        const int64_t row = (int64_t)(s.key - (unsigned long long)__ldg(a.pack_key_off + p));
        const double *r = a.acc + (int64_t)s.uid * 4 + c;
        const float4 g = make_float4(__double2float_rn(r[0]), __double2float_rn(r[1]), __double2float_rn(r[2]),
                                     __double2float_rn(r[3]));
        float *wp = a.w[p] + row * D + c, *s1p = a.s1[p] + row * D + c;
        float *s2p = a.o.opt == 1 ? a.s2[p] + row * D + c : nullptr;
        float4 w4 = *reinterpret_cast<float4 *>(wp), s14 = *reinterpret_cast<float4 *>(s1p);
        float4 s24 = s2p ? *reinterpret_cast<float4 *>(s2p) : make_float4(0.f, 0.f, 0.f, 0.f);
        opt_step4(a.o, g, w4, s14, s24);
        *reinterpret_cast<float4 *>(wp) = w4;
        *reinterpret_cast<float4 *>(s1p) = s14;
        if (s2p) *reinterpret_cast<float4 *>(s2p) = s24;
    }
}

__global__ void k_di_reset(Slot *table, uint64_t n, unsigned long long *counters) {
    const ulonglong2 e = make_ulonglong2(~0ull, ~0ull);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        reinterpret_cast<ulonglong2 *>(table)[i] = e;
    if (blockIdx.x == 0 && threadIdx.x < 2) counters[threadIdx.x] = 0;
}

}  // namespace
}  // namespace picasso

using namespace picasso;

#define DCK(x)                                                                  \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            ctx->last_msg = std::string(#x ": ") + cudaGetErrorString(e_);      \
            return PICASSO_ERR_CUDA;                                            \
        }                                                                       \
    } while (0)

namespace picasso {
int launch_segsum_any(picasso_ctx *ctx, int D, const UpdateArgs &u, cudaStream_t s);
UpdateArgs make_update_args(picasso_ctx *ctx, const float *grad_out, float lr, int64_t step, const int32_t *su,
                            const int32_t *sseg);
}

// Eq. 2: BS_micro = min over ops of RBound_op / RInstance_op, then the batch evenly divided into
// ceil(batch / BS_micro) micro-batches ("By default, we evenly divide data into micro batches to
// attain a load balancing", L409-410).
extern "C" picasso_status picasso_micro_batch_size(int32_t n_ops, const double *rbound, const double *rinstance,
                                                   int32_t batch, int32_t *bs_micro, int32_t *n_micro) {
    if (n_ops <= 0 || !rbound || !rinstance || batch < 0 || !bs_micro || !n_micro) return PICASSO_ERR_INVALID_ARG;
    double bs = INFINITY;
    for (int32_t i = 0; i < n_ops; ++i) {
        if (!(rbound[i] >= 0) || !(rinstance[i] >= 0)) return PICASSO_ERR_INVALID_ARG;
        if (rinstance[i] > 0) bs = std::min(bs, rbound[i] / rinstance[i]);
    }
    if (batch == 0) {
        *n_micro = 0;
        *bs_micro = 0;
        return PICASSO_OK;
    }
    const int64_t b = std::isinf(bs) ? batch : (int64_t)std::floor(bs);
    if (b < 1) return PICASSO_ERR_CAPACITY;  // not even one instance fits the bound
    const int64_t n = (batch + std::min<int64_t>(b, batch) - 1) / std::min<int64_t>(b, batch);
    *n_micro = (int32_t)n;
    *bs_micro = (int32_t)((batch + n - 1) / n);
    return PICASSO_OK;
}

extern "C" picasso_status picasso_dinterleave_begin(picasso_ctx *ctx, void *stream) {
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound || ctx->world != 1 || !ctx->di_table) return PICASSO_ERR_STATE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    k_di_reset<<<(unsigned)ctx->num_sms * 4, 256, 0, s>>>(ctx->di_table, ctx->di_cap, ctx->di_counters);
    DCK(cudaGetLastError());
    ctx->di_active = true;
    ctx->di_micro = 0;
    ctx->last_stream = s;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_packed_lookup_bwd_accumulate(picasso_ctx *ctx, const float *grad_out, void *stream) {
    if (!ctx) return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound || !ctx->fwd_done || !ctx->di_active) return PICASSO_ERR_STATE;
    if (!grad_out && ctx->B > 0) return PICASSO_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ctx->launches_bwd = 0;
    if (ctx->N > 0) {
        UpdateArgs u = make_update_args(ctx, grad_out, 0.f, 1, ctx->su, ctx->sseg);
        u.gbuf = ctx->gbuf;
        for (int32_t p = 0; p < ctx->P; ++p) {  // the micro-batch's G rows (pack layout)
            u.pack = p;
            u.long_cnt = ctx->long_cnt + p;
            u.pack_key_off = ctx->pack_key_off[p];
            u.weight = ctx->w[p];
            u.state1 = ctx->s1[p];
            u.state2 = ctx->s2[p];
            ctx->launches_bwd += launch_segsum_any(ctx, ctx->pack_dim[p], u, s);
        }
        DiArgs a{};
        a.P = ctx->P;
        a.pack_ustart = ctx->pack_ustart;
        a.unique_gkey = ctx->row_keys();  // the rows of the segment-sum's G (run order after a sorted index)
        a.pack_key_off = ctx->pack_key_off_d;
        a.pack_dim = ctx->pack_dim_d;
        a.pack_gbase = ctx->pack_gbase;
        a.gbuf = ctx->gbuf;
        a.table = ctx->di_table;
        a.mask = (uint32_t)(ctx->di_cap - 1);
        a.acc = ctx->di_acc;
        a.acc_cap4 = ctx->di_acc_cap4;
        a.off = ctx->di_off;
        a.list = ctx->di_list;
        a.list_cap = ctx->opts.max_step_unique;
        a.counters = ctx->di_counters;
        a.err = ctx->err;
        k_di_slot<<<(unsigned)ctx->num_sms * 4, 256, 0, s>>>(a);
        k_di_add<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(a);
        ctx->launches_bwd += 2;
    }
    DCK(cudaGetLastError());
    ++ctx->di_micro;
    ctx->fwd_done = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_dinterleave_apply(picasso_ctx *ctx, float lr, int64_t step, void *stream) {
    if (!ctx || step < 1) return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound || !ctx->di_active || ctx->fwd_done) return PICASSO_ERR_STATE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const UpdateArgs u = make_update_args(ctx, nullptr, lr, step, nullptr, nullptr);
    DiApply a{};
    a.P = ctx->P;
    a.table = ctx->di_table;
    a.acc = ctx->di_acc;
    a.list = ctx->di_list;
    a.counters = ctx->di_counters;
    a.list_cap = ctx->opts.max_step_unique;
    a.pack_key_off = ctx->pack_key_off_d;
    a.pack_dim = ctx->pack_dim_d;
    a.w = ctx->di_w;
    a.s1 = ctx->di_s1;
    a.s2 = ctx->di_s2;
    a.o = OptParams{u.opt, u.lr, u.eps, u.beta1, u.beta2, u.adam_ss};
    int maxD = 4;
    for (int32_t d : ctx->pack_dim) maxD = std::max(maxD, d);
    k_di_apply<<<(unsigned)ctx->num_sms * 8, 256, 0, s>>>(a, maxD);
    DCK(cudaGetLastError());
    ctx->launches_bwd = 1;
    ctx->di_active = false;
    ctx->last_stream = s;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_dinterleave_stats(picasso_ctx *ctx, int64_t *rows, int64_t *floats) {
    if (!ctx || !rows || !floats) return PICASSO_ERR_INVALID_ARG;
    if (!ctx->bound || !ctx->di_counters) return PICASSO_ERR_STATE;
    DCK(cudaStreamSynchronize(ctx->last_stream));
    unsigned long long c[2];
    DCK(cudaMemcpy(c, ctx->di_counters, sizeof(c), cudaMemcpyDeviceToHost));
    *rows = (int64_t)c[0];
    *floats = (int64_t)c[1] * 4;
    return PICASSO_OK;
}
