// optim.cuh — the sparse optimizer step on one 4-float chunk of a row (reading O10):
// Adagrad (torch sparse form): acc += G^2; w -= lr * (G / (sqrt(acc) + eps))
// lazy Adam (torch SparseAdam form): m += (G - m)(1 - b1); v += (G^2 - v)(1 - b2);
//                                     w -= ss * (m / (sqrt(v) + eps)), ss = lr sqrt(1-b2^t)/(1-b1^t)
// Every operation rounds (no FMA contraction), in the order the oracle uses.  Used by the
// kernels that apply an update outside k_update.cu (D-Interleaving's accumulated step, the
// host-DRAM cold tier).
#pragma once
#include "common.cuh"

namespace picasso {

struct OptParams {
    int32_t opt;  // 0 Adagrad, 1 lazy Adam
    float lr, eps, beta1, beta2, adam_ss;
};

__device__ __forceinline__ void opt_step4(const OptParams &o, const float4 g4, float4 &w4, float4 &s14, float4 &s24) {
    const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
    float ww[4] = {w4.x, w4.y, w4.z, w4.w};
    float ss[4] = {s14.x, s14.y, s14.z, s14.w};
    float v2[4] = {s24.x, s24.y, s24.z, s24.w};
    if (o.opt == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float acc = __fadd_rn(ss[e], __fmul_rn(gg[e], gg[e]));
            ss[e] = acc;
            ww[e] = __fsub_rn(ww[e], __fmul_rn(o.lr, __fdiv_rn(gg[e], __fadd_rn(__fsqrt_rn(acc), o.eps))));
        }
    } else {
        const float omb1 = __fsub_rn(1.0f, o.beta1), omb2 = __fsub_rn(1.0f, o.beta2);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float mo = ss[e], vo = v2[e];
            const float mn = __fadd_rn(__fmul_rn(__fsub_rn(gg[e], mo), omb1), mo);
            const float vn = __fadd_rn(__fmul_rn(__fsub_rn(__fmul_rn(gg[e], gg[e]), vo), omb2), vo);
            ss[e] = mn;
            v2[e] = vn;
            ww[e] = __fsub_rn(ww[e], __fmul_rn(o.adam_ss, __fdiv_rn(mn, __fadd_rn(__fsqrt_rn(vn), o.eps))));
        }
    }
    w4 = make_float4(ww[0], ww[1], ww[2], ww[3]);
    s14 = make_float4(ss[0], ss[1], ss[2], ss[3]);
    s24 = make_float4(v2[0], v2[1], v2[2], v2[3]);
}

}  // namespace picasso
