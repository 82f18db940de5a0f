// introspect.cu — test-facing getters of the multi-GPU intermediates (synchronising).
#include "ctx.h"

extern "C" picasso_status picasso_get_owner_unique(picasso_ctx *ctx, int32_t pack, int64_t *dst, int64_t cap,
                                                   int64_t *n) {
    if (!ctx || !n || pack < 0 || pack >= ctx->P || !ctx->bound || ctx->world < 2) return PICASSO_ERR_INVALID_ARG;
    if (ctx->mp.p2p) return PICASSO_ERR_STATE;  // the peer-memory owner keeps a direct table, no unique list
    if (cudaStreamSynchronize(ctx->last_stream) != cudaSuccess) return PICASSO_ERR_CUDA;
    std::vector<int32_t> us(ctx->P + 1);
    if (cudaMemcpy(us.data(), ctx->mp.opack_ustart, sizeof(int32_t) * (ctx->P + 1), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return PICASSO_ERR_CUDA;
    const int64_t U = us[pack + 1] - us[pack];
    *n = U;
    if (dst && cap > 0 && U > 0) {
        std::vector<unsigned long long> g(U);
        if (cudaMemcpy(g.data(), ctx->mp.ouid_key + us[pack], sizeof(unsigned long long) * U, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
            return PICASSO_ERR_CUDA;
        std::vector<int64_t> k(U);
        for (int64_t i = 0; i < U; ++i) k[i] = (int64_t)(g[i] - (unsigned long long)ctx->pack_key_off[pack]);
        if (cudaMemcpy(dst, k.data(), sizeof(int64_t) * std::min(U, cap), cudaMemcpyHostToDevice) != cudaSuccess)
            return PICASSO_ERR_CUDA;
    }
    return PICASSO_OK;
}

void p2p_host_counts(picasso_ctx *ctx);

extern "C" picasso_status picasso_get_send_counts(picasso_ctx *ctx, int64_t *host_counts) {
    if (ctx && ctx->mp.p2p) p2p_host_counts(ctx);
    if (!ctx || !host_counts || ctx->world < 2 || ctx->mp.sk.empty()) return PICASSO_ERR_INVALID_ARG;
    for (int r = 0; r < ctx->world; ++r) host_counts[r] = ctx->mp.sk[r];
    return PICASSO_OK;
}

// Requested local rows of bucket (owner, pack) in send-slot order (both exchanges use the
// stable layout: owner-major, pack, uid order inside a bucket).
extern "C" picasso_status picasso_get_send_list(picasso_ctx *ctx, int32_t owner, int32_t pack, int64_t *dst,
                                                int64_t cap, int64_t *n) {
    if (!ctx || !n || ctx->world < 2 || !ctx->bound || owner < 0 || owner >= ctx->world || pack < 0 || pack >= ctx->P)
        return PICASSO_ERR_INVALID_ARG;
    if (cudaStreamSynchronize(ctx->last_stream) != cudaSuccess) return PICASSO_ERR_CUDA;
    const int b = owner * ctx->P + pack;
    int64_t se[2];
    if (cudaMemcpy(se, ctx->mp.bstart + b, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
        return PICASSO_ERR_CUDA;
    *n = se[1] - se[0];
    if (dst && cap > 0 && *n > 0) {
        std::vector<int32_t> v(*n);
        if (cudaMemcpy(v.data(), ctx->mp.send_keys + se[0], sizeof(int32_t) * *n, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
            return PICASSO_ERR_CUDA;
        for (int64_t i = 0; i < std::min(*n, cap); ++i) dst[i] = v[i];
    }
    return PICASSO_OK;
}
