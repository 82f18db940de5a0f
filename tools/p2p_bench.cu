// p2p_bench.cu — NVLink ceiling for the exchange's access patterns (measurement tool, not part of
// the library): every GPU stores (or loads) rows of 4*D bytes into (from) its peers' memory,
// all GPUs at once (the all-to-all of the row-sharded step), with 16-B thread stores to
// contiguous or randomly placed row slots, versus cudaMemcpyPeerAsync of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/p2p_bench tools/p2p_bench.cu
//   ./tools/bin/p2p_bench [MB per peer] [D]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// every peer at once, as the exchange kernels do: thread e -> (peer k, row r, chunk c).
// push: my rows for peer k -> k's receive block for me, slot perm[r] (perm == nullptr: slot r)
__global__ void k_push(const float4 *__restrict__ src, float4 *const *dst, int npeer, const int32_t *perm, int64_t n,
                       int v4) {
    const int64_t per = n * v4, tot = per * npeer;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / per);
        const int64_t w = e - k * per, r = w / v4;
        const int c = (int)(w - r * v4);
        const int64_t d = perm ? perm[r] : r;
        __stcg(dst[k] + d * v4 + c, __ldg(src + e));
    }
}
// pull: rows perm[r] of peer k's block for me -> my receive block for k (loads over NVLink)
__global__ void k_pull(const float4 *const *src, float4 *__restrict__ dst, int npeer, const int32_t *perm, int64_t n,
                       int v4) {
    const int64_t per = n * v4, tot = per * npeer;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / per);
        const int64_t w = e - k * per, r = w / v4;
        const int c = (int)(w - r * v4);
        const int64_t sr = perm ? perm[r] : r;
        dst[e] = __ldcv(src[k] + sr * v4 + c);
    }
}

// push with 32-byte (256-bit) stores: half the store instructions / transactions of 16-B stores
__global__ void k_push8(const float *__restrict__ src, float *const *dst, int npeer, int64_t n, int d) {
    const int v8 = d / 8;
    const int64_t per = n * v8, tot = per * npeer;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / per);
        const int64_t w = e - k * per;
        const float *s = src + e * 8;
        float *o = dst[k] + w * 8;
        float v[8];
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "l"(s));
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                     "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                     : "memory");
    }
}
// push through the TMA unit: each block stages 8-KB tiles in shared memory (double buffered) and
// issues one cp.async.bulk shared -> peer global per tile
__global__ void __launch_bounds__(256) k_push_tma(const float4 *__restrict__ src, float4 *const *dst, int npeer,
                                                  int64_t n, int v4) {
    constexpr int TB = 8192, TV = TB / 16;
    __shared__ __align__(128) float4 buf[2][TV];
    const int64_t per = n * v4;  // float4 per peer
    const int64_t ntile = (per + TV - 1) / TV;
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntile * npeer; t += gridDim.x) {
        const int k = (int)(t / ntile);
        const int64_t t0 = (t - (int64_t)k * ntile) * TV;
        const int cnt = (int)(per - t0 < TV ? per - t0 : TV);
        if (threadIdx.x == 0)  // the buffer of two tiles ago has been read by the bulk copy
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) buf[b][i] = __ldg(src + (int64_t)k * per + t0 + i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[b][0]);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[k] + t0), "r"(sa),
                         "r"(cnt * 16)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        b ^= 1;
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
    const double mb = argc > 1 ? atof(argv[1]) : 20.0;
    const int D = argc > 2 ? atoi(argv[2]) : 128;
    const int v4 = D / 4;
    int G = 0;
    CK(cudaGetDeviceCount(&G));
    if (G < 2) { printf("needs >= 2 GPUs\n"); return 0; }
    const int64_t rows = (int64_t)(mb * 1e6 / (4.0 * D));
    const size_t bytes = (size_t)rows * D * 4;
    std::vector<float4 *> src(G), dst(G);
    std::vector<int32_t *> perm(G);
    std::vector<cudaStream_t> st(G);
    std::vector<int32_t> hp(rows);
    for (int64_t i = 0; i < rows; ++i) hp[i] = (int32_t)i;
    uint64_t x = 88172645463325252ull;
    for (int64_t i = rows - 1; i > 0; --i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        std::swap(hp[i], hp[x % (uint64_t)(i + 1)]);
    }
    int sms = 0;
    for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        if (g == 0) CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
        for (int q = 0; q < G; ++q)
            if (q != g) CK(cudaDeviceEnablePeerAccess(q, 0));
        CK(cudaMalloc(&src[g], bytes * G));   // one block of rows per destination peer
        CK(cudaMalloc(&dst[g], bytes * G));   // one receive block per source peer
        CK(cudaMalloc(&perm[g], rows * 4));
        CK(cudaMemcpy(perm[g], hp.data(), rows * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(src[g], 1, bytes * G));
        CK(cudaStreamCreate(&st[g]));
    }
    // per GPU: device arrays of the peers' receive blocks (push) and send blocks (pull)
    std::vector<float4 **> pdst(G), psrc(G);
    for (int g = 0; g < G; ++g) {
        std::vector<float4 *> hd, hs;
        for (int q = 0; q < G; ++q)
            if (q != g) {
                hd.push_back(dst[q] + (size_t)g * rows * v4);
                hs.push_back(src[q] + (size_t)g * rows * v4);
            }
        CK(cudaSetDevice(g));
        CK(cudaMalloc(&pdst[g], sizeof(float4 *) * hd.size()));
        CK(cudaMalloc(&psrc[g], sizeof(float4 *) * hs.size()));
        CK(cudaMemcpy(pdst[g], hd.data(), sizeof(float4 *) * hd.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(psrc[g], hs.data(), sizeof(float4 *) * hs.size(), cudaMemcpyHostToDevice));
    }
    auto run = [&](const char *name, int mode) {
        float best = 1e30f, tot = 0;
        const int it = 10;
        for (int rep = 0; rep < it + 2; ++rep) {
            for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
            std::vector<cudaEvent_t> e0(G), e1(G);
            for (int g = 0; g < G; ++g) {
                CK(cudaSetDevice(g));
                cudaEventCreate(&e0[g]);
                cudaEventCreate(&e1[g]);
                cudaEventRecord(e0[g], st[g]);
                if (mode == 0) k_push<<<sms * 8, 256, 0, st[g]>>>(src[g], pdst[g], G - 1, nullptr, rows, v4);
                if (mode == 1) k_push<<<sms * 8, 256, 0, st[g]>>>(src[g], pdst[g], G - 1, perm[g], rows, v4);
                if (mode == 3) k_pull<<<sms * 8, 256, 0, st[g]>>>(psrc[g], dst[g], G - 1, perm[g], rows, v4);
                if (mode == 4)
                    k_push8<<<sms * 8, 256, 0, st[g]>>>(reinterpret_cast<const float *>(src[g]),
                                                        reinterpret_cast<float *const *>(pdst[g]), G - 1, rows, D);
                if (mode == 5) k_push_tma<<<sms * 2, 256, 0, st[g]>>>(src[g], pdst[g], G - 1, rows, v4);
                if (mode == 6) k_push_tma<<<sms * 4, 256, 0, st[g]>>>(src[g], pdst[g], G - 1, rows, v4);
                if (mode == 2)
                    for (int q = 0; q < G; ++q)
                        if (q != g)
                            CK(cudaMemcpyPeerAsync(dst[q] + (size_t)g * rows * v4, q, src[g] + (size_t)q * rows * v4,
                                                   g, bytes, st[g]));
                cudaEventRecord(e1[g], st[g]);
            }
            float worst = 0;
            for (int g = 0; g < G; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventSynchronize(e1[g]));
                float ms;
                cudaEventElapsedTime(&ms, e0[g], e1[g]);
                worst = ms > worst ? ms : worst;
                cudaEventDestroy(e0[g]);
                cudaEventDestroy(e1[g]);
            }
            if (rep >= 2) { tot += worst; best = worst < best ? worst : best; }
        }
        const double out = (double)bytes * (G - 1);  // bytes each GPU sends (or receives)
        printf("%-34s G=%d  %.1f MB/GPU  mean %8.1f us  %7.0f GB/s per GPU per direction (best %7.0f)\n", name, G,
               out / 1e6, tot / it * 1e3, out / (tot / it * 1e-3) / 1e9, out / (best * 1e-3) / 1e9);
    };
    run("push, contiguous slots (16-B stores)", 0);
    run("push, random row slots (16-B stores)", 1);
    run("cudaMemcpyPeerAsync", 2);
    run("pull, random rows (16-B loads)", 3);
    run("push, contiguous (32-B stores)", 4);
    run("push, TMA bulk 8-KB tiles (2 CTA/SM)", 5);
    run("push, TMA bulk 8-KB tiles (4 CTA/SM)", 6);
    return 0;
}
