// gather_bench.cu — ceiling of the embedding hot path's access pattern on this GPU: gather
// random 4*D-byte rows of a large table by an index list and write them densely (the one-hot
// forward), versus a dense copy of the same bytes.  Not part of the library; a measurement
// tool for DESIGN.md's roofline discussion.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
//   ./gather_bench [rows_in_table] [n_gather] [D]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// one warp per row group: U rows in flight per warp, float4 per lane (D = 128)
template <int U>
__global__ void __launch_bounds__(256) k_gather_warp(const float4 *__restrict__ tab, const int64_t *__restrict__ idx,
                                                     float4 *__restrict__ out, int64_t n, int v4) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = w * U; r0 < n; r0 += nw * U) {
        float4 v[U];
        int64_t myidx = (r0 + lane < n && lane < U) ? idx[r0 + lane] : 0;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int64_t row = __shfl_sync(0xffffffffu, myidx, k);
            if (r0 + k < n) v[k] = __ldg(tab + row * v4 + lane);
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (r0 + k < n) __stcs(out + (r0 + k) * v4 + lane, v[k]);
    }
}

// one thread per 16 B: fully independent loads (max MLP, no shuffles)
__global__ void k_gather_thread(const float4 *__restrict__ tab, const int64_t *__restrict__ idx, float4 *__restrict__ out,
                                int64_t n, int v4) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = i; e < n * v4; e += stride) {
        const int64_t r = e / v4;
        const int c = (int)(e - r * v4);
        __stcs(out + e, __ldg(tab + __ldg(idx + r) * v4 + c));
    }
}

__global__ void k_copy(const float4 *__restrict__ a, float4 *__restrict__ b, int64_t n4) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = i; e < n4; e += stride) __stcs(b + e, __ldg(a + e));
}

int main(int argc, char **argv) {
    const int64_t rows = argc > 1 ? atoll(argv[1]) : 46875000;
    const int64_t n = argc > 2 ? atoll(argv[2]) : 425984;
    const int D = argc > 3 ? atoi(argv[3]) : 128;
    const int v4 = D / 4;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float4 *tab, *out, *flush;
    int64_t *idx;
    CK(cudaMalloc(&tab, rows * D * 4));
    CK(cudaMalloc(&out, n * D * 4));
    CK(cudaMalloc(&idx, n * 8));
    const size_t fl = 256ull << 20;
    CK(cudaMalloc(&flush, fl));
    CK(cudaMemset(tab, 0, rows * D * 4));
    std::vector<int64_t> h(n);
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < n; ++i) {  // uniform random rows (distinct with high probability)
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = (int64_t)(x % (uint64_t)rows);
    }
    CK(cudaMemcpy(idx, h.data(), n * 8, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 2.0 * n * D * 4 + n * 8.0;
    auto run = [&](const char *name, auto launch) {
        float best = 1e9, tot = 0;
        const int it = 20;
        for (int i = 0; i < it + 3; ++i) {
            CK(cudaMemsetAsync(flush, i, fl));
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 3) { tot += ms; best = ms < best ? ms : best; }
        }
        printf("%-28s mean %8.2f us  best %8.2f us  %7.0f GB/s (mean)\n", name, tot / it * 1e3, best * 1e3,
               bytes / (tot / it * 1e-3) / 1e9);
    };
    for (int occ : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, sizeof nm, "warp U=8 blocks=%dxSM", occ);
        run(nm, [&] { k_gather_warp<8><<<sms * occ, 256>>>(tab, idx, out, n, v4); });
        snprintf(nm, sizeof nm, "warp U=16 blocks=%dxSM", occ);
        run(nm, [&] { k_gather_warp<16><<<sms * occ, 256>>>(tab, idx, out, n, v4); });
        snprintf(nm, sizeof nm, "warp U=4 blocks=%dxSM", occ);
        run(nm, [&] { k_gather_warp<4><<<sms * occ, 256>>>(tab, idx, out, n, v4); });
    }
    run("thread-per-16B", [&] { k_gather_thread<<<sms * 16, 256>>>(tab, idx, out, n, v4); });
    run("dense copy (same bytes)", [&] { k_copy<<<sms * 16, 256>>>(tab, out, n * v4); });
    return 0;
}
