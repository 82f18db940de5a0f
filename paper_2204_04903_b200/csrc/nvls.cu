// nvls.cu — HybridHash hot-row gradient reduce + broadcast through NVLink SHARP (NVLS) multicast
// (PAPER.md L380-382 Shuffle&Stitch over the fabric, L459-522 HybridHash).
//
// Every rank's hot-row gradient buffer (hot_g: the rows of the replicated hot slots, and hot_touch:
// their occurrence counts) is bound into one multicast object, so the same offset has a unicast
// address (this rank's copy, written by the segment-sum) and a multicast address (all ranks'
// copies).  After the step's backward barrier, k_nvls_allreduce has every rank take 1/W of the
// float4 chunks: multimem.ld_reduce sums the chunk over all ranks inside the NVSwitch and
// multimem.st writes the sum back to every rank's copy — a one-shot reduce + broadcast with W x
// fewer bytes per rank than a ring, no NCCL launch, no host involvement.  One rank reduces each
// chunk and broadcasts it, so every replica receives bitwise the same sums (the replicas' updates
// stay identical, reading O17).  A barrier after the kernel orders the broadcasts before any
// rank's hot-row update reads them.
//
// Setup (host, once, collective over the ranks): rank 0 creates the multicast object and exports
// it as a POSIX file descriptor (picasso_nvls_create); the caller passes the descriptor to the other
// ranks' processes (SCM_RIGHTS over a Unix socket, embedding.py); every rank imports it and adds its
// device (picasso_nvls_open); after all ranks have opened, each binds its own device memory and
// maps the unicast and multicast views (picasso_nvls_bind).  Requires multicast-capable NVSwitch
// GPUs (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED); the caller falls back to the NCCL AllReduce when
// any call fails.
#include <cuda.h>

#include <cstring>
#include <type_traits>

#include "ctx.h"

namespace picasso {
namespace {

__device__ __forceinline__ float4 mm_ld_reduce_add(const float *mc) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(mc)
                 : "memory");
    return v;
}
__device__ __forceinline__ void mm_st(float *mc, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// chunks [0, n4_g) of hot_g and [t_off4, t_off4 + n4_t) of hot_touch; rank r takes the r-th 1/W
__global__ void __launch_bounds__(256) k_nvls_allreduce(float *mc, int64_t n4_g, int64_t t_off4, int64_t n4_t,
                                                        int rank, int W) {
    asm volatile("fence.proxy.alias;" ::: "memory");  // unicast writes (segment-sum) before multicast reads
    const int64_t total = n4_g + n4_t;
    const int64_t lo = total * rank / W, hi = total * (rank + 1) / W;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    // 4 reductions in flight per thread: the switch round trip is long
    for (int64_t i0 = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < hi; i0 += 4 * nth) {
        float4 v[4];
        int64_t c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = i0 + k * nth;
            c[k] = i < n4_g ? i : t_off4 + (i - n4_g);
            if (i < hi) v[k] = mm_ld_reduce_add(mc + 4 * c[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i0 + k * nth < hi) mm_st(mc + 4 * c[k], v[k]);
    }
    asm volatile("fence.proxy.alias;" ::: "memory");
}

}  // namespace
}  // namespace picasso

using namespace picasso;

// Driver-API entry points resolved through the runtime (cudaGetDriverEntryPoint): the library does
// not link libcuda, so it still loads where no driver is installed (the CPU build / test host).
namespace {
struct Drv {
    decltype(&cuGetErrorString) GetErrorString = nullptr;
    decltype(&cuMulticastGetGranularity) MulticastGetGranularity = nullptr;
    decltype(&cuMulticastCreate) MulticastCreate = nullptr;
    decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle = nullptr;
    decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle = nullptr;
    decltype(&cuMulticastAddDevice) MulticastAddDevice = nullptr;
    decltype(&cuMemGetAllocationGranularity) MemGetAllocationGranularity = nullptr;
    decltype(&cuMemCreate) MemCreate = nullptr;
    decltype(&cuMulticastBindMem) MulticastBindMem = nullptr;
    decltype(&cuMemAddressReserve) MemAddressReserve = nullptr;
    decltype(&cuMemMap) MemMap = nullptr;
    decltype(&cuMemSetAccess) MemSetAccess = nullptr;
    decltype(&cuMemUnmap) MemUnmap = nullptr;
    decltype(&cuMemAddressFree) MemAddressFree = nullptr;
    decltype(&cuMulticastUnbind) MulticastUnbind = nullptr;
    decltype(&cuMemRelease) MemRelease = nullptr;
    bool ok = false;
};
const Drv &drv() {
    static Drv d = [] {
        Drv x;
        bool ok = true;
        auto get = [&](const char *name, auto &fp) {
            void *p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) ok = false;
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(p);
        };
        get("cuGetErrorString", x.GetErrorString);
        get("cuMulticastGetGranularity", x.MulticastGetGranularity);
        get("cuMulticastCreate", x.MulticastCreate);
        get("cuMemExportToShareableHandle", x.MemExportToShareableHandle);
        get("cuMemImportFromShareableHandle", x.MemImportFromShareableHandle);
        get("cuMulticastAddDevice", x.MulticastAddDevice);
        get("cuMemGetAllocationGranularity", x.MemGetAllocationGranularity);
        get("cuMemCreate", x.MemCreate);
        get("cuMulticastBindMem", x.MulticastBindMem);
        get("cuMemAddressReserve", x.MemAddressReserve);
        get("cuMemMap", x.MemMap);
        get("cuMemSetAccess", x.MemSetAccess);
        get("cuMemUnmap", x.MemUnmap);
        get("cuMemAddressFree", x.MemAddressFree);
        get("cuMulticastUnbind", x.MulticastUnbind);
        get("cuMemRelease", x.MemRelease);
        cudaGetLastError();
        x.ok = ok;
        return x;
    }();
    return d;
}
}  // namespace

#define DRV(x)                                                                 \
    do {                                                                       \
        if (!drv().ok) {                                                       \
            ctx->last_msg = "CUDA driver entry points unavailable";            \
            return PICASSO_ERR_CUDA;                                           \
        }                                                                      \
        CUresult r_ = drv().x;                                                 \
        if (r_ != CUDA_SUCCESS) {                                              \
            const char *m_ = nullptr;                                          \
            drv().GetErrorString(r_, &m_);                                     \
            ctx->last_msg = std::string(#x ": ") + (m_ ? m_ : "?");            \
            return PICASSO_ERR_CUDA;                                           \
        }                                                                      \
    } while (0)

static picasso_status nvls_check(picasso_ctx *ctx) {
    if (!ctx || ctx->world < 2 || !ctx->bound || !ctx->mp.p2p || ctx->mp.p2p_loop || ctx->opts.cache_max_bytes <= 0)
        return PICASSO_ERR_INVALID_ARG;
    return PICASSO_OK;
}

static void nvls_sizes(picasso_ctx *ctx, size_t gran) {
    MultiState &mp = ctx->mp;
    const int64_t K = std::max<int64_t>(mp.k_max, 1);
    const int64_t arena = ctx->opts.cache_max_bytes / 4 + 4 * ctx->P;
    const size_t g_bytes = ((size_t)(arena / 2 + 4) * 4 + 255) / 256 * 256;  // hot_g, as the workspace carve
    mp.nvls_touch_off = g_bytes;
    const size_t raw = g_bytes + (size_t)2 * K * 4 + 256;
    mp.nvls_bytes = (raw + gran - 1) / gran * gran;
}

extern "C" picasso_status picasso_nvls_create(picasso_ctx *ctx, int32_t *fd_out) {
    picasso_status st = nvls_check(ctx);
    if (st) return st;
    if (!fd_out) return PICASSO_ERR_INVALID_ARG;
    *fd_out = -1;
    MultiState &mp = ctx->mp;
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)ctx->world;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = 1;
    // one size for the multicast object and every rank's bound allocation: a multiple of both the
    // multicast and the device-allocation granularity
    size_t gran = 0, agran = 0;
    DRV(MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM));
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PICASSO_ERR_CUDA;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    DRV(MemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    nvls_sizes(ctx, std::max(gran, agran));
    if (ctx->rank != 0) return PICASSO_OK;  // rank 0 creates; the others import its descriptor
    prop.size = mp.nvls_bytes;
    CUmemGenericAllocationHandle mc;
    DRV(MulticastCreate(&mc, &prop));
    mp.nvls_mc = (unsigned long long)mc;
    int fd = -1;
    DRV(MemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    *fd_out = fd;
    return PICASSO_OK;
}

extern "C" picasso_status picasso_nvls_open(picasso_ctx *ctx, int32_t fd) {
    picasso_status st = nvls_check(ctx);
    if (st) return st;
    MultiState &mp = ctx->mp;
    if (ctx->rank != 0) {
        if (fd < 0) return PICASSO_ERR_INVALID_ARG;
        CUmemGenericAllocationHandle mc;
        DRV(MemImportFromShareableHandle(&mc, reinterpret_cast<void *>((uintptr_t)fd),
                                         CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
        mp.nvls_mc = (unsigned long long)mc;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PICASSO_ERR_CUDA;
    DRV(MulticastAddDevice((CUmemGenericAllocationHandle)mp.nvls_mc, (CUdevice)dev));
    return PICASSO_OK;
}

extern "C" picasso_status picasso_nvls_bind(picasso_ctx *ctx) {
    picasso_status st = nvls_check(ctx);
    if (st) return st;
    MultiState &mp = ctx->mp;
    if (!mp.nvls_mc) return PICASSO_ERR_STATE;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PICASSO_ERR_CUDA;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as the multicast object
    CUmemGenericAllocationHandle uc;  // nvls_bytes: the multicast object's size (picasso_nvls_create)
    DRV(MemCreate(&uc, mp.nvls_bytes, &ap, 0));
    mp.nvls_uc = (unsigned long long)uc;
    {
        const CUresult r = drv().MulticastBindMem((CUmemGenericAllocationHandle)mp.nvls_mc, 0, uc, 0, mp.nvls_bytes, 0);
        if (r != CUDA_SUCCESS) {
            const char *m = nullptr;
            drv().GetErrorString(r, &m);
            ctx->last_msg = std::string("cuMulticastBindMem: ") + (m ? m : "?") + " (bytes " +
                            std::to_string(mp.nvls_bytes) + ")";
            return PICASSO_ERR_CUDA;
        }
    }
    CUdeviceptr uva = 0, mva = 0;
    DRV(MemAddressReserve(&uva, mp.nvls_bytes, 0, 0, 0));
    DRV(MemMap(uva, mp.nvls_bytes, 0, uc, 0));
    DRV(MemAddressReserve(&mva, mp.nvls_bytes, 0, 0, 0));
    DRV(MemMap(mva, mp.nvls_bytes, 0, (CUmemGenericAllocationHandle)mp.nvls_mc, 0));
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV(MemSetAccess(uva, mp.nvls_bytes, &acc, 1));
    DRV(MemSetAccess(mva, mp.nvls_bytes, &acc, 1));
    mp.nvls_uva = (unsigned long long)uva;
    mp.nvls_mva = (unsigned long long)mva;
    if (cudaMemset(reinterpret_cast<void *>(uva), 0, mp.nvls_bytes) != cudaSuccess) return PICASSO_ERR_CUDA;
    // the hot-row gradient rows and counts now live in the multicast-bound memory
    mp.hot_g = reinterpret_cast<float *>(uva);
    mp.hot_touch = reinterpret_cast<float *>(uva + mp.nvls_touch_off);
    mp.nvls = true;
    return PICASSO_OK;
}

// the step's hot-row reduce + broadcast (between the backward's barriers, p2p_host.cu)
picasso_status nvls_allreduce(picasso_ctx *ctx, cudaStream_t s) {
    MultiState &mp = ctx->mp;
    const int64_t n4_g = (mp.hot_g_floats + 3) / 4, n4_t = (mp.hot_k + 3) / 4;
    if (n4_g + n4_t == 0) return PICASSO_OK;
    k_nvls_allreduce<<<(unsigned)ctx->num_sms, 256, 0, s>>>(reinterpret_cast<float *>(mp.nvls_mva), n4_g,
                                                             (int64_t)(mp.nvls_touch_off / 16), n4_t, ctx->rank,
                                                             ctx->world);
    ctx->launches_bwd += 1;
    return cudaGetLastError() == cudaSuccess ? PICASSO_OK : PICASSO_ERR_CUDA;
}

void nvls_release(picasso_ctx *ctx) {
    MultiState &mp = ctx->mp;
    const Drv &d = drv();
    if (!d.ok) return;
    if (mp.nvls_mva) {
        d.MemUnmap((CUdeviceptr)mp.nvls_mva, mp.nvls_bytes);
        d.MemAddressFree((CUdeviceptr)mp.nvls_mva, mp.nvls_bytes);
    }
    if (mp.nvls_uva) {
        d.MemUnmap((CUdeviceptr)mp.nvls_uva, mp.nvls_bytes);
        d.MemAddressFree((CUdeviceptr)mp.nvls_uva, mp.nvls_bytes);
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (mp.nvls_mc && mp.nvls_uc) d.MulticastUnbind((CUmemGenericAllocationHandle)mp.nvls_mc, (CUdevice)dev, 0, mp.nvls_bytes);
    if (mp.nvls_uc) d.MemRelease((CUmemGenericAllocationHandle)mp.nvls_uc);
    if (mp.nvls_mc) d.MemRelease((CUmemGenericAllocationHandle)mp.nvls_mc);
    mp.nvls_mva = mp.nvls_uva = mp.nvls_uc = mp.nvls_mc = 0;
    mp.nvls = false;
}
