// common.cuh — device-side helpers shared by the sm_100a kernels of the packed embedding path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace picasso {

// Per-field constants, uploaded once at bind time (one 48-byte record per field).
struct FieldInfo {
    int64_t base;     // table_base[t]: first pack key of the field's table
    int64_t rows;     // V_t
    uint64_t salt;    // HASH-mode salt of the table
    int64_t col;      // first output column of the field
    int32_t pack;     // pack of the field's table
    int32_t dim;      // D_t
    int32_t table;    // t
    int32_t pad;
};

// Hash-table slot of the fused Unique (one 16-byte record; memset 0xFF = empty).
struct Slot {
    unsigned long long key;  // global key (pack key + pack key offset); ~0 = empty
    unsigned int minpos;     // smallest packed-stream position holding the key
    int uid;                 // global unique index (first-occurrence order)
};

enum ErrBits : int { ERR_ID_RANGE = 1, ERR_CAPACITY = 2, ERR_OFFSETS = 8 };  // (4: ERR_PEER_TIMEOUT, p2p.h)

// fp64 accumulator of four columns (gradient sums, reading O6)
struct alignas(16) dbl4 {
    double x, y, z, w;
};

constexpr unsigned long long kEmptyKey = ~0ull;

// SplitMix64 output mix (reading O4 of DESIGN.md).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Raw categorical ID -> row of its table.  HASH: multiply-high range map of mix64(raw^salt).
__device__ __forceinline__ int64_t row_of(int mode, int64_t raw, const FieldInfo &fi, int *err) {
    if (mode == 1) return (int64_t)__umul64hi(mix64((uint64_t)raw ^ fi.salt), (uint64_t)fi.rows);
    if (raw < 0 || raw >= fi.rows) {
        atomicOr(err, ERR_ID_RANGE);
        return 0;
    }
    return raw;
}

// Slot index for a key (independent of the row mapping).
__device__ __forceinline__ uint32_t slot_hash(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDull;
    k ^= k >> 33;
    return (uint32_t)k;
}

// first index i in [lo, hi) with a[i] > v  (a non-decreasing)
template <typename T, typename V>
__device__ __forceinline__ int64_t upper_bound_dev(const T *a, int64_t lo, int64_t hi, V v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) <= (T)v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float4 ldg_f4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

// 32-byte (256-bit) global accesses, sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256 — half the load
// instructions of 16-byte accesses for the same bytes in flight
struct f8 {
    float v[8];
};
__device__ __forceinline__ f8 ldg_f8(const float *p) {  // read-only data (non-coherent path)
    f8 r;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ f8 ld_f8(const float *p) {  // data this kernel also writes
    f8 r;
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st_f8(float *p, const f8 &x) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(x.v[0]), "f"(x.v[1]), "f"(x.v[2]),
                 "f"(x.v[3]), "f"(x.v[4]), "f"(x.v[5]), "f"(x.v[6]), "f"(x.v[7])
                 : "memory");
}
__device__ __forceinline__ void stcs_f8(float *p, const f8 &x) {  // streaming (evict-first) store
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(x.v[0]), "f"(x.v[1]),
                 "f"(x.v[2]), "f"(x.v[3]), "f"(x.v[4]), "f"(x.v[5]), "f"(x.v[6]), "f"(x.v[7])
                 : "memory");
}

__device__ __forceinline__ void stcs_f4(float *p, float4 v) {
    __stcs(reinterpret_cast<float4 *>(p), v);
}

// IEEE round-to-nearest adds/divides that the compiler may not contract into FMA.
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float s) {
    return make_float4(__fdiv_rn(a.x, s), __fdiv_rn(a.y, s), __fdiv_rn(a.z, s), __fdiv_rn(a.w, s));
}

constexpr int kWarp = 32;

}  // namespace picasso
