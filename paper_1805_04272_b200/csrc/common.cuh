// common.cuh -- device helpers shared by the libmlsort kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mlsort {

constexpr int kThreads = 512;            // threads per CTA for K1 / K3
constexpr int kWarps = kThreads / 32;

// Device-side status word written by the kernels and read once per sort.
struct DevStatus {
    unsigned long long bad_index;   // lowest non-finite key index (ULLONG_MAX = none)
    unsigned long long tail_lo;     // keys < input_lo
    unsigned long long tail_hi;     // keys > input_hi
    unsigned long long violations;  // adjacent order violations found by the verify pass
    unsigned long long big_count;   // coarse buckets routed to the overflow path
    unsigned long long big_elems;   // elements in those buckets
    unsigned long long max_coarse;  // largest coarse bucket
    unsigned long long overflow;    // big buckets that still need the K4 radix pass
    unsigned long long ticket;      // dynamic CTA ticket (K4 persistent loop)
    unsigned long long region_overflow;   // K1 pieces that did not fit their coarse region
    unsigned long long ticket3;     // dynamic coarse-bucket ticket (K3 local-sort persistent loop)
    unsigned long long local_repairs;   // coarse buckets re-sorted in K3 after an inversion
    unsigned long long mid_count;   // coarse buckets handed from the primary to the secondary K3 pass
    unsigned long long ticket3b;    // ticket of the secondary K3 pass
    unsigned long long k3_violations;   // order violations found inside K3 slices (cluster K3)
    unsigned long long item_count;  // K3 round items emitted by k3_cut
    unsigned long long seg_count;   // giant runs handed to the host-driven radix pass
    unsigned long long ticket3c;    // k3_cut ticket
    unsigned long long ticket3d;    // K3 round-pass ticket
    unsigned long long item_overflow;   // items / segments that did not fit their lists
    unsigned long long posfix_fallbacks;   // coarse buckets whose position-based fix-up (K3 step 4p) left an
                                            // inversion and went through the rank-bucket walk
    unsigned long long pad[2];
};

// A K3 round item: the rank buckets [f_lo, f_hi) of coarse bucket c, cnt keys, sorted into the
// output range [out, out + cnt).  A segment: an output range [out, out + len) that still needs
// the stable radix pass (flags bit0: all keys bit-identical).
struct K3Item {
    uint32_t c, f_lo, f_hi, cnt;
    unsigned long long out;
};
struct K3Seg {
    unsigned long long out, len;
    uint32_t flags, pad;
};

// ---- start of coarse bucket c's region: c * capc, or the exact padded layout of a retry
__device__ __forceinline__ size_t region_base(const unsigned long long* rbase, uint32_t c, uint32_t capc) {
    return rbase ? (size_t)rbase[c] : (size_t)c * capc;
}

// ---- IEEE-754 totalOrder as unsigned integers (reading A10): negative -> ~bits,
// non-negative -> bits | sign.  Equal order bits <=> bit-identical keys.
template <typename K> struct KeyTraits;
template <> struct KeyTraits<float> {
    using Bits = uint32_t;
    __device__ __forceinline__ static Bits to_ord(float x) {
        uint32_t u = __float_as_uint(x);
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    }
    __device__ __forceinline__ static float from_ord(Bits o) {
        return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
    }
    __device__ __forceinline__ static bool finite(float x) {
        return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
    }
};
template <> struct KeyTraits<double> {
    using Bits = unsigned long long;
    __device__ __forceinline__ static Bits to_ord(double x) {
        unsigned long long u = (unsigned long long)__double_as_longlong(x);
        return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    }
    __device__ __forceinline__ static double from_ord(Bits o) {
        return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
    }
    __device__ __forceinline__ static bool finite(double x) {
        return ((unsigned long long)__double_as_longlong(x) & 0x7ff0000000000000ull) !=
               0x7ff0000000000000ull;
    }
};

// ---- block-wide exclusive scan of one uint32 per thread (NT threads).
// `scratch` needs NT/32 + 1 words of shared memory.  Returns the exclusive prefix;
// *total receives the block sum.  Contains two __syncthreads().
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* scratch,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? scratch[lane] : 0u;
        uint32_t s = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NT / 32) scratch[lane] = s - w;
        if (lane == NT / 32 - 1) scratch[NT / 32] = s;
    }
    __syncthreads();
    uint32_t excl = scratch[warp] + x - v;
    *total = scratch[NT / 32];
    return excl;
}

template <int NT>
__device__ __forceinline__ uint32_t block_reduce_sum(uint32_t v, uint32_t* scratch) {
    uint32_t t;
    block_exclusive_scan<NT>(v, scratch, &t);
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// bulk L2 prefetch of [p, p + bytes) (cp.async.bulk.prefetch.L2; 16-B granularity)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    // bulk L2 prefetch: 16-B aligned address and size
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t a0 = a & ~(uintptr_t)15;
    uint32_t sz = (uint32_t)(((a + bytes + 15) & ~(uintptr_t)15) - a0);
    const char* q = reinterpret_cast<const char*>(a0);
    while (sz) {
        const uint32_t chunk = sz > 65536u ? 65536u : sz;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(chunk) : "memory");
        q += chunk;
        sz -= chunk;
    }
}

}  // namespace mlsort
