// k3_sort.cuh -- K3: gather one coarse bucket from every tile, place its keys into their
// rank buckets and sort inside each bucket (§2 l.86: "N numbers are put into their
// corresponding estimate ranking buckets ... only the numbers inside each bucket need to
// be sorted").
//
// A thread-block cluster of R CTAs (distributed shared memory) owns one coarse bucket c,
// whose elements K1 left contiguous in the bucket's region; CTA r owns the fine sub-range
// [r*kr, (r+1)*kr) of its rank buckets.  Phase A: CTA r streams the r-th 1/R of the region
// (coalesced) and routes every element to the CTA that owns its fine bucket: per warp and
// batch of 32*kU elements, per-owner counts are packed into one 64-bit word, warp-scanned
// and reserved with one local shared-memory atomic per owner in a fixed per-source segment
// of the owner's receive buffer; the element stores go straight into the owner's shared
// memory and the per-source counts are published to every owner.  Phase B (after a cluster barrier, all local):
// counting sort by fine bucket (the placement), per-bucket insertion sort by
// (key, index) (the fix-up), an adjacent-pair check (reading A14), and a coalesced store.
// Two CTAs fit on one SM, so one CTA's memory phase overlaps the other's sort phase.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mlsort {

constexpr int kK3Threads = 256;
constexpr int kK3Warps = kK3Threads / 32;
constexpr int kU = 4;            // 32-element rounds per reservation batch
constexpr int kCtrlBytes = 1024; // per-CTA control words: counters, scan scratch, big-bucket queue

struct K3Params {
    uint32_t capc;          // region capacity (elements) of every coarse bucket
    uint32_t num_coarse;    // C
    uint32_t owner_shift;   // owner = fine >> owner_shift
    uint32_t kr;            // fine buckets per owner CTA = 2^owner_shift
    uint32_t cap;           // receive capacity (elements) per CTA
    uint32_t pad;
};

template <typename KeyT, bool PERM>
struct K3Layout {
    using Bits = typename KeyTraits<KeyT>::Bits;
    // [ctrl 1 KiB][recv_key cap][sorted_key cap][hist kr][recv_idx cap][sorted_idx cap][recv_fine cap]
    // [sorted_fine cap]
    static __host__ __device__ size_t bytes(uint32_t cap, uint32_t kr) {
        return kCtrlBytes + (size_t)cap * sizeof(Bits) * 2 + (size_t)kr * 4 + (PERM ? (size_t)cap * 8 : 0) +
               (size_t)cap * 4 + 16;
    }
};

template <typename KeyT, bool PERM>
__device__ __forceinline__ bool precedes(typename KeyTraits<KeyT>::Bits ka, uint32_t ia,
                                         typename KeyTraits<KeyT>::Bits kb, uint32_t ib) {
    if (PERM) return ka < kb || (ka == kb && ia < ib);
    return ka < kb;
}

__device__ __forceinline__ unsigned long long shfl_up_u64(unsigned long long v, int o) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, o);
    const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), o);
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
    const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
    const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
    return ((unsigned long long)hi << 32) | lo;
}

#ifdef MLSORT_K3_TRACE
__device__ unsigned long long* g_k3_trace = nullptr;   // [blocks][16] globaltimer stamps
#define K3_STAMP(slot)                                                                           \
    do {                                                                                         \
        if (g_k3_trace && threadIdx.x == 0) {                                                    \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
            g_k3_trace[(size_t)blockIdx.x * 16 + (slot)] = t_;                                   \
        }                                                                                        \
    } while (0)
#else
#define K3_STAMP(slot) do {} while (0)
#endif

constexpr uint32_t kRankMax = 64;     // larger rank buckets are sorted block-wide
constexpr uint32_t kBigQ = 40;        // queued big buckets per CTA (fits the ctrl area)

// Block-wide in-place bitonic sort of key/idx[s, e) by (key, index) for any length: the
// all-ascending ("flip") formulation, with the virtual +inf padding beyond e never touched.
// All threads of the CTA must call it.
template <typename KeyT, bool PERM>
__device__ __forceinline__ void cmpx(typename KeyTraits<KeyT>::Bits* key, uint32_t* idx, uint32_t a, uint32_t b) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    const Bits ka = key[a], kb = key[b];
    const uint32_t ia = PERM ? idx[a] : 0u, ib = PERM ? idx[b] : 0u;
    const bool gt = PERM ? (ka > kb || (ka == kb && ia > ib)) : (ka > kb);
    if (gt) {
        key[a] = kb;
        key[b] = ka;
        if (PERM) {
            idx[a] = ib;
            idx[b] = ia;
        }
    }
}

template <typename KeyT, bool PERM, int NT>
__device__ void block_bitonic_sort_nt(typename KeyTraits<KeyT>::Bits* key, uint32_t* idx, uint32_t s, uint32_t e) {
    const uint32_t n = e - s;
    uint32_t L = 1;
    while (L < n) L <<= 1;
    key += s;
    if (PERM) idx += s;
    for (uint32_t k = 2; k <= L; k <<= 1) {
        const uint32_t h = k >> 1;
        for (uint32_t t = threadIdx.x; t < L / 2; t += NT) {      // flip step
            const uint32_t blk = t / h, i = t - blk * h;
            const uint32_t a = blk * k + i, b = blk * k + k - 1 - i;
            if (b < n) cmpx<KeyT, PERM>(key, idx, a, b);
        }
        __syncthreads();
        for (uint32_t j = h >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < L / 2; t += NT) {
                const uint32_t a = 2 * t - (t & (j - 1)), b = a + j;
                if (b < n) cmpx<KeyT, PERM>(key, idx, a, b);
            }
            __syncthreads();
        }
    }
}

template <typename KeyT, bool PERM>
__device__ __forceinline__ void block_bitonic_sort(typename KeyTraits<KeyT>::Bits* key, uint32_t* idx, uint32_t s,
                                                   uint32_t e) {
    block_bitonic_sort_nt<KeyT, PERM, kK3Threads>(key, idx, s, e);
}

}  // namespace mlsort
