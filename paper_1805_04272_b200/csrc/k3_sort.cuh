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

template <typename KeyT, bool PERM, int R>
__global__ void __launch_bounds__(kK3Threads, 3)
k3_cluster_sort(K3Params p, const KeyT* __restrict__ reg_keys, const uint16_t* __restrict__ reg_fine,
                const uint32_t* __restrict__ reg_idx, const unsigned long long* __restrict__ starts,
                KeyT* __restrict__ out_keys,
                uint32_t* __restrict__ out_perm, unsigned long long* __restrict__ range_start,
                DevStatus* __restrict__ st, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_mark,
                const unsigned long long* __restrict__ rbase) {
    static_assert(R <= 8, "owner counts are packed in 8-bit fields of one u64");
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    // ctrl words: [0..7] local per-owner counters, [16..48] scan scratch, [64 .. 64+R*R) counts
    // (source s -> owner o at 64 + s*R + o, written remotely by every source), [160..) big queue
    uint32_t* ctrl = reinterpret_cast<uint32_t*>(smem);
    uint32_t* scratch = ctrl + 16;
    uint32_t* counts = ctrl + 64;
    Bits* recv_key = reinterpret_cast<Bits*>(smem + kCtrlBytes);
    Bits* sorted_key = recv_key + p.cap;
    uint32_t* hist = reinterpret_cast<uint32_t*>(sorted_key + p.cap);
    uint32_t* recv_idx = hist + p.kr;
    uint32_t* sorted_idx = recv_idx + (PERM ? p.cap : 0);
    uint16_t* recv_fine = reinterpret_cast<uint16_t*>(sorted_idx + (PERM ? p.cap : 0));
    uint16_t* sorted_fine = recv_fine + p.cap;

    const int r = (int)cg::this_cluster().block_rank();
    const uint32_t c = blockIdx.x / R;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t seg = p.cap / R;                 // slots reserved for each source CTA

    K3_STAMP(0);
    const unsigned long long S0 = starts[c], S1 = starts[c + 1];
    const unsigned long long n_c = S1 - S0;
    if (n_c == 0) return;                                       // uniform across the cluster
    auto register_big = [&]() {
        if (atomicExch(&big_mark[c], 1u) == 0u) {
            const unsigned long long k = atomicAdd(&st->big_count, 1ull);
            big_list[k] = c;
            atomicAdd(&st->big_elems, n_c);
            atomicMax(&st->max_coarse, n_c);
        }
    };
    if (n_c > (unsigned long long)R * p.cap) {                  // overflow path (K4)
        if (r == 0 && tid == 0) register_big();
        return;
    }
    // start the cluster barrier phase that guarantees every CTA of the cluster runs before the
    // first distributed-shared-memory store; finish it after the local prologue
    __cluster_barrier_arrive_relaxed();
    if (tid < R) ctrl[tid] = 0;
    const size_t off_key = (size_t)((unsigned char*)recv_key - smem);
    const size_t off_fine = (size_t)((unsigned char*)recv_fine - smem);
    const size_t off_idx = (size_t)((unsigned char*)recv_idx - smem);

    // ---------------- phase A: stream this CTA's share of the region of c, route by owner
    const uint32_t e0 = (uint32_t)(((unsigned long long)r * n_c) / R);
    const uint32_t e1 = (uint32_t)(((unsigned long long)(r + 1) * n_c) / R);
    const size_t rb0 = region_base(rbase, c, p.capc);
    const uint32_t fmask = p.kr - 1u;
    __syncthreads();                                   // local counters zeroed
    __cluster_barrier_wait();
    K3_STAMP(1);
    for (uint32_t b0 = e0 + warp * 32 * kU; b0 < e1; b0 += kK3Warps * 32 * kU) {
        KeyT key[kU];
        uint32_t fine[kU], idx[kU], own[kU];
        unsigned long long mycnt = 0;              // 8-bit count per owner for this lane
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t i = b0 + u * 32 + lane;
            own[u] = 0xffu;
            if (i < e1) {
                key[u] = reg_keys[rb0 + i];
                fine[u] = reg_fine[rb0 + i];
                idx[u] = PERM ? reg_idx[rb0 + i] : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (b0 + u * 32 + lane < e1) {
                own[u] = fine[u] >> p.owner_shift;
                mycnt += 1ull << (8 * own[u]);
            }
        }
        unsigned long long incl = mycnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = shfl_up_u64(incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned long long tot = shfl_u64(incl, 31);
        unsigned long long run = incl - mycnt;       // exclusive prefix per owner
        uint32_t base = 0;
        if (lane < R) {
            const uint32_t t_o = (uint32_t)((tot >> (8 * lane)) & 0xffu);
            if (t_o) base = atomicAdd(&ctrl[lane], t_o);     // local counter, no remote atomics
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t o = own[u];
            const uint32_t bo = __shfl_sync(0xffffffffu, base, o & 31);
            if (o < (uint32_t)R) {
                const uint32_t slot = bo + (uint32_t)((run >> (8 * o)) & 0xffu);
                run += 1ull << (8 * o);
                if (slot < seg) {
                    const uint32_t at_ = (uint32_t)r * seg + slot;
                    unsigned char* rb = cg::this_cluster().map_shared_rank(smem, (int)o);
                    reinterpret_cast<Bits*>(rb + off_key)[at_] = KeyTraits<KeyT>::to_ord(key[u]);
                    reinterpret_cast<uint16_t*>(rb + off_fine)[at_] = (uint16_t)(fine[u] & fmask);
                    if (PERM) reinterpret_cast<uint32_t*>(rb + off_idx)[at_] = idx[u];
                }
            }
        }
    }
    K3_STAMP(2);
    __syncthreads();                                   // local per-owner counts are final
    if (tid < R * R) {                                 // publish them to every owner
        const int o2 = tid / R, o = tid % R;
        uint32_t* rc = cg::this_cluster().map_shared_rank(counts, o2);
        rc[r * R + o] = ctrl[o];
    }
    cg::this_cluster().sync();                         // all routed elements and counts visible
    K3_STAMP(3);

    uint32_t my_off = 0, cnt = 0;
    bool overflow = false;
    for (int s = 0; s < R; ++s) {
        for (int o = 0; o < R; ++o) {
            const uint32_t v = counts[s * R + o];
            overflow |= v > seg;
            if (o < r) my_off += v;
            if (o == r) cnt += v;
        }
    }
    K3_STAMP(4);
    if (overflow) {   // a skewed fine range overflowed a segment: whole bucket -> K4
        if (tid == 0) register_big();
        return;
    }
    if (r == 0 && tid == 0) atomicMax(&st->max_coarse, n_c);

    // ---------------- phase B: counting sort by fine bucket (placement)
    for (uint32_t f = tid; f < p.kr; f += kK3Threads) hist[f] = 0;
    uint32_t* bigq = ctrl + 160;           // [0] count, then (s, e) pairs of big rank buckets
    if (tid == 0) bigq[0] = 0;
    __syncthreads();
    for (int s = 0; s < R; ++s) {
        const uint32_t fs = counts[s * R + r];
        for (uint32_t e = tid; e < fs; e += kK3Threads) atomicAdd(&hist[recv_fine[s * seg + e]], 1u);
    }
    __syncthreads();
    {
        const uint32_t per = (p.kr + kK3Threads - 1) / kK3Threads;
        const uint32_t f0 = min(p.kr, tid * per), f1 = min(p.kr, f0 + per);
        uint32_t local = 0;
        for (uint32_t f = f0; f < f1; ++f) local += hist[f];
        uint32_t total;
        uint32_t run = block_exclusive_scan<kK3Threads>(local, scratch, &total);
        for (uint32_t f = f0; f < f1; ++f) {
            const uint32_t h = hist[f];
            hist[f] = run;
            run += h;
        }
    }
    __syncthreads();
    for (int s = 0; s < R; ++s) {
        const uint32_t fs = counts[s * R + r];
        for (uint32_t e0 = tid; e0 < fs; e0 += kK3Threads) {
            const uint32_t e = s * seg + e0;
            const uint32_t f = recv_fine[e];
            const uint32_t pos = atomicAdd(&hist[f], 1u);
            sorted_key[pos] = recv_key[e];
            sorted_fine[pos] = (uint16_t)f;
            if (PERM) sorted_idx[pos] = recv_idx[e];
        }
    }
    __syncthreads();   // hist[f] = end of rank bucket f; the receive buffers are free now
    K3_STAMP(5);

    // ---------------- per-bucket fix-up: every element computes its rank inside its
    // rank bucket by counting the bucket's elements that precede it under (key, index)
    // (reading A9/A10); buckets larger than kRankMax (clamped tails collect in the end
    // buckets, heavy duplicates share one) are queued for a block-wide sort.
    Bits* final_key = recv_key;
    uint32_t* final_idx = recv_idx;
    for (uint32_t pos = tid; pos < cnt; pos += kK3Threads) {
        const uint32_t f = sorted_fine[pos];
        const uint32_t s = f ? hist[f - 1] : 0u, e = hist[f];
        const Bits kv = sorted_key[pos];
        const uint32_t iv = PERM ? sorted_idx[pos] : 0u;
        if (e - s > kRankMax) {
            if (pos == s) {
                const uint32_t q = atomicAdd(&bigq[0], 1u);
                if (q < kBigQ) {
                    bigq[1 + 2 * q] = s;
                    bigq[2 + 2 * q] = e;
                }
            }
            continue;
        }
        uint32_t rank = 0;
        for (uint32_t q = s; q < e; ++q) {
            const Bits kq = sorted_key[q];
            if (PERM) rank += (kq < kv || (kq == kv && sorted_idx[q] < iv)) ? 1u : 0u;
            else rank += (kq < kv || (kq == kv && q < pos)) ? 1u : 0u;
        }
        final_key[s + rank] = kv;
        if (PERM) final_idx[s + rank] = iv;
    }
    __syncthreads();
    K3_STAMP(6);
    {
        const uint32_t nbig = min(bigq[0], kBigQ);
        for (uint32_t q = 0; q < nbig; ++q) {
            const uint32_t s = bigq[1 + 2 * q], e = bigq[2 + 2 * q];
            block_bitonic_sort<KeyT, PERM>(sorted_key, sorted_idx, s, e);
            for (uint32_t i = s + tid; i < e; i += kK3Threads) {
                final_key[i] = sorted_key[i];
                if (PERM) final_idx[i] = sorted_idx[i];
            }
        }
        if (bigq[0] > kBigQ && tid == 0) atomicAdd(&st->k3_violations, 1ull);   // not expected; forces repair
    }
    __syncthreads();
    K3_STAMP(7);

    // ---------------- verify adjacent pairs inside this slice (reading A14), store
    const unsigned long long dst = S0 + my_off;
    if (tid == 0) range_start[(size_t)c * R + r] = cnt ? dst : ~0ull;
    uint32_t viol = 0;
    for (uint32_t e = tid; e < cnt; e += kK3Threads) {
        const Bits b = final_key[e];
        if (e > 0) {
            const Bits a = final_key[e - 1];
            const bool ok = PERM ? precedes<KeyT, true>(a, final_idx[e - 1], b, final_idx[e]) : (a <= b);
            viol += ok ? 0u : 1u;
        }
        out_keys[dst + e] = KeyTraits<KeyT>::from_ord(b);
        if (PERM) out_perm[dst + e] = final_idx[e];
    }
    viol = __reduce_add_sync(0xffffffffu, viol);
    if (lane == 0 && viol) atomicAdd(&st->k3_violations, (unsigned long long)viol);
    K3_STAMP(8);
}

}  // namespace mlsort
