// k3_local.cuh -- K3 (v5): one CTA sorts one whole coarse bucket inside its shared memory
// (§2 l.86: "N numbers are put into their corresponding estimate ranking buckets
// ... only the numbers inside each bucket need to be sorted").
//
// K1 left coarse bucket c contiguous in its region (keys, rank-bucket ids, input indices).
// Persistent CTAs take coarse buckets from a ticket counter and, per bucket:
//   1. histogram of the rank buckets (shared-memory atomics on packed u16 counters)  -- A3
//   2. exclusive scan -> start of every rank bucket                                  -- A4
//   3. placement: every key goes to start[f]++ in shared memory (order-preserving
//      unsigned key bits; index alongside for perm sorts)                            -- A5
//   4. fix-up in place: rank buckets of 2-8 elements by register sorting networks, up to 24 by
//      insertion, larger ones by a block bitonic sort                                  -- A6
//   4p. key-only 32-bit keys at <= 1 key per rank bucket (C2): position-based fix-up instead --
//      two passes of 20-key window sorts over the placed array (k3l_posfix); the order check
//      of step 5 sends a coarse bucket it leaves unsorted through step 4               -- A6
//   5. the store is fused with an adjacent-order check of the whole coarse bucket; an
//      inversion (non-monotone model or float effects) re-sorts it in smem  -- A7 (A14)
// The primary pass runs two 512-thread CTAs per SM (two coarse buckets in flight hide each
// other's phase latencies) with a capacity of ~1.3x the average coarse bucket; larger buckets
// go to a secondary pass of one 1024-thread CTA per SM with the whole 227 KB, and only
// buckets beyond that to K4.  While a CTA works on a bucket it has already taken the next
// ticket and asked the L2 to prefetch that bucket's region (cp.async.bulk.prefetch).
// Placement order inside a rank bucket is arbitrary (atomics); the fix-up compares the input
// index as the tie-breaker, so the result is the unique stable order (reading A9).
#pragma once

#include "common.cuh"
#include <algorithm>

#include "k3_sort.cuh"
#include "k3_big.cuh"
#include "k3_posfix_net.cuh"

namespace mlsort {

// Optional per-phase cycle accounting for scripts/k3_bench.cu (-DMLSORT_K3L_TIMING): thread 0
// of every CTA accumulates clock64 deltas per phase into g_k3l_phase[blockIdx.x][8].
#ifdef MLSORT_K3L_TIMING
__device__ unsigned long long g_k3l_phase[1024][8];
#define K3L_T(i)                                                                 \
    do {                                                                         \
        if (threadIdx.x == 0) {                                                  \
            const long long t_ = clock64();                                      \
            k3l_acc[i] += t_ - k3l_prev;                                         \
            k3l_prev = t_;                                                       \
        }                                                                        \
    } while (0)
#else
#define K3L_T(i) do {} while (0)
#endif

constexpr int kL3Threads = 512;         // primary pass: two CTAs per SM
constexpr int kL3ThreadsBig = 1024;     // secondary pass (larger coarse buckets): one CTA per SM
constexpr uint32_t kL3RankMax = 24;     // rank buckets up to this size: insertion sort by one thread
constexpr uint32_t kL3BigQ = 48;        // queued larger rank buckets per coarse bucket
constexpr int kL3FineRegs = 5;
#ifndef MLSORT_K3_LATE_PF
#define MLSORT_K3_LATE_PF 0     // 1: prefetch the next bucket after the scan instead of at the ticket
#endif          // 128-bit vectors of fine ids kept in registers per thread

struct K3LParams {
    uint32_t capc;          // region capacity (elements) per coarse bucket
    uint32_t num_coarse;    // C
    uint32_t kfine;         // rank buckets per coarse bucket (2^fine_bits)
    uint32_t cap;           // largest coarse bucket this pass holds in shared memory
    uint32_t secondary;     // 0: pass over all coarse buckets; 1: pass over mid_list
    uint32_t to_mid;        // too-large buckets go to mid_list (1, primary of two passes) or to
                            // K4's big_list (0)
    uint32_t item_cap;      // ITEMS pass: capacity of the item list (k3_big.cuh)
    uint32_t fshift;        // coarse-bucket passes: rank bucket = fine id >> fshift (experiments)
    uint32_t premid;        // primary pass: K2 already listed the too-large buckets (skip them)
    uint32_t posfix;        // key-only 32-bit keys: position-based fix-up (step 4p) before the walk
    uint32_t tails_first;   // primary pass: ticket 0 = coarse bucket C-1 (both tail buckets start first)
};

// The rank-bucket histogram holds two u16 counters per 32-bit word (a coarse bucket never
// exceeds 65535 elements here); words rounded up to 4 so the key array after it is 16-B aligned.
__host__ __device__ inline uint32_t k3l_hist_words(uint32_t kfine) { return ((kfine + 1u) / 2u + 3u) & ~3u; }

constexpr uint32_t kL3WarpQ = 64;       // per-warp fix-up queue entries (power of two)
__host__ __device__ constexpr size_t k3l_queue_bytes(int nt) { return (size_t)(nt / 32) * 2 * kL3WarpQ * 4; }

// smem: ctrl | per-warp fix-up queues | hist (u16 pairs) | skey[cap] | sidx[cap] (perm)
inline size_t k3l_smem_bytes(size_t ks, bool perm, uint32_t kfine, uint32_t cap, int nt) {
    return kCtrlBytes + k3l_queue_bytes(nt) + (size_t)k3l_hist_words(kfine) * 4 + (size_t)cap * ks +
           (perm ? (size_t)cap * 4 : 0);
}

// largest cap with k3l_smem_bytes(...) <= budget
inline uint32_t k3l_cap_for(size_t budget, size_t ks, bool perm, uint32_t kfine, int nt) {
    const size_t fixed = kCtrlBytes + k3l_queue_bytes(nt) + (size_t)k3l_hist_words(kfine) * 4;
    if (budget <= fixed) return 0;
    const size_t leb = ks + (perm ? 4 : 0);
    uint64_t cap = std::min<uint64_t>((budget - fixed) / leb, 65535ull);
    while (cap > 0 && k3l_smem_bytes(ks, perm, kfine, (uint32_t)cap, nt) > budget) --cap;
    return (uint32_t)cap;
}

template <typename KeyT, bool PERM>
__device__ __forceinline__ void prefetch_bucket(const KeyT* reg_keys, const uint16_t* reg_fine, const uint32_t* reg_idx,
                                                size_t rb, unsigned long long n) {
    if (n == 0) return;
    prefetch_l2(reg_keys + rb, (uint32_t)(n * sizeof(KeyT)));
    prefetch_l2(reg_fine + rb, (uint32_t)(n * 2));
    if (PERM) prefetch_l2(reg_idx + rb, (uint32_t)(n * 4));
}

// counter f lives in half (f & 1) of word f >> 1
__device__ __forceinline__ void hist_inc(uint32_t* h2, uint32_t f) { atomicAdd(&h2[f >> 1], 1u << ((f & 1u) << 4)); }
__device__ __forceinline__ uint32_t hist_inc_ret(uint32_t* h2, uint32_t f) {
    const uint32_t sh = (f & 1u) << 4;
    return (atomicAdd(&h2[f >> 1], 1u << sh) >> sh) & 0xffffu;
}
__device__ __forceinline__ uint32_t hist_get(const uint32_t* h2, uint32_t f) {
    return (h2[f >> 1] >> ((f & 1u) << 4)) & 0xffffu;
}
__device__ __forceinline__ void hist_add8(uint32_t* h2, const uint4 v) {
    hist_inc(h2, v.x & 0xffffu);
    hist_inc(h2, v.x >> 16);
    hist_inc(h2, v.y & 0xffffu);
    hist_inc(h2, v.y >> 16);
    hist_inc(h2, v.z & 0xffffu);
    hist_inc(h2, v.z >> 16);
    hist_inc(h2, v.w & 0xffffu);
    hist_inc(h2, v.w >> 16);
}

// eight consecutive keys from a 16-B aligned address
template <typename KeyT> __device__ __forceinline__ void load8(const KeyT* p, KeyT (&k)[8]);
template <> __device__ __forceinline__ void load8<float>(const float* p, float (&k)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
}
template <> __device__ __forceinline__ void load8<double>(const double* p, double (&k)[8]) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double2 v = __ldg(q + i);
        k[2 * i] = v.x;
        k[2 * i + 1] = v.y;
    }
}


// compare-exchange of (key, index) records in registers: afterwards (ka, ia) precedes (kb, ib)
template <typename KeyT, bool PERM>
__device__ __forceinline__ void k3l_cx(typename KeyTraits<KeyT>::Bits& ka, uint32_t& ia,
                                       typename KeyTraits<KeyT>::Bits& kb, uint32_t& ib) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    if (!PERM) {
        const Bits lo = ka < kb ? ka : kb, hi = ka < kb ? kb : ka;
        ka = lo;
        kb = hi;
    } else {
        const bool sw = kb < ka || (kb == ka && ib < ia);
        const Bits tk = sw ? kb : ka;
        kb = sw ? ka : kb;
        ka = tk;
        const uint32_t ti = sw ? ib : ia;
        ib = sw ? ia : ib;
        ia = ti;
    }
}

// sort the 2..N records at [s, s + len) in place (N = 4 or 8): pad to N with the maximum
// record (it sorts last, so the first len outputs are the bucket), then Batcher's odd-even
// merge network (5 / 19 comparators) in registers
template <typename KeyT, bool PERM, int N>
__device__ __forceinline__ void k3l_sortn(typename KeyTraits<KeyT>::Bits* key, uint32_t* idx, uint32_t s,
                                          uint32_t len) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    Bits k[N];
    uint32_t i[N];
#pragma unroll
    for (uint32_t q = 0; q < N; ++q) {
        k[q] = q < len ? key[s + q] : ~(Bits)0;
        i[q] = PERM ? (q < len ? idx[s + q] : 0xffffffffu) : 0u;
    }
#define K3L_CX(a, b) k3l_cx<KeyT, PERM>(k[a], i[a], k[b], i[b])
    if (N == 4) {
        K3L_CX(0, 1); K3L_CX(2, 3);
        K3L_CX(0, 2); K3L_CX(1, 3);
        K3L_CX(1, 2);
    } else {
        K3L_CX(0, 1); K3L_CX(2, 3); K3L_CX(4, 5); K3L_CX(6, 7);
        K3L_CX(0, 2); K3L_CX(1, 3); K3L_CX(4, 6); K3L_CX(5, 7);
        K3L_CX(1, 2); K3L_CX(5, 6);
        K3L_CX(0, 4); K3L_CX(1, 5); K3L_CX(2, 6); K3L_CX(3, 7);
        K3L_CX(2, 4); K3L_CX(3, 5);
        K3L_CX(1, 2); K3L_CX(3, 4); K3L_CX(5, 6);
    }
#undef K3L_CX
#pragma unroll
    for (uint32_t q = 0; q < N; ++q) {
        if (q < len) {
            key[s + q] = k[q];
            if (PERM) idx[s + q] = i[q];
        }
    }
}

// stable insertion sort of [s, e) in shared memory by one thread (short runs: the cost is the
// run length plus its inversions; `top`, the largest record so far, stays in registers)
template <typename KeyT, bool PERM>
__device__ __forceinline__ void k3l_insertion(typename KeyTraits<KeyT>::Bits* key, uint32_t* idx, uint32_t s,
                                              uint32_t e) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    if (e <= s + 1) return;
    Bits top = key[s];
    uint32_t topi = PERM ? idx[s] : 0u;
    for (uint32_t i = s + 1; i < e; ++i) {
        const Bits k = key[i];
        const uint32_t x = PERM ? idx[i] : 0u;
        if (precedes<KeyT, PERM>(k, x, top, topi)) {
            uint32_t j = i;
            key[j] = top;
            if (PERM) idx[j] = topi;
            --j;
            while (j > s && precedes<KeyT, PERM>(k, x, key[j - 1], PERM ? idx[j - 1] : 0u)) {
                key[j] = key[j - 1];
                if (PERM) idx[j] = idx[j - 1];
                --j;
            }
            key[j] = k;
            if (PERM) idx[j] = x;
        } else {
            top = k;
            topi = x;
        }
    }
}

template <typename T> struct K3Out { using Bits = T; __device__ static T conv(T v) { return v; } };
template <> struct K3Out<float> {
    using Bits = uint32_t;
    __device__ static float conv(uint32_t v) { return KeyTraits<float>::from_ord(v); }
};
template <> struct K3Out<double> {
    using Bits = unsigned long long;
    __device__ static double conv(unsigned long long v) { return KeyTraits<double>::from_ord(v); }
};

// out[0, n) = conv(src[0, n)) with 16-byte stores (scalar head up to the first aligned slot)
template <typename T, int NT>
__device__ __forceinline__ void k3l_store(const typename K3Out<T>::Bits* src, uint32_t n, T* out) {
    constexpr uint32_t V = 16 / sizeof(T);
    const uint32_t head = min(n, (uint32_t)(((16u - ((uint32_t)reinterpret_cast<uintptr_t>(out) & 15u)) & 15u) / sizeof(T)));
    if (threadIdx.x < head) out[threadIdx.x] = K3Out<T>::conv(src[threadIdx.x]);
    const uint32_t nv = (n - head) / V;
    T* o = out + head;
    const typename K3Out<T>::Bits* sp = src + head;
    for (uint32_t v = threadIdx.x; v < nv; v += NT) {
        if (V == 4) {
            float4 q;
            uint32_t* qq = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
                const T t = K3Out<T>::conv(sp[4 * v + c]);
                qq[c] = *reinterpret_cast<const uint32_t*>(&t);
            }
            __stcs(reinterpret_cast<float4*>(o) + v, q);     // streaming: keep L2 for the regions
        } else {
            double2 q;
            unsigned long long* qq = reinterpret_cast<unsigned long long*>(&q);
#pragma unroll
            for (uint32_t c = 0; c < 2; ++c) {
                const T t = K3Out<T>::conv(sp[2 * v + c]);
                qq[c] = *reinterpret_cast<const unsigned long long*>(&t);
            }
            __stcs(reinterpret_cast<double2*>(o) + v, q);
        }
    }
    for (uint32_t i = head + nv * V + threadIdx.x; i < n; i += NT) out[i] = K3Out<T>::conv(src[i]);
}

// k3l_store of the keys fused with the order check of reading A14: every thread also compares
// each element it stores with its predecessor, (key, index) strictly increasing for perm sorts
// (indices are distinct), keys non-decreasing otherwise.  Returns this thread's "inversion seen".
template <typename KeyT, bool PERM, int NT>
__device__ __forceinline__ bool k3l_store_verify(const typename KeyTraits<KeyT>::Bits* src, const uint32_t* sidx,
                                                 uint32_t n, KeyT* out) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    constexpr uint32_t V = 16 / sizeof(KeyT);
    bool bad = false;
    auto chk = [&](uint32_t i, Bits cur) {
        if (i == 0) return;
        const Bits prev = src[i - 1];
        bad |= PERM ? !precedes<KeyT, true>(prev, sidx[i - 1], cur, sidx[i]) : cur < prev;
    };
    const uint32_t head = min(n, (uint32_t)(((16u - ((uint32_t)reinterpret_cast<uintptr_t>(out) & 15u)) & 15u) / sizeof(KeyT)));
    if (threadIdx.x < head) {
        const Bits c = src[threadIdx.x];
        chk(threadIdx.x, c);
        out[threadIdx.x] = K3Out<KeyT>::conv(c);
    }
    const uint32_t nv = (n - head) / V;
    KeyT* o = out + head;
    auto tail = [&](bool b) {                  // the elements behind the last whole vector
        bad = b;
        for (uint32_t i = head + nv * V + threadIdx.x; i < n; i += NT) {
            const Bits c = src[i];
            chk(i, c);
            out[i] = K3Out<KeyT>::conv(c);
        }
        return bad;
    };
    // key-only, src + head 16-B aligned (the kernel shifts the array by the output's
    // misalignment): one 128-bit shared load per vector, the predecessor from the lane below
    if (!PERM && ((uint32_t)reinterpret_cast<uintptr_t>(src + head) & 15u) == 0u) {
        const uint32_t lane = threadIdx.x & 31u;
        for (uint32_t vb = threadIdx.x - lane; vb < nv; vb += NT) {      // warp-uniform trip count
            const uint32_t v = vb + lane;
            const bool ok = v < nv;
            const uint32_t i0 = head + V * v;
            Bits c[V];
            if (ok) {
                if constexpr (V == 4) {
                    const uint4 t = *reinterpret_cast<const uint4*>(src + i0);
                    c[0] = (Bits)t.x; c[1] = (Bits)t.y; c[2] = (Bits)t.z; c[V - 1] = (Bits)t.w;
                } else {
                    const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(src + i0);
                    c[0] = (Bits)t.x; c[V - 1] = (Bits)t.y;
                }
            } else {
#pragma unroll
                for (uint32_t q = 0; q < V; ++q) c[q] = (Bits)0;
            }
            Bits prev = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
            if (lane == 0u && ok) prev = i0 ? src[i0 - 1] : c[0];
            if (!ok) continue;
#pragma unroll
            for (uint32_t q = 0; q < V; ++q) {
                bad |= c[q] < prev;
                prev = c[q];
            }
            if (V == 4) {
                float4 qv;
                uint32_t* qq = reinterpret_cast<uint32_t*>(&qv);
#pragma unroll
                for (uint32_t q = 0; q < V; ++q) {
                    const KeyT t = K3Out<KeyT>::conv(c[q]);
                    qq[q] = *reinterpret_cast<const uint32_t*>(&t);
                }
                __stcs(reinterpret_cast<float4*>(o) + v, qv);
            } else {
                double2 qv;
                unsigned long long* qq = reinterpret_cast<unsigned long long*>(&qv);
#pragma unroll
                for (uint32_t q = 0; q < V; ++q) {
                    const KeyT t = K3Out<KeyT>::conv(c[q]);
                    qq[q] = *reinterpret_cast<const unsigned long long*>(&t);
                }
                __stcs(reinterpret_cast<double2*>(o) + v, qv);
            }
        }
        return tail(bad);
    }
    for (uint32_t v = threadIdx.x; v < nv; v += NT) {
        const uint32_t i0 = head + V * v;
        Bits c[V];
#pragma unroll
        for (uint32_t q = 0; q < V; ++q) c[q] = src[i0 + q];
        Bits prev = i0 ? src[i0 - 1] : c[0];
        uint32_t pi = (PERM && i0) ? sidx[i0 - 1] : 0u;
#pragma unroll
        for (uint32_t q = 0; q < V; ++q) {
            if (PERM) {
                const uint32_t ci = sidx[i0 + q];
                if (i0 + q) bad |= !(prev < c[q] || (prev == c[q] && pi < ci));
                pi = ci;
            } else {
                bad |= c[q] < prev;
            }
            prev = c[q];
        }
        if (V == 4) {
            float4 qv;
            uint32_t* qq = reinterpret_cast<uint32_t*>(&qv);
#pragma unroll
            for (uint32_t q = 0; q < V; ++q) {
                const KeyT t = K3Out<KeyT>::conv(c[q]);
                qq[q] = *reinterpret_cast<const uint32_t*>(&t);
            }
            __stcs(reinterpret_cast<float4*>(o) + v, qv);
        } else {
            double2 qv;
            unsigned long long* qq = reinterpret_cast<unsigned long long*>(&qv);
#pragma unroll
            for (uint32_t q = 0; q < V; ++q) {
                const KeyT t = K3Out<KeyT>::conv(c[q]);
                qq[q] = *reinterpret_cast<const unsigned long long*>(&t);
            }
            __stcs(reinterpret_cast<double2*>(o) + v, qv);
        }
    }
    return tail(bad);
}

// ---- 4p. position-based fix-up (key-only, 32-bit keys).  After the placement the coarse
// bucket is ordered by rank bucket, and for a monotone model the rank buckets are key ranges
// (Eq. 4), so sorting ANY window of consecutive positions only reorders keys inside their rank
// buckets.  Pass A sorts the windows [20w, 20w + 20) in registers (one window per thread,
// 103-comparator network); pass B merges the sorted upper 8 of window w with the sorted lower 12
// of window w + 1 (37 comparators).  A rank bucket of up to 9 keys lies inside an A window or
// inside a B window ([20w + 12, 20w + 32)), so it ends up sorted; at one key per rank bucket on
// average (B = N) a longer one is a 1e-7 event per bucket, and the always-on order check of
// the store sends such a coarse bucket (and the two that hold the clamped tails) through the
// rank-bucket walk.  No per-bucket bookkeeping: ~0.5 warp instructions per key instead of ~1.8.
// The 80-byte thread stride makes every 128-bit shared access conflict-free (16-byte unit
// (5l + v) mod 8 is distinct over the 8 lanes of a phase).  skey[n, 20 nw) holds 0xFFFFFFFF.
#define MLSORT_CX(a, b) { const uint32_t lo_ = min(k[a], k[b]); k[b] = max(k[a], k[b]); k[a] = lo_; }
template <int NT>
__device__ __forceinline__ void k3l_posfix(uint32_t* skey, uint32_t nw) {
    for (uint32_t w = threadIdx.x; w < nw; w += NT) {
        uint4* p4 = reinterpret_cast<uint4*>(skey + 20u * w);
        uint32_t k[20];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const uint4 q = p4[v];
            k[4 * v] = q.x; k[4 * v + 1] = q.y; k[4 * v + 2] = q.z; k[4 * v + 3] = q.w;
        }
        MLSORT_SORT20(MLSORT_CX)
#pragma unroll
        for (int v = 0; v < 5; ++v) p4[v] = make_uint4(k[4 * v], k[4 * v + 1], k[4 * v + 2], k[4 * v + 3]);
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w + 1u < nw; w += NT) {
        uint4* p4 = reinterpret_cast<uint4*>(skey + 20u * w + 12u);
        uint32_t k[20];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const uint4 q = p4[v];
            k[4 * v] = q.x; k[4 * v + 1] = q.y; k[4 * v + 2] = q.z; k[4 * v + 3] = q.w;
        }
        MLSORT_MERGE20(MLSORT_CX)
        constexpr int pm[20] = MLSORT_MERGE20_PERM;
#pragma unroll
        for (int v = 0; v < 5; ++v)
            p4[v] = make_uint4(k[pm[4 * v]], k[pm[4 * v + 1]], k[pm[4 * v + 2]], k[pm[4 * v + 3]]);
    }
    __syncthreads();
}

// ITEMS = true: the round pass over the items of k3_cut (k3_big.cuh): work item t sorts the rank
// buckets [f_lo, f_hi) of coarse bucket c -- it reads c's whole region and keeps only those --
// into the output range starting at `out`; everything else is the same code.
template <typename KeyT, bool PERM, int NT, bool ITEMS = false>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : 2)
k3_local_sort(K3LParams p, const KeyT* __restrict__ reg_keys, const uint16_t* __restrict__ reg_fine,
              const uint32_t* __restrict__ reg_idx, const unsigned long long* __restrict__ starts,
              KeyT* __restrict__ out_keys, uint32_t* __restrict__ out_perm,
              unsigned long long* __restrict__ range_start, DevStatus* __restrict__ st,
              uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_mark, uint32_t* __restrict__ mid_list,
              unsigned long long* __restrict__ ticket, const unsigned long long* __restrict__ rbase,
              const K3Item* __restrict__ item_list = nullptr) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    // ctrl words: [1] next ticket, [2] big-queue count, [8..72) scan scratch,
    // [80 .. 80+2*kL3BigQ) big-queue (start, end) pairs
    uint32_t* ctrl = reinterpret_cast<uint32_t*>(smem);
    uint32_t* scratch = ctrl + 8;
    uint32_t* bigq = ctrl + 80;
    uint32_t* wqueue = reinterpret_cast<uint32_t*>(smem + kCtrlBytes);
    uint32_t* h2 = reinterpret_cast<uint32_t*>(smem + kCtrlBytes + k3l_queue_bytes(NT));   // u16 counter pairs
    Bits* skey0 = reinterpret_cast<Bits*>(h2 + k3l_hist_words(p.kfine));      // 16-B aligned
    uint32_t* sidx = reinterpret_cast<uint32_t*>(skey0 + p.cap);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (st->region_overflow) return;       // K1 overflowed a region: incomplete regions, re-run follows
    // work items: coarse ids 0..C-1 (primary), mid_list[0..mid_count) (secondary) or the
    // k3_cut items (ITEMS)
    const uint32_t items = ITEMS ? (uint32_t)min(st->item_count, (unsigned long long)p.item_cap)
                                 : (p.secondary ? (uint32_t)st->mid_count : p.num_coarse);
    // primary pass: ticket 0 is the last coarse bucket, so both end buckets -- the clamped tails
    // sit in their outer rank buckets and cost a block-wide sort -- start first instead of one of
    // them being the kernel's tail
    auto coarse_of = [&](uint32_t t) {
        return ITEMS ? item_list[t].c : (p.secondary ? mid_list[t] : (p.tails_first ? (t == 0u ? p.num_coarse - 1u : t - 1u) : t));
    };
    if (tid == 0) {
        const uint32_t t0 = (uint32_t)atomicAdd(ticket, 1ull);
        ctrl[1] = t0;
        if (t0 < items) {
            const uint32_t c0 = coarse_of(t0);
            const unsigned long long s0 = starts[c0], n0 = starts[c0 + 1] - s0;
            if (ITEMS || n0 <= p.cap)
                prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, region_base(rbase, c0, p.capc), n0);
        }
    }
#ifdef MLSORT_K3L_TIMING
    long long k3l_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long k3l_prev = clock64();
#endif
    while (true) {
        __syncthreads();                       // smem of the previous bucket is free; ctrl[1] visible
        K3L_T(0);
        const uint32_t t = ctrl[1];
        if (t >= items) break;
        uint32_t c, n, nreg, f_lo = 0u, kf = ITEMS ? p.kfine : (p.kfine >> p.fshift);
        unsigned long long S0;
        if (ITEMS) {
            const K3Item it = item_list[t];
            c = it.c;
            S0 = it.out;
            n = it.cnt;                        // keys of this item
            f_lo = it.f_lo;
            kf = it.f_hi - it.f_lo;            // its rank buckets
            nreg = (uint32_t)(starts[c + 1] - starts[c]);   // keys in c's region (all read)
        } else {
            c = coarse_of(t);
            S0 = starts[c];
            n = (uint32_t)min(starts[c + 1] - S0, (unsigned long long)0xffffffffull);
            nreg = n;
        }
        const uint32_t hw = (kf + 1u) / 2u;            // histogram words
        const uint32_t hwp = k3l_hist_words(kf);       // padded to a multiple of 4
        __syncthreads();                       // everyone read ctrl[1]
        if (tid == 0) {                        // take the next bucket now and prefetch it into L2
            const uint32_t t1 = (uint32_t)atomicAdd(ticket, 1ull);
            ctrl[1] = t1;
            ctrl[2] = 0;
#if !MLSORT_K3_LATE_PF
            if (t1 < items) {
                const uint32_t c1 = coarse_of(t1);
                const unsigned long long s1 = starts[c1], n1 = starts[c1 + 1] - s1;
                if (ITEMS || n1 <= p.cap)
                    prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, region_base(rbase, c1, p.capc), n1);
            }
#endif
        }
        // the next bucket's region is asked into L2 after this bucket's scan (step 2), about
        // half a bucket ahead of its use: an earlier prefetch was partly evicted before use
        auto prefetch_next = [&]() {
            if (!MLSORT_K3_LATE_PF || tid != 0) return;
            const uint32_t t1 = ctrl[1];
            if (t1 < items) {
                const uint32_t c1 = coarse_of(t1);
                const unsigned long long s1 = starts[c1], n1 = starts[c1 + 1] - s1;
                if (n1 <= p.cap) prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, region_base(rbase, c1, p.capc), n1);
            }
        };
        if (n == 0) {
            prefetch_next();
            if (!ITEMS && tid == 0) range_start[c] = ~0ull;
            continue;
        }
        if (n > p.cap) {                       // too large for this pass
            prefetch_next();
            if (ITEMS) {                       // (k3_cut never emits one)
                if (tid == 0) atomicAdd(&st->item_overflow, 1ull);
                continue;
            }
            if (tid == 0) {
                atomicMax(&st->max_coarse, (unsigned long long)n);
                if (p.premid) {
                    // (K2 listed it for the concurrent secondary pass)
                } else if (p.to_mid) {
                    mid_list[atomicAdd(&st->mid_count, 1ull)] = c;
                } else if (atomicExch(&big_mark[c], 1u) == 0u) {
                    const unsigned long long k = atomicAdd(&st->big_count, 1ull);
                    big_list[k] = c;
                    atomicAdd(&st->big_elems, (unsigned long long)n);
                }
            }
            continue;
        }
        if (!ITEMS && tid == 0) {
            range_start[c] = S0;
            atomicMax(&st->max_coarse, (unsigned long long)n);
        }
        const size_t rb = region_base(rbase, c, p.capc);
        const KeyT* gk = reg_keys + rb;
        const uint16_t* gf = reg_fine + rb;
        const uint32_t* gi = PERM ? reg_idx + rb : nullptr;
        const uint32_t n8 = nreg >> 3;
        const uint4* g8 = reinterpret_cast<const uint4*>(gf);
        // rank bucket of a region element inside this work item (ITEMS: f - f_lo, else f);
        // >= kf means "not in this item" (unsigned compare)
        auto rel = [&](uint32_t f) { return ITEMS ? f - f_lo : (f >> p.fshift); };
        auto hinc8 = [&](const uint4 v) {
            if (!ITEMS && p.fshift == 0) {
                hist_add8(h2, v);
            } else {
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t f = rel((w4[k >> 1] >> (16 * (k & 1))) & 0xffffu);
                    if (f < kf) hist_inc(h2, f);
                }
            }
        };

        // ---- 1. histogram of rank buckets (8 ids per 128-bit load; rows are 16-B aligned)
        for (uint32_t w = tid; w < hwp; w += NT) h2[w] = 0u;
        __syncthreads();
        // the first kL3FineRegs 128-bit vectors of fine ids per thread stay in registers for the
        // placement (a second read of them from L2 missed to DRAM: ncu v7 read 1.34x the bytes)
        uint4 fr[kL3FineRegs];
#pragma unroll
        for (int k = 0; k < kL3FineRegs; ++k) {
            const uint32_t i = tid + k * NT;
            fr[k] = i < n8 ? __ldg(g8 + i) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int k = 0; k < kL3FineRegs; ++k)
            if (tid + k * NT < n8) hinc8(fr[k]);
        for (uint32_t i = tid + kL3FineRegs * NT; i < n8; i += NT) hinc8(__ldg(g8 + i));
        for (uint32_t q = (n8 << 3) + tid; q < nreg; q += NT) {
            const uint32_t f = rel(gf[q]);
            if (!ITEMS || f < kf) hist_inc(h2, f);
        }
        __syncthreads();
        K3L_T(1);
        // ---- 2. exclusive scan of the counters: thread t scans its own WPT consecutive words
        // (128-bit loads, WPT a multiple of 4) in registers, then one block-wide scan of the
        // per-thread totals
        {
            // (an ODD number of 16-byte vectors per thread: the lane stride is then an odd multiple
            // of 16 B and the 128-bit accesses are bank-conflict-free; 4 vectors per thread were
            // 4-way conflicts, 12.6 M of the 56.7 M shared wavefronts of C2's K3)
            const uint32_t wpt = (((((hwp + NT - 1) / NT) + 3u) >> 2) | 1u) << 2;
            const uint32_t tw0 = min(hwp, (uint32_t)tid * wpt), tw1 = min(hwp, tw0 + wpt);
            uint4* h8 = reinterpret_cast<uint4*>(h2);
            uint32_t tot = 0;
            for (uint32_t w = tw0; w < tw1; w += 4) {
                const uint4 v = h8[w >> 2];
                tot += (v.x & 0xffffu) + (v.x >> 16) + (v.y & 0xffffu) + (v.y >> 16) + (v.z & 0xffffu) +
                       (v.z >> 16) + (v.w & 0xffffu) + (v.w >> 16);
            }
            uint32_t x = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t yy = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += yy;
            }
            if (lane == 31) scratch[warp] = x;
            __syncthreads();
            if (warp == 0) {
                constexpr int kW = NT / 32;
                const uint32_t tt = lane < kW ? scratch[lane] : 0u;
                uint32_t z = tt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t yy = __shfl_up_sync(0xffffffffu, z, o);
                    if (lane >= o) z += yy;
                }
                if (lane < kW) scratch[32 + lane] = z - tt;
            }
            __syncthreads();
            uint32_t run = scratch[32 + warp] + x - tot;
            auto ex2 = [&](uint32_t v) {               // two counters -> two exclusive starts
                const uint32_t lo = v & 0xffffu, r = run | ((run + lo) << 16);
                run += lo + (v >> 16);
                return r;
            };
            for (uint32_t w = tw0; w < tw1; w += 4) {
                uint4 v = h8[w >> 2];
                v.x = ex2(v.x);
                v.y = ex2(v.y);
                v.z = ex2(v.z);
                v.w = ex2(v.w);
                h8[w >> 2] = v;
            }
        }
        __syncthreads();
        prefetch_next();
        K3L_T(2);
        // The sorted keys start `off` elements into the 16-B aligned array, off = the output
        // range's misalignment, so the store reads shared memory and writes global memory with
        // 128-bit accesses at the same element (scalar 4-byte shared loads at a 16-byte lane
        // stride were 4-way bank conflicts: 10.5 M of the 56.7 M shared wavefronts of C2's K3).
        constexpr uint32_t kVec = 16u / (uint32_t)sizeof(KeyT);
        uint32_t off = (uint32_t)(reinterpret_cast<uintptr_t>(out_keys + S0) / sizeof(KeyT)) & (kVec - 1u);
        if (n + off > p.cap) off = 0u;
        Bits* skey = skey0 + off;
        // step 4p works on the physical array skey0[0, npos): `off` minimum pads in front, the
        // keys, maximum pads up to the last window's end; it applies when that fits
        const uint32_t npos = ((off + n + 19u) / 20u) * 20u;
        bool pos = false;
        if constexpr (!PERM && !ITEMS && sizeof(Bits) == 4) {
            pos = p.posfix && npos <= p.cap;
            if (pos) {
                if (tid < off) skey0[tid] = (Bits)0;
                for (uint32_t q = off + n + tid; q < npos; q += NT) skey0[q] = ~(Bits)0;
            }
        }
        // ---- 3. placement into rank-bucket order (ids + keys as 128-bit vectors)
        auto place8 = [&](uint32_t i, const uint4 fv) {
            KeyT kv[8];
            load8<KeyT>(gk + 8 * (size_t)i, kv);
            uint32_t iv[8];
            if (PERM) {
                const uint4 a = __ldg(reinterpret_cast<const uint4*>(gi) + 2 * i);
                const uint4 b = __ldg(reinterpret_cast<const uint4*>(gi) + 2 * i + 1);
                iv[0] = a.x; iv[1] = a.y; iv[2] = a.z; iv[3] = a.w;
                iv[4] = b.x; iv[5] = b.y; iv[6] = b.z; iv[7] = b.w;
            }
            const uint32_t fw[4] = {fv.x, fv.y, fv.z, fv.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t f = rel((fw[k >> 1] >> (16 * (k & 1))) & 0xffffu);
                if (ITEMS && f >= kf) continue;
                const uint32_t pos = hist_inc_ret(h2, f);
                skey[pos] = KeyTraits<KeyT>::to_ord(kv[k]);
                if (PERM) sidx[pos] = iv[k];
            }
        };
#pragma unroll
        for (int k = 0; k < kL3FineRegs; ++k)
            if (tid + k * NT < n8) place8(tid + k * NT, fr[k]);
        for (uint32_t i = tid + kL3FineRegs * NT; i < n8; i += NT) place8(i, __ldg(g8 + i));
        for (uint32_t q = (n8 << 3) + tid; q < nreg; q += NT) {
            const uint32_t f = rel(gf[q]);
            if (ITEMS && f >= kf) continue;
            const uint32_t pos = hist_inc_ret(h2, f);
            skey[pos] = KeyTraits<KeyT>::to_ord(gk[q]);
            if (PERM) sidx[pos] = gi[q];
        }
        __syncthreads();                       // counter f = end of rank bucket f
        K3L_T(3);
        // ---- 4. fix-up in place ("only the numbers inside each bucket need to be sorted").
        // Warp v walks 32 counter words (64 rank buckets) per batch.  Buckets of 0-1 elements
        // (~70 % of them) need nothing; those of 2-4 and of 5-8 are compacted into two per-warp
        // queues (ballot + prefix) and sorted 32 at a time, one per lane, by padded 4- and
        // 8-element networks in registers; up to kL3RankMax by insertion in their own lane, longer ones
        // (tails clamped into the end buckets, heavy duplicates) queued for a block-wide sort.
        auto walk = [&]() {
        {
            uint32_t* wq = wqueue + warp * 2 * kL3WarpQ;        // 2..4-element buckets
            uint32_t* wq8 = wq + kL3WarpQ;                      // 5..8-element buckets
            uint32_t qn = 0, qd = 0, qn8 = 0, qd8 = 0;          // warp-uniform: queued / sorted
            const uint32_t lt = (1u << lane) - 1u;
            for (uint32_t wb = (uint32_t)warp * 32u; wb < hw; wb += NT) {
                const uint32_t w = wb + lane;
                uint32_t sb[2] = {0u, 0u}, len[2] = {0u, 0u};
                if (w < hw) {
                    const uint32_t v = h2[w];
                    sb[0] = w ? (h2[w - 1] >> 16) : 0u;
                    sb[1] = v & 0xffffu;
                    len[0] = sb[1] - sb[0];
                    len[1] = (v >> 16) - sb[1];
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (len[h] > 8u) {                          // rare: by their own lane / block
                        if (len[h] <= kL3RankMax) {
                            k3l_insertion<KeyT, PERM>(skey, sidx, sb[h], sb[h] + len[h]);
                        } else {
                            const uint32_t q = atomicAdd(&ctrl[2], 1u);
                            if (q < kL3BigQ) {
                                bigq[2 * q] = sb[h];
                                bigq[2 * q + 1] = sb[h] + len[h];
                            }
                        }
                    }
                    const uint32_t ent = sb[h] | (len[h] << 16);
                    const bool need = len[h] - 2u <= 2u;
                    const uint32_t m = __ballot_sync(0xffffffffu, need);
                    if (need) wq[(qn + __popc(m & lt)) & (kL3WarpQ - 1u)] = ent;
                    qn += __popc(m);
                    const bool need8 = len[h] - 5u <= 3u;
                    const uint32_t m8 = __ballot_sync(0xffffffffu, need8);
                    if (m8) {
                        if (need8) wq8[(qn8 + __popc(m8 & lt)) & (kL3WarpQ - 1u)] = ent;
                        qn8 += __popc(m8);
                    }
                    __syncwarp();
                    if (qn - qd >= 32u) {
                        const uint32_t e = wq[(qd + lane) & (kL3WarpQ - 1u)];
                        k3l_sortn<KeyT, PERM, 4>(skey, sidx, e & 0xffffu, e >> 16);
                        qd += 32u;
                        __syncwarp();
                    }
                    if (qn8 - qd8 >= 32u) {
                        const uint32_t e = wq8[(qd8 + lane) & (kL3WarpQ - 1u)];
                        k3l_sortn<KeyT, PERM, 8>(skey, sidx, e & 0xffffu, e >> 16);
                        qd8 += 32u;
                        __syncwarp();
                    }
                }
            }
            if (lane < qn - qd) {
                const uint32_t e = wq[(qd + lane) & (kL3WarpQ - 1u)];
                k3l_sortn<KeyT, PERM, 4>(skey, sidx, e & 0xffffu, e >> 16);
            }
            if (lane < qn8 - qd8) {
                const uint32_t e = wq8[(qd8 + lane) & (kL3WarpQ - 1u)];
                k3l_sortn<KeyT, PERM, 8>(skey, sidx, e & 0xffffu, e >> 16);
            }
        }
        __syncthreads();
        // ---- 5. large rank buckets (tails collected in the end buckets, heavy duplicates):
        // block-wide bitonic sort in shared memory
        const uint32_t nbig = ctrl[2];
        if (nbig <= kL3BigQ)
            for (uint32_t q = 0; q < nbig; ++q) block_bitonic_sort_nt<KeyT, PERM, NT>(skey, sidx, bigq[2 * q], bigq[2 * q + 1]);
        if (nbig > kL3BigQ) block_bitonic_sort_nt<KeyT, PERM, NT>(skey, sidx, 0, n);
        };
        // ---- 5b./7. coalesced store of the sorted coarse bucket to its output range, fused with
        // the adjacent-order check of reading A14 over the WHOLE coarse bucket.  It runs for every
        // model and every fix-up: mode 0 = step 4p done (an inversion left: a rank bucket longer
        // than the windows guarantee -> the walk), mode 1 = the walk (an inversion left: a
        // non-monotone model, or an ulp-level non-monotone network output -> mode 2, a re-sort of
        // the whole coarse bucket in shared memory) -- never a wrong output.
        int mode = 1;
        if constexpr (!PERM && !ITEMS && sizeof(Bits) == 4) {
            if (pos) {
                k3l_posfix<NT>(reinterpret_cast<uint32_t*>(skey0), npos / 20u);
                mode = 0;
            }
        }
        K3L_T(4);
        for (;;) {
            if (mode == 1) {
                walk();
            } else if (mode == 2) {
                block_bitonic_sort_nt<KeyT, PERM, NT>(skey, sidx, 0, n);
                if (tid == 0) atomicAdd(&st->local_repairs, 1ull);
            }
            const bool bad = k3l_store_verify<KeyT, PERM, NT>(skey, sidx, n, out_keys + S0);
            if (!__syncthreads_or(bad) || mode == 2) break;
            if (mode == 0 && tid == 0) atomicAdd(&st->posfix_fallbacks, 1ull);
            ++mode;
        }
        K3L_T(5);
        if (PERM) k3l_store<uint32_t, NT>(sidx, n, out_perm + S0);
        K3L_T(6);
    }
#ifdef MLSORT_K3L_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 1024)
        for (int i = 0; i < 8; ++i) g_k3l_phase[blockIdx.x][i] = (unsigned long long)k3l_acc[i];
#endif
}

}  // namespace mlsort
