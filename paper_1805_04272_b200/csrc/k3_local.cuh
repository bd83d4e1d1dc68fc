// k3_local.cuh -- K3 (v2): one CTA sorts one whole coarse bucket inside its shared memory
// (§2 l.86: "N numbers are put into their corresponding estimate ranking buckets
// ... only the numbers inside each bucket need to be sorted").
//
// K1 left coarse bucket c contiguous in its region (keys, fine bucket ids, input indices).
// A persistent CTA takes coarse buckets from a ticket counter and, per bucket:
//   1. histogram of the fine rank buckets (shared-memory atomics)            -- A3
//   2. exclusive scan -> start of every rank bucket                           -- A4
//   3. placement: every key goes to start[f]++ in shared memory (order-preserving
//      unsigned key bits; index alongside for perm sorts)                     -- A5
//   4. fix-up: each rank bucket is sorted by (totalOrder key, input index) -- insertion sort
//      for small buckets, a block-wide bitonic sort for the rare large ones  -- A6
//   5. adjacent-pair verify over the whole coarse bucket, coalesced store    -- A7
// While it works on bucket c it has already taken the next ticket and asked the L2 to
// prefetch that bucket's region (cp.async.bulk.prefetch), so the next bucket's loads hit L2.
// Placement order inside a rank bucket is arbitrary (atomics); the fix-up compares the
// input index as the tie-breaker, so the result is the unique stable order (reading A9).
#pragma once

#include "common.cuh"
#include "k3_sort.cuh"

namespace mlsort {

constexpr int kL3Threads = 1024;
constexpr uint32_t kInsMax = 32;        // rank buckets up to this size: per-thread insertion sort
constexpr uint32_t kL3BigQ = 48;        // queued larger rank buckets per coarse bucket

struct K3LParams {
    uint32_t capc;          // region capacity (elements) per coarse bucket
    uint32_t num_coarse;    // C
    uint32_t kfine;         // rank buckets per coarse bucket (2^fine_bits)
    uint32_t cap;           // largest coarse bucket this kernel holds in shared memory
};

// histogram words rounded up to 4 so the key array after it is 16-B aligned
__host__ __device__ inline uint32_t k3l_hist_words(uint32_t kfine) { return (kfine + 3u) & ~3u; }

inline size_t k3l_smem_bytes(size_t ks, bool perm, uint32_t kfine, uint32_t cap) {
    return kCtrlBytes + (size_t)k3l_hist_words(kfine) * 4 + (size_t)cap * ks + (perm ? (size_t)cap * 4 : 0);
}

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

template <typename KeyT, bool PERM>
__device__ __forceinline__ void prefetch_bucket(const KeyT* reg_keys, const uint16_t* reg_fine, const uint32_t* reg_idx,
                                                size_t rb, unsigned long long n) {
    if (n == 0) return;
    prefetch_l2(reg_keys + rb, (uint32_t)(n * sizeof(KeyT)));
    prefetch_l2(reg_fine + rb, (uint32_t)(n * 2));
    if (PERM) prefetch_l2(reg_idx + rb, (uint32_t)(n * 4));
}

__device__ __forceinline__ void hist_add8(uint32_t* hist, const uint4 v) {
    atomicAdd(&hist[v.x & 0xffffu], 1u);
    atomicAdd(&hist[v.x >> 16], 1u);
    atomicAdd(&hist[v.y & 0xffffu], 1u);
    atomicAdd(&hist[v.y >> 16], 1u);
    atomicAdd(&hist[v.z & 0xffffu], 1u);
    atomicAdd(&hist[v.z >> 16], 1u);
    atomicAdd(&hist[v.w & 0xffffu], 1u);
    atomicAdd(&hist[v.w >> 16], 1u);
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

template <typename KeyT, bool PERM>
__global__ void __launch_bounds__(kL3Threads, 1)
k3_local_sort(K3LParams p, const KeyT* __restrict__ reg_keys, const uint16_t* __restrict__ reg_fine,
              const uint32_t* __restrict__ reg_idx, const unsigned long long* __restrict__ starts,
              KeyT* __restrict__ out_keys, uint32_t* __restrict__ out_perm,
              unsigned long long* __restrict__ range_start, DevStatus* __restrict__ st,
              uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_mark, unsigned long long* __restrict__ ticket) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    // ctrl words: [0] current ticket, [1] next ticket, [2] big-queue count, [8..40) scan
    // scratch, [64 .. 64+2*kL3BigQ) big-queue (s, e) pairs
    uint32_t* ctrl = reinterpret_cast<uint32_t*>(smem);
    uint32_t* scratch = ctrl + 8;
    uint32_t* bigq = ctrl + 64;
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + kCtrlBytes);
    Bits* skey = reinterpret_cast<Bits*>(hist + k3l_hist_words(p.kfine));
    uint32_t* sidx = reinterpret_cast<uint32_t*>(skey + p.cap);

    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t C = p.num_coarse;
    if (tid == 0) {
        const uint32_t t0 = (uint32_t)atomicAdd(ticket, 1ull);
        ctrl[1] = t0;
        if (t0 < C) {
            const unsigned long long s0 = starts[t0], n0 = starts[t0 + 1] - s0;
            if (n0 <= p.cap) prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, (size_t)t0 * p.capc, n0);
        }
    }
    unsigned long long viol_total = 0;
    while (true) {
        __syncthreads();                       // smem of the previous bucket is free; ctrl[1] visible
        const uint32_t c = ctrl[1];
        if (c >= C) break;
        const unsigned long long S0 = starts[c];
        const uint32_t n = (uint32_t)min(starts[c + 1] - S0, (unsigned long long)0xffffffffull);
        __syncthreads();                       // everyone read ctrl[1]
        if (tid == 0) {                        // take the next bucket now and prefetch it into L2
            const uint32_t t1 = (uint32_t)atomicAdd(ticket, 1ull);
            ctrl[1] = t1;
            ctrl[2] = 0;
            if (t1 < C) {
                const unsigned long long s1 = starts[t1], n1 = starts[t1 + 1] - s1;
                if (n1 <= p.cap) prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, (size_t)t1 * p.capc, n1);
            }
        }
        if (n == 0) {
            if (tid == 0) range_start[c] = ~0ull;
            continue;
        }
        if (n > p.cap) {                       // overflow path (K4)
            if (tid == 0) {
                if (atomicExch(&big_mark[c], 1u) == 0u) {
                    const unsigned long long k = atomicAdd(&st->big_count, 1ull);
                    big_list[k] = c;
                    atomicAdd(&st->big_elems, (unsigned long long)n);
                    atomicMax(&st->max_coarse, (unsigned long long)n);
                }
            }
            continue;
        }
        if (tid == 0) {
            range_start[c] = S0;
            atomicMax(&st->max_coarse, (unsigned long long)n);
        }
        const size_t rb = (size_t)c * p.capc;
        const KeyT* gk = reg_keys + rb;
        const uint16_t* gf = reg_fine + rb;
        const uint32_t* gi = PERM ? reg_idx + rb : nullptr;

        // ---- 1. histogram of rank buckets (8 fine ids per 128-bit load; rows are 16-B aligned)
        for (uint32_t f = tid; f < p.kfine; f += kL3Threads) hist[f] = 0u;
        __syncthreads();
        const uint32_t n8 = n >> 3;
        const uint4* g8 = reinterpret_cast<const uint4*>(gf);
        {
            uint32_t i = tid;
            for (; i + kL3Threads < n8; i += 2 * kL3Threads) {      // two loads in flight
                const uint4 v = __ldg(g8 + i), w = __ldg(g8 + i + kL3Threads);
                hist_add8(hist, v);
                hist_add8(hist, w);
            }
            if (i < n8) hist_add8(hist, __ldg(g8 + i));
            for (uint32_t t = (n8 << 3) + tid; t < n; t += kL3Threads) atomicAdd(&hist[gf[t]], 1u);
        }
        __syncthreads();
        // ---- 2. exclusive scan of the rank-bucket counts: warp w scans rows of 32 counters
        // of its contiguous chunk (conflict-free), then the warp totals are scanned.
        {
            const int warp = tid >> 5;
            constexpr int kW = kL3Threads / 32;
            const uint32_t chunk = (p.kfine + kW - 1) / kW;
            const uint32_t b0 = min(p.kfine, (uint32_t)warp * chunk), b1 = min(p.kfine, b0 + chunk);
            uint32_t carry = 0;
            for (uint32_t r = b0; r < b1; r += 32) {
                const uint32_t f = r + lane;
                const uint32_t v = f < b1 ? hist[f] : 0u;
                uint32_t x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (f < b1) hist[f] = carry + x - v;             // exclusive within the chunk
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) scratch[warp] = carry;
            __syncthreads();
            if (warp == 0) {
                const uint32_t t = lane < kW ? scratch[lane] : 0u;
                uint32_t x = t;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (lane < kW) scratch[lane] = x - t;
            }
            __syncthreads();
            const uint32_t add = scratch[warp];
            if (add)
                for (uint32_t f = b0 + lane; f < b1; f += 32) hist[f] += add;
        }
        __syncthreads();
        // ---- 3. placement into rank-bucket order: groups of 8 (fine ids + keys loaded as
        // 128-bit vectors, issued before the shared-memory atomics that consume them)
        {
            uint32_t i = tid;
            for (; i < n8; i += kL3Threads) {
                const uint4 fv = __ldg(g8 + i);
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
                    const uint32_t f = (fw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
                    const uint32_t pos = atomicAdd(&hist[f], 1u);
                    skey[pos] = KeyTraits<KeyT>::to_ord(kv[k]);
                    if (PERM) sidx[pos] = iv[k];
                }
            }
            for (uint32_t t = (n8 << 3) + tid; t < n; t += kL3Threads) {
                const uint32_t pos = atomicAdd(&hist[gf[t]], 1u);
                skey[pos] = KeyTraits<KeyT>::to_ord(gk[t]);
                if (PERM) sidx[pos] = gi[t];
            }
        }
        __syncthreads();                       // hist[f] = end of rank bucket f
        // ---- 4. fix-up: sort every rank bucket by (key, index)
        for (uint32_t f = tid; f < p.kfine; f += kL3Threads) {
            const uint32_t s = f ? hist[f - 1] : 0u, e = hist[f];
            const uint32_t len = e - s;
            if (len <= 1) continue;
            if (len <= kInsMax) {
                for (uint32_t i = s + 1; i < e; ++i) {
                    const Bits kv = skey[i];
                    const uint32_t iv = PERM ? sidx[i] : 0u;
                    uint32_t j = i;
                    while (j > s) {
                        const Bits kp = skey[j - 1];
                        const bool gt = PERM ? (kp > kv || (kp == kv && sidx[j - 1] > iv)) : (kp > kv);
                        if (!gt) break;
                        skey[j] = kp;
                        if (PERM) sidx[j] = sidx[j - 1];
                        --j;
                    }
                    skey[j] = kv;
                    if (PERM) sidx[j] = iv;
                }
            } else {
                const uint32_t q = atomicAdd(&ctrl[2], 1u);
                if (q < kL3BigQ) {
                    bigq[2 * q] = s;
                    bigq[2 * q + 1] = e;
                }
            }
        }
        __syncthreads();
        {
            const uint32_t nbig = ctrl[2];
            if (nbig > kL3BigQ) {              // many large rank buckets: sort the whole coarse bucket
                block_bitonic_sort_nt<KeyT, PERM, kL3Threads>(skey, sidx, 0, n);
            } else {
                for (uint32_t q = 0; q < nbig; ++q)
                    block_bitonic_sort_nt<KeyT, PERM, kL3Threads>(skey, sidx, bigq[2 * q], bigq[2 * q + 1]);
            }
        }
        __syncthreads();
        // ---- 5. verify adjacent pairs of the whole coarse bucket (A14), coalesced store
        uint32_t viol = 0;
        for (uint32_t i = tid; i < n; i += kL3Threads) {
            const Bits b = skey[i];
            if (i > 0) {
                const Bits a = skey[i - 1];
                const bool ok = PERM ? precedes<KeyT, true>(a, sidx[i - 1], b, sidx[i]) : (a <= b);
                viol += ok ? 0u : 1u;
            }
            out_keys[S0 + i] = KeyTraits<KeyT>::from_ord(b);
            if (PERM) out_perm[S0 + i] = sidx[i];
        }
        viol_total += viol;
    }
    const uint32_t v = __reduce_add_sync(0xffffffffu, (uint32_t)viol_total);
    if (lane == 0 && v) atomicAdd(&st->violations, (unsigned long long)v);
}

}  // namespace mlsort
