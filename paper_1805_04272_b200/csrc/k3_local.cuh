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
//   4. fix-up fused with the store: every position ranks its element inside its rank bucket
//      by counting the bucket's elements that precede it under (totalOrder key, input index)
//      and writes it to its final position; large buckets get a block bitonic sort     -- A6
//   5. when the weights are not provably monotone: the stored output is checked at every
//      rank-bucket boundary and an inversion re-sorts the whole coarse bucket    -- A7 (A14)
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
constexpr uint32_t kL3RankMax = 64;     // rank buckets up to this size: rank by counting
constexpr uint32_t kL3BigQ = 48;        // queued larger rank buckets per coarse bucket

struct K3LParams {
    uint32_t capc;          // region capacity (elements) per coarse bucket
    uint32_t num_coarse;    // C
    uint32_t kfine;         // rank buckets per coarse bucket (2^fine_bits)
    uint32_t cap;           // largest coarse bucket this pass holds in shared memory
    uint32_t verify;        // 1: check every rank-bucket boundary (weights not provably monotone)
    uint32_t secondary;     // 0: pass over all coarse buckets; 1: pass over mid_list
    uint32_t to_mid;        // too-large buckets go to mid_list (1, primary of two passes) or to
                            // K4's big_list (0)
};

// The rank-bucket histogram holds two u16 counters per 32-bit word (a coarse bucket never
// exceeds 65535 elements here); words rounded up to 4 so the key array after it is 16-B aligned.
__host__ __device__ inline uint32_t k3l_hist_words(uint32_t kfine) { return ((kfine + 1u) / 2u + 3u) & ~3u; }

// smem: ctrl | hist (u16 pairs) | skey[cap] | sidx[cap] (perm) | sfine[cap] u16
inline size_t k3l_smem_bytes(size_t ks, bool perm, uint32_t kfine, uint32_t cap) {
    return kCtrlBytes + (size_t)k3l_hist_words(kfine) * 4 + (size_t)cap * ks + (perm ? (size_t)cap * 4 : 0) +
           (size_t)cap * 2;
}

// largest cap with k3l_smem_bytes(...) <= budget
inline uint32_t k3l_cap_for(size_t budget, size_t ks, bool perm, uint32_t kfine) {
    const size_t fixed = kCtrlBytes + (size_t)k3l_hist_words(kfine) * 4;
    if (budget <= fixed) return 0;
    const size_t leb = ks + (perm ? 4 : 0) + 2;
    uint64_t cap = std::min<uint64_t>((budget - fixed) / leb, 65535ull);
    while (cap > 0 && k3l_smem_bytes(ks, perm, kfine, (uint32_t)cap) > budget) --cap;
    return (uint32_t)cap;
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


template <typename KeyT, bool PERM, int NT>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : 2)
k3_local_sort(K3LParams p, const KeyT* __restrict__ reg_keys, const uint16_t* __restrict__ reg_fine,
              const uint32_t* __restrict__ reg_idx, const unsigned long long* __restrict__ starts,
              KeyT* __restrict__ out_keys, uint32_t* __restrict__ out_perm,
              unsigned long long* __restrict__ range_start, DevStatus* __restrict__ st,
              uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_mark, uint32_t* __restrict__ mid_list,
              unsigned long long* __restrict__ ticket, const unsigned long long* __restrict__ rbase) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    // ctrl words: [1] next ticket, [2] big-queue count, [8..40) scan scratch,
    // [64 .. 64+3*kL3BigQ) big-queue (start, end, rank bucket) triples
    uint32_t* ctrl = reinterpret_cast<uint32_t*>(smem);
    uint32_t* scratch = ctrl + 8;
    uint32_t* bigq = ctrl + 64;
    uint32_t* h2 = reinterpret_cast<uint32_t*>(smem + kCtrlBytes);          // u16 counter pairs
    Bits* skey = reinterpret_cast<Bits*>(h2 + k3l_hist_words(p.kfine));
    uint32_t* sidx = reinterpret_cast<uint32_t*>(skey + p.cap);
    uint16_t* sfine = reinterpret_cast<uint16_t*>(sidx + (PERM ? p.cap : 0));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // work items: coarse ids 0..C-1 (primary) or mid_list[0..mid_count) (secondary)
    const uint32_t items = p.secondary ? (uint32_t)st->mid_count : p.num_coarse;
    auto coarse_of = [&](uint32_t t) { return p.secondary ? mid_list[t] : t; };
    const uint32_t hw = (p.kfine + 1u) / 2u;           // histogram words
    if (tid == 0) {
        const uint32_t t0 = (uint32_t)atomicAdd(ticket, 1ull);
        ctrl[1] = t0;
        if (t0 < items) {
            const uint32_t c0 = coarse_of(t0);
            const unsigned long long s0 = starts[c0], n0 = starts[c0 + 1] - s0;
            if (n0 <= p.cap) prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, region_base(rbase, c0, p.capc), n0);
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
        const uint32_t c = coarse_of(t);
        const unsigned long long S0 = starts[c];
        const uint32_t n = (uint32_t)min(starts[c + 1] - S0, (unsigned long long)0xffffffffull);
        __syncthreads();                       // everyone read ctrl[1]
        if (tid == 0) {                        // take the next bucket now and prefetch it into L2
            const uint32_t t1 = (uint32_t)atomicAdd(ticket, 1ull);
            ctrl[1] = t1;
            ctrl[2] = 0;
            if (t1 < items) {
                const uint32_t c1 = coarse_of(t1);
                const unsigned long long s1 = starts[c1], n1 = starts[c1 + 1] - s1;
                if (n1 <= p.cap) prefetch_bucket<KeyT, PERM>(reg_keys, reg_fine, reg_idx, region_base(rbase, c1, p.capc), n1);
            }
        }
        if (n == 0) {
            if (tid == 0) range_start[c] = ~0ull;
            continue;
        }
        if (n > p.cap) {                       // too large for this pass
            if (tid == 0) {
                atomicMax(&st->max_coarse, (unsigned long long)n);
                if (p.to_mid) {
                    mid_list[atomicAdd(&st->mid_count, 1ull)] = c;
                } else if (atomicExch(&big_mark[c], 1u) == 0u) {
                    const unsigned long long k = atomicAdd(&st->big_count, 1ull);
                    big_list[k] = c;
                    atomicAdd(&st->big_elems, (unsigned long long)n);
                }
            }
            continue;
        }
        if (tid == 0) {
            range_start[c] = S0;
            atomicMax(&st->max_coarse, (unsigned long long)n);
        }
        const size_t rb = region_base(rbase, c, p.capc);
        const KeyT* gk = reg_keys + rb;
        const uint16_t* gf = reg_fine + rb;
        const uint32_t* gi = PERM ? reg_idx + rb : nullptr;
        const uint32_t n8 = n >> 3;
        const uint4* g8 = reinterpret_cast<const uint4*>(gf);

        // ---- 1. histogram of rank buckets (8 ids per 128-bit load; rows are 16-B aligned)
        for (uint32_t w = tid; w < hw; w += NT) h2[w] = 0u;
        __syncthreads();
        {
            uint32_t i = tid;
            for (; i + NT < n8; i += 2 * NT) {                    // two loads in flight
                const uint4 v = __ldg(g8 + i), w = __ldg(g8 + i + NT);
                hist_add8(h2, v);
                hist_add8(h2, w);
            }
            if (i < n8) hist_add8(h2, __ldg(g8 + i));
            for (uint32_t q = (n8 << 3) + tid; q < n; q += NT) hist_inc(h2, gf[q]);
        }
        __syncthreads();
        K3L_T(1);
        // ---- 2. exclusive scan of the counters: warp w owns a contiguous chunk of words; 8 rows
        // of 32 words are loaded and warp-scanned independently (ILP), then chained by their
        // totals; finally the warp totals are scanned across the CTA
        {
            constexpr int kW = NT / 32;
            const uint32_t chunk = (((hw + kW - 1) / kW) + 31u) & ~31u;
            const uint32_t b0 = min(hw, (uint32_t)warp * chunk), b1 = min(hw, b0 + chunk);
            uint32_t carry = 0;
            for (uint32_t r0 = b0; r0 < b1; r0 += 256) {
                uint32_t v[8], x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t w = r0 + 32 * k + lane;
                    v[k] = w < b1 ? h2[w] : 0u;
                    x[k] = (v[k] & 0xffffu) + (v[k] >> 16);
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t yy = __shfl_up_sync(0xffffffffu, x[k], o);
                        if (lane >= o) x[k] += yy;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t w = r0 + 32 * k + lane;
                    const uint32_t lo = v[k] & 0xffffu;
                    const uint32_t ex = carry + x[k] - (lo + (v[k] >> 16));
                    if (w < b1) h2[w] = ex | ((ex + lo) << 16);
                    carry += __shfl_sync(0xffffffffu, x[k], 31);
                }
            }
            if (lane == 0) scratch[warp] = carry;
            __syncthreads();
            if (warp == 0) {
                const uint32_t tt = lane < kW ? scratch[lane] : 0u;
                uint32_t x = tt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t yy = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += yy;
                }
                if (lane < kW) scratch[lane] = x - tt;
            }
            __syncthreads();
            const uint32_t add = scratch[warp];
            if (add)
                for (uint32_t w = b0 + lane; w < b1; w += 32) h2[w] += add | (add << 16);
        }
        __syncthreads();
        K3L_T(2);
        // ---- 3. placement into rank-bucket order (ids + keys as 128-bit vectors)
        for (uint32_t i = tid; i < n8; i += NT) {
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
                const uint32_t pos = hist_inc_ret(h2, f);
                skey[pos] = KeyTraits<KeyT>::to_ord(kv[k]);
                sfine[pos] = (uint16_t)f;
                if (PERM) sidx[pos] = iv[k];
            }
        }
        for (uint32_t q = (n8 << 3) + tid; q < n; q += NT) {
            const uint32_t f = gf[q];
            const uint32_t pos = hist_inc_ret(h2, f);
            skey[pos] = KeyTraits<KeyT>::to_ord(gk[q]);
            sfine[pos] = (uint16_t)f;
            if (PERM) sidx[pos] = gi[q];
        }
        __syncthreads();                       // counter f = end of rank bucket f
        K3L_T(3);
        // ---- 4. fix-up fused with the store ("only the numbers inside each bucket need to
        // be sorted"): each position ranks its element inside its rank bucket [s, e) by counting
        // the elements that precede it under (totalOrder key, index) and writes it to its final
        // output position.  Buckets of <= 4 elements (98 % of the keys for a Poisson(1) fill) use
        // a fixed predicated compare sequence, up to kL3RankMax a loop, larger ones are queued
        // for a block-wide sort.
        for (uint32_t pos = tid; pos < n; pos += NT) {
            const uint32_t f = sfine[pos];
            const uint32_t e = hist_get(h2, f), s = f ? hist_get(h2, f - 1) : 0u;
            const uint32_t len = e - s;
            const Bits kv = skey[pos];
            const uint32_t iv = PERM ? sidx[pos] : pos;
            uint32_t rank = 0;
#if defined(MLSORT_K3L_EXPT) && MLSORT_K3L_EXPT == 2
            if (false) {                       // experiment: no ranking
#else
            if (len > 1) {
#endif
                if (len <= 4) {                // the common case: fixed, predicated compares
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        if (q < len) {
                            const Bits kq = skey[s + q];
                            const uint32_t iq = PERM ? sidx[s + q] : s + q;
                            rank += (kq < kv || (kq == kv && iq < iv)) ? 1u : 0u;
                        }
                    }
                } else if (len <= kL3RankMax) {
                    for (uint32_t q = s; q < e; ++q) {
                        const Bits kq = skey[q];
                        const uint32_t iq = PERM ? sidx[q] : q;
                        rank += (kq < kv || (kq == kv && iq < iv)) ? 1u : 0u;
                    }
                } else {                       // large bucket: block-wide sort below
                    if (pos == s) {
                        const uint32_t q = atomicAdd(&ctrl[2], 1u);
                        if (q < kL3BigQ) {
                            bigq[3 * q] = s;
                            bigq[3 * q + 1] = e;
                            bigq[3 * q + 2] = f;
                        }
                    }
                    continue;
                }
            }
#if defined(MLSORT_K3L_EXPT) && MLSORT_K3L_EXPT == 1
            if (rank == 0xffffffffu) out_keys[S0] = KeyTraits<KeyT>::from_ord(kv);   // experiment: no store
#else
            out_keys[S0 + s + rank] = KeyTraits<KeyT>::from_ord(kv);
            if (PERM) out_perm[S0 + s + rank] = iv;
#endif
        }
        __syncthreads();
        K3L_T(4);
        // ---- 5. large rank buckets (tails collected in the end buckets, heavy duplicates):
        // block-wide bitonic sort in shared memory, then store
        const uint32_t nbig = ctrl[2];
        if (nbig <= kL3BigQ) {
            for (uint32_t q = 0; q < nbig; ++q) {
                const uint32_t s = bigq[3 * q], e = bigq[3 * q + 1];
                block_bitonic_sort_nt<KeyT, PERM, NT>(skey, sidx, s, e);
                for (uint32_t i = s + tid; i < e; i += NT) {
                    out_keys[S0 + i] = KeyTraits<KeyT>::from_ord(skey[i]);
                    if (PERM) out_perm[S0 + i] = sidx[i];
                }
            }
        }
        __syncthreads();                       // this CTA's output stores are visible to it
        K3L_T(5);
        // ---- 5b. weights not provably monotone: verify every rank-bucket boundary on the stored
        // output (the last element of every non-empty bucket against the first of the next one)
        bool bad = false;
        for (uint32_t f0 = tid; p.verify && f0 < p.kfine; f0 += 4 * NT) {
            Bits ka[4], kb[4];
            uint32_t ia[4], ib[4];
            bool chk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t f = f0 + u * NT;
                const uint32_t e = f < p.kfine ? hist_get(h2, f) : 0u;
                const uint32_t s = (f < p.kfine && f) ? hist_get(h2, f - 1) : 0u;
                chk[u] = e > s && e < n;
                if (chk[u]) {
                    ka[u] = KeyTraits<KeyT>::to_ord(out_keys[S0 + e - 1]);
                    kb[u] = KeyTraits<KeyT>::to_ord(out_keys[S0 + e]);
                    if (PERM) {
                        ia[u] = out_perm[S0 + e - 1];
                        ib[u] = out_perm[S0 + e];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (chk[u]) bad |= PERM ? !precedes<KeyT, true>(ka[u], ia[u], kb[u], ib[u]) : (kb[u] < ka[u]);
        }
        // ---- 6. an inversion between rank buckets (ulp-level non-monotone network output, or a
        // non-monotone model), or too many large buckets: sort the whole coarse bucket
        if (__syncthreads_or(bad) || nbig > kL3BigQ) {
            block_bitonic_sort_nt<KeyT, PERM, NT>(skey, sidx, 0, n);
            for (uint32_t i = tid; i < n; i += NT) {
                out_keys[S0 + i] = KeyTraits<KeyT>::from_ord(skey[i]);
                if (PERM) out_perm[S0 + i] = sidx[i];
            }
            if (tid == 0 && nbig <= kL3BigQ) atomicAdd(&st->local_repairs, 1ull);
        }
        K3L_T(6);
    }
#ifdef MLSORT_K3L_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 1024)
        for (int i = 0; i < 8; ++i) g_k3l_phase[blockIdx.x][i] = (unsigned long long)k3l_acc[i];
#endif
}

}  // namespace mlsort
