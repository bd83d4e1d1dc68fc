// k4_overflow.cuh -- K4 overflow path, K5 boundary verify, and the conventional-sort
// fallback (a stable LSD radix sort).
//
// The paper sorts the keys that its model cannot place well with "conventional sorting
// algorithms (like Quick Sort)" (§3 l.121, tails) and SPEC escalates to a full
// comparison sort when verification fails.  Here a coarse bucket too large
// for K3's distributed shared memory (heavy duplicates, e.g. BASELINE C5, or a skewed
// model) is first gathered in tile order with each tile's piece sorted by input index, so
// the gathered run is in input order; an all-equal run is then already final (stable
// copy-through), otherwise a stable LSD radix sort by key finishes it.  The same radix
// sort, applied to the whole input, is the fallback when the verify pass finds a
// violation (non-monotone weights, reading A14).
#pragma once

#include "common.cuh"
#include "k3_sort.cuh"

namespace mlsort {

// ------------------------------------------------------------------ K4 copy-out
// Persistent CTAs take big coarse buckets from big_list, copy the bucket's region (K1 left it
// contiguous) to the bucket's output range and test whether all keys are equal.
// flags[k] bit0: all keys bit-identical (a key-only run is then final; a perm run only needs
// its indices sorted).
template <typename KeyT, bool PERM>
__global__ void __launch_bounds__(kK3Threads)
k4_big_copy(uint32_t capc, uint32_t R, const KeyT* __restrict__ reg_keys, const uint32_t* __restrict__ reg_idx,
            const unsigned long long* __restrict__ starts, KeyT* __restrict__ out_keys,
            uint32_t* __restrict__ out_perm, unsigned long long* __restrict__ range_start,
            DevStatus* __restrict__ st, const uint32_t* __restrict__ big_list, uint32_t* __restrict__ flags,
            unsigned long long* __restrict__ ticket, const unsigned long long* __restrict__ rbase) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    __shared__ uint32_t s_k;
    __shared__ unsigned long long s_min, s_max;
    const int tid = threadIdx.x;
    const unsigned long long nbig = st->big_count;
    while (true) {
        if (tid == 0) {
            s_k = (uint32_t)atomicAdd(ticket, 1ull);
            s_min = ~0ull;
            s_max = 0ull;
        }
        __syncthreads();
        const uint32_t k = s_k;
        if (k >= nbig) return;
        const uint32_t c = big_list[k];
        const unsigned long long S0 = starts[c], n_c = starts[c + 1] - S0;
        if (tid == 0) range_start[(size_t)c * R] = S0;
        const size_t rb0 = region_base(rbase, c, capc);
        Bits vmin = ~(Bits)0, vmax = 0;
        for (unsigned long long i = tid; i < n_c; i += kK3Threads) {
            const KeyT key = reg_keys[rb0 + i];
            const Bits ob = KeyTraits<KeyT>::to_ord(key);
            vmin = ob < vmin ? ob : vmin;
            vmax = ob > vmax ? ob : vmax;
            out_keys[S0 + i] = key;
            if (PERM) out_perm[S0 + i] = reg_idx[rb0 + i];
        }
        if (vmin != ~(Bits)0) {
            atomicMin(&s_min, (unsigned long long)vmin);
            atomicMax(&s_max, (unsigned long long)vmax);
        }
        __syncthreads();
        if (tid == 0) {
            const bool equal = (s_min == s_max);
            flags[k] = equal ? 1u : 0u;
            if (!equal || PERM) atomicAdd(&st->overflow, 1ull);   // needs the K4 radix pass
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K5 boundary verify
// Every K3 slice / K4 run recorded its output start; check the pair that straddles it.
template <typename KeyT, bool PERM>
__global__ void k5_boundary_verify(const unsigned long long* __restrict__ range_start, uint64_t num,
                                   const KeyT* __restrict__ out_keys, const uint32_t* __restrict__ out_perm,
                                   DevStatus* __restrict__ st) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= num) return;
    const unsigned long long s = range_start[i];
    if (s == ~0ull || s == 0) return;
    const auto a = KeyTraits<KeyT>::to_ord(out_keys[s - 1]);
    const auto b = KeyTraits<KeyT>::to_ord(out_keys[s]);
    const bool ok = PERM ? precedes<KeyT, true>(a, out_perm[s - 1], b, out_perm[s]) : (a <= b);
    if (!ok) atomicAdd(&st->violations, 1ull);
}

// ------------------------------------------------------------------ LSD radix sort (stable)
constexpr int kRadixThreads = 512;
constexpr int kRadixItems = 16;
constexpr int kRadixChunk = kRadixThreads * kRadixItems;   // 8192

template <typename KeyT>
__global__ void k_to_ord(const KeyT* __restrict__ in, typename KeyTraits<KeyT>::Bits* __restrict__ out,
                         uint32_t* __restrict__ iota, uint64_t n, uint64_t iota_base) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        out[i] = KeyTraits<KeyT>::to_ord(in[i]);
        if (iota) iota[i] = (uint32_t)(iota_base + i);
    }
}
template <typename KeyT>
__global__ void k_from_ord(const typename KeyTraits<KeyT>::Bits* __restrict__ in, KeyT* __restrict__ out,
                           uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = KeyTraits<KeyT>::from_ord(in[i]);
}

// digit of element: from the key bits (field 0) or from the 32-bit payload (field 1)
template <typename Bits>
__device__ __forceinline__ uint32_t radix_digit(Bits k, uint32_t v, int field, int shift) {
    return field == 0 ? (uint32_t)((k >> shift) & 255u) : ((v >> shift) & 255u);
}

template <typename Bits>
__global__ void __launch_bounds__(kRadixThreads)
k_radix_hist(const Bits* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n, int field,
             int shift, uint32_t nchunks, uint32_t* __restrict__ ghist) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += kRadixThreads) h[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kRadixChunk;
    for (int k = 0; k < kRadixItems; ++k) {
        const uint64_t e = base + threadIdx.x + (uint64_t)k * kRadixThreads;
        if (e < n) atomicAdd(&h[radix_digit<Bits>(keys[e], vals ? vals[e] : 0u, field, shift)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += kRadixThreads) ghist[(size_t)d * nchunks + blockIdx.x] = h[d];
}

// Parallel in-place exclusive scan of m u32 entries: k_scan_blocks scans tiles of kScanTile
// entries and records each tile's total, k_radix_scan (one CTA) scans the tile totals, and
// k_scan_add adds every tile's offset.
constexpr int kScanTile = 16384;
static __global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* __restrict__ a, uint64_t m, uint32_t* __restrict__ tot) {
    __shared__ uint32_t scratch[64];
    const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile;
    const uint64_t s = t0 + threadIdx.x * 16ull;
    uint32_t v[16], local = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        v[i] = (s + i < m) ? a[s + i] : 0u;
        local += v[i];
    }
    uint32_t total;
    uint32_t run = block_exclusive_scan<1024>(local, scratch, &total);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (s + i < m) a[s + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = total;
}
static __global__ void k_scan_add(uint32_t* __restrict__ a, uint64_t m, const uint32_t* __restrict__ tot) {
    const uint32_t add = tot[blockIdx.x];
    if (!add) return;
    const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile;
    for (uint32_t i = threadIdx.x; i < kScanTile; i += blockDim.x)
        if (t0 + i < m) a[t0 + i] += add;
}

// in-place exclusive scan of m entries with one CTA (digit-major order)
static __global__ void __launch_bounds__(1024) k_radix_scan(uint32_t* __restrict__ a, uint64_t m) {
    __shared__ uint32_t scratch[64];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint64_t per = 16;
    for (uint64_t b = 0; b < m; b += 1024 * per) {
        const uint64_t s = b + threadIdx.x * per;
        uint32_t local = 0;
        for (uint64_t i = s; i < min(m, s + per); ++i) local += a[i];
        uint32_t total;
        uint32_t run = block_exclusive_scan<1024>(local, scratch, &total) + carry;
        for (uint64_t i = s; i < min(m, s + per); ++i) {
            const uint32_t v = a[i];
            a[i] = run;
            run += v;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
}

// Stable scatter: warp w owns elements [w*512, (w+1)*512) of the chunk, processed in lane order.
template <typename Bits>
__global__ void __launch_bounds__(kRadixThreads)
k_radix_scatter(const Bits* __restrict__ kin, const uint32_t* __restrict__ vin, Bits* __restrict__ kout,
                uint32_t* __restrict__ vout, uint64_t n, int field, int shift, uint32_t nchunks,
                const uint32_t* __restrict__ ghist) {
    constexpr int W = kRadixThreads / 32;
    __shared__ uint16_t wcnt[W][256];
    __shared__ uint32_t goff[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < W * 256; i += kRadixThreads) (&wcnt[0][0])[i] = 0;
    for (int d = threadIdx.x; d < 256; d += kRadixThreads) goff[d] = ghist[(size_t)d * nchunks + blockIdx.x];
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kRadixChunk + (uint64_t)warp * 32 * kRadixItems;
    Bits k[kRadixItems];
    uint32_t v[kRadixItems], rank[kRadixItems], dig[kRadixItems];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t e = base + (uint64_t)r * 32 + lane;
        const bool ok = e < n;
        k[r] = ok ? kin[e] : (Bits)0;
        v[r] = (ok && vin) ? vin[e] : 0u;
        dig[r] = ok ? radix_digit<Bits>(k[r], v[r], field, shift) : 256u + lane;   // unique dummy
        const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
        const uint32_t before = ok ? wcnt[warp][dig[r]] : 0u;
        rank[r] = before + __popc(peers & lt);
        __syncwarp();
        if (ok && (peers & lt) == 0) wcnt[warp][dig[r]] = (uint16_t)(before + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps for each digit
    for (int d = threadIdx.x; d < 256; d += kRadixThreads) {
        uint32_t run = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = (uint16_t)run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t e = base + (uint64_t)r * 32 + lane;
        if (e < n) {
            const uint64_t dst = (uint64_t)goff[dig[r]] + wcnt[warp][dig[r]] + rank[r];
            kout[dst] = k[r];
            if (vout) vout[dst] = v[r];
        }
    }
}

// ------------------------------------------------------------------ batched overflow sort
// The overflow buckets are sorted together: their ranges are gathered into one contiguous
// array (order-preserving key bits + index), that array is radix-sorted once, and the result is
// scattered back range by range.  Valid because the network is monotone: every key of an
// earlier coarse bucket precedes every key of a later one, so the sorted union splits into the
// sorted buckets in order.
template <typename KeyT>
__global__ void k_seg_gather(const unsigned long long* __restrict__ seg, uint32_t nseg, const KeyT* __restrict__ keys,
                             const uint32_t* __restrict__ perm, typename KeyTraits<KeyT>::Bits* __restrict__ tk,
                             uint32_t* __restrict__ tv) {
    for (uint32_t g = blockIdx.x; g < nseg; g += gridDim.x) {
        const unsigned long long src = seg[3 * g], dst = seg[3 * g + 1], len = seg[3 * g + 2];
        for (unsigned long long i = threadIdx.x; i < len; i += blockDim.x) {
            tk[dst + i] = KeyTraits<KeyT>::to_ord(keys[src + i]);
            if (tv) tv[dst + i] = perm[src + i];
        }
    }
}
template <typename KeyT>
__global__ void k_seg_scatter(const unsigned long long* __restrict__ seg, uint32_t nseg,
                              const typename KeyTraits<KeyT>::Bits* __restrict__ tk, const uint32_t* __restrict__ tv,
                              KeyT* __restrict__ keys, uint32_t* __restrict__ perm) {
    for (uint32_t g = blockIdx.x; g < nseg; g += gridDim.x) {
        const unsigned long long src = seg[3 * g], dst = seg[3 * g + 1], len = seg[3 * g + 2];
        for (unsigned long long i = threadIdx.x; i < len; i += blockDim.x) {
            keys[src + i] = KeyTraits<KeyT>::from_ord(tk[dst + i]);
            if (tv) perm[src + i] = tv[dst + i];
        }
    }
}

// ------------------------------------------------------------------ misc
template <typename KeyT>
__global__ void k_gather_payload(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ payload,
                                 uint32_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = payload[perm[i]];
}

}  // namespace mlsort
