// k4_overflow.cuh -- K5 boundary verify, and the stable LSD radix sort that finishes what the
// rank buckets cannot.
//
// The paper sorts the keys its model cannot place well with "conventional sorting algorithms
// (like Quick Sort)" (§3 l.121, tails), and SPEC escalates to a full comparison sort
// when verification fails.  Here the radix sort (8-bit digits, stable,
// digit-major chunk histograms, smem-staged coalesced scatter) sorts (a) the SEGMENTS k3_cut
// hands over -- a single rank bucket larger than a CTA whose keys differ, or an all-equal run
// of a permutation sort, which only needs its input indices ordered (k3_big.cuh) -- gathered
// into one array, sorted once and scattered back (valid because the monotone network orders
// the segments), and (b) the whole input when a verify pass finds a violation (a non-monotone
// model, reading A14).
#pragma once

#include "common.cuh"
#include "k3_sort.cuh"

namespace mlsort {

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
        if (e < n) {   // read only the array the digit comes from
            const uint32_t d = field == 0 ? (uint32_t)((keys[e] >> shift) & 255u) : ((vals[e] >> shift) & 255u);
            atomicAdd(&h[d], 1u);
        }
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
// Every element's rank among the chunk's elements of its digit is computed first; the chunk is
// then laid out in digit order in shared memory and written out position by position, so the
// consecutive threads of a warp store consecutive addresses of one digit's run (coalesced)
// instead of 32 scattered 4-byte stores per warp instruction.
template <typename Bits>
__global__ void __launch_bounds__(kRadixThreads)
k_radix_scatter(const Bits* __restrict__ kin, const uint32_t* __restrict__ vin, Bits* __restrict__ kout,
                uint32_t* __restrict__ vout, uint64_t n, int field, int shift, uint32_t nchunks,
                const uint32_t* __restrict__ ghist) {
    constexpr int W = kRadixThreads / 32;
    __shared__ uint16_t wcnt[W][256];
    __shared__ uint32_t goff[256], loff[257];
    extern __shared__ __align__(16) unsigned char rsm[];     // chunk in digit order (dynamic)
    Bits* sk = reinterpret_cast<Bits*>(rsm);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kRadixChunk);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < W * 256; i += kRadixThreads) (&wcnt[0][0])[i] = 0;
    for (int d = threadIdx.x; d < 256; d += kRadixThreads) goff[d] = ghist[(size_t)d * nchunks + blockIdx.x];
    __syncthreads();
    const uint64_t cbase = (uint64_t)blockIdx.x * kRadixChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kRadixChunk, n - cbase);
    const uint64_t base = cbase + (uint64_t)warp * 32 * kRadixItems;
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
    // exclusive prefix over warps for each digit, and the chunk-local start of each digit
    if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        uint32_t run = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = (uint16_t)run;
            run += c;
        }
        loff[d] = run;                                // digit total (scanned below)
    }
    __syncthreads();
    if (threadIdx.x < 32) {                           // exclusive scan of the 256 digit totals
        uint32_t t[8], sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            t[i] = loff[threadIdx.x * 8 + i];
            sum += t[i];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t run = x - sum;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            loff[threadIdx.x * 8 + i] = run;
            run += t[i];
        }
        if (threadIdx.x == 31) loff[256] = run;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t e = base + (uint64_t)r * 32 + lane;
        if (e < n) {
            const uint32_t lp = loff[dig[r]] + wcnt[warp][dig[r]] + rank[r];
            sk[lp] = k[r];
            if (vout) sv[lp] = v[r];
        }
    }
    __syncthreads();
    for (uint32_t lp = threadIdx.x; lp < cnt; lp += kRadixThreads) {
        const Bits kk = sk[lp];
        const uint32_t vv = vout ? sv[lp] : 0u;
        const uint32_t d = radix_digit<Bits>(kk, vv, field, shift);
        const uint64_t dst = (uint64_t)goff[d] + (lp - loff[d]);
        kout[dst] = kk;
        if (vout) vout[dst] = vv;
    }
}

template <typename Bits>
constexpr size_t radix_scatter_smem() { return (size_t)kRadixChunk * (sizeof(Bits) + 4); }

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

// all-equal runs: the radix key is the run's ordinal g (runs are gathered in output order), the
// value the input index; only the indices are scattered back
template <typename Bits>
__global__ void k_seg_gather_ordinal(const unsigned long long* __restrict__ seg, uint32_t nseg,
                                     const uint32_t* __restrict__ perm, Bits* __restrict__ tk,
                                     uint32_t* __restrict__ tv) {
    for (uint32_t g = blockIdx.x; g < nseg; g += gridDim.x) {
        const unsigned long long src = seg[3 * g], dst = seg[3 * g + 1], len = seg[3 * g + 2];
        for (unsigned long long i = threadIdx.x; i < len; i += blockDim.x) {
            tk[dst + i] = (Bits)g;
            tv[dst + i] = perm[src + i];
        }
    }
}
static __global__ void k_seg_scatter_perm(const unsigned long long* __restrict__ seg, uint32_t nseg,
                                          const uint32_t* __restrict__ tv, uint32_t* __restrict__ perm) {
    for (uint32_t g = blockIdx.x; g < nseg; g += gridDim.x) {
        const unsigned long long src = seg[3 * g], dst = seg[3 * g + 1], len = seg[3 * g + 2];
        for (unsigned long long i = threadIdx.x; i < len; i += blockDim.x) perm[src + i] = tv[dst + i];
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
