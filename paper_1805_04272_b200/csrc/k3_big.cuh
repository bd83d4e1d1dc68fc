// k3_big.cuh -- K3 for coarse buckets larger than one CTA's shared memory (skewed models:
// BASELINE C3/C4; heavy duplicates: C5).
//
// PAPER.md §2 l.86: "only the numbers inside each bucket need to be sorted".  A coarse bucket
// too large for k3_local_sort is cut at rank-bucket boundaries into ITEMS of consecutive rank
// buckets that each fit one CTA; the round pass of k3_local_sort (ITEMS = true) then sorts
// every item exactly like a coarse bucket, reading the coarse region and keeping only the
// item's rank buckets.  A single rank bucket larger than a CTA (many copies of one key, or the
// clamped end buckets of a poorly fitted tail) is copied to its output range here; an
// all-equal key-only run is then final, anything else becomes a SEGMENT for the stable radix
// pass (k4_overflow.cuh).  Output ranges follow the rank-bucket prefix sums, so with a
// monotone model the items and segments tile the coarse bucket's output range in order; K5
// checks every item / segment boundary (reading A14).
#pragma once

#include "common.cuh"

namespace mlsort {

constexpr int kCutThreads = 1024;
constexpr int kMaxGiants = 32;      // giant rank buckets per coarse bucket handled one by one
constexpr uint32_t kCutGroups = 16384;   // k3_cut cuts at groups of 2^gshift rank buckets

struct K3CutParams {
    uint32_t capc;          // fixed region capacity (regions at c * capc unless rbase)
    uint32_t kfine;         // rank buckets per coarse bucket
    uint32_t cap;           // keys one round-pass CTA holds
    uint32_t item_cap;      // capacity of the item list
    uint32_t seg_cap;       // capacity of the segment list
    uint32_t gshift;        // rank buckets are cut in groups of 2^gshift (kfine >> gshift <= kCutGroups)
};

// items of at most `cap` keys: rank bucket f starts a new item when the running prefix P(f)
// enters a new multiple of T = cap/2 or when f or f-1 is heavy (more than cap - T keys); so a
// light item holds < T + (cap - T) = cap keys and a heavy rank bucket is an item of its own
__device__ __forceinline__ bool k3c_starts(uint32_t f, const uint32_t* P, uint32_t T, uint32_t heavy) {
    if (f == 0) return true;
    const uint32_t c0 = P[f] - P[f - 1], c1 = P[f + 1] - P[f];
    if (c0 > heavy || c1 > heavy) return true;
    return P[f] / T != P[f - 1] / T;
}

template <typename KeyT, bool PERM>
__global__ void __launch_bounds__(kCutThreads, 1)
k3_cut(K3CutParams p, const KeyT* __restrict__ reg_keys, const uint16_t* __restrict__ reg_fine,
       const uint32_t* __restrict__ reg_idx, const unsigned long long* __restrict__ starts,
       const uint32_t* __restrict__ big_list, DevStatus* __restrict__ st, K3Item* __restrict__ items,
       K3Seg* __restrict__ segs, KeyT* __restrict__ out_keys, uint32_t* __restrict__ out_perm,
       unsigned long long* __restrict__ range_start, const unsigned long long* __restrict__ rbase) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* P = reinterpret_cast<uint32_t*>(smem);               // [K + 1] group counts -> prefix
    uint32_t* S = P + (p.kfine >> p.gshift) + 1;                    // [K + 1] item starts / giant map
    __shared__ uint32_t s_t, s_nitems, s_ngiant, s_base, s_whole, s_ovf;
    __shared__ uint32_t scratch[kCutThreads / 32 + 1];
    __shared__ uint32_t g_f[kMaxGiants], g_cur[kMaxGiants];
    __shared__ unsigned long long g_out[kMaxGiants], g_min[kMaxGiants], g_max[kMaxGiants];
    const int tid = threadIdx.x;
    const uint32_t K = p.kfine >> p.gshift;          // groups of rank buckets
    const uint32_t gs = p.gshift;
    const uint32_t T = max(1u, p.cap / 2), heavy = p.cap - T;
    const uint32_t per = (K + kCutThreads - 1) / kCutThreads;       // rank buckets per thread
    const uint32_t f0 = min(K, (uint32_t)tid * per), f1 = min(K, f0 + per);
    // a region overflowed in K1: the regions are incomplete (the call re-runs with an exact
    // layout), and a region's count may exceed what it holds -- read nothing
    if (st->region_overflow) return;
    while (true) {
        if (tid == 0) s_t = (uint32_t)atomicAdd(&st->ticket3c, 1ull);
        __syncthreads();
        const uint32_t t = s_t;
        if (t >= (uint32_t)st->big_count) break;
        const uint32_t c = big_list[t];
        const unsigned long long S0 = starts[c];
        const uint32_t n = (uint32_t)(starts[c + 1] - S0);
        const size_t rb = region_base(rbase, c, p.capc);
        if (tid == 0) range_start[c] = S0;
        // ---- histogram of the rank buckets (u32 counters)
        for (uint32_t f = tid; f <= K; f += kCutThreads) P[f] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kCutThreads) atomicAdd(&P[(uint32_t)reg_fine[rb + i] >> gs], 1u);
        __syncthreads();
        // ---- exclusive prefix P[f], P[K] = n
        {
            uint32_t loc = 0;
            for (uint32_t f = f0; f < f1; ++f) loc += P[f];
            uint32_t tot;
            uint32_t run = block_exclusive_scan<kCutThreads>(loc, scratch, &tot);
            for (uint32_t f = f0; f < f1; ++f) {
                const uint32_t v = P[f];
                P[f] = run;
                run += v;
            }
            if (tid == 0) P[K] = tot;
        }
        __syncthreads();
        // ---- item starts, item index by a block scan of the start flags
        uint32_t nst = 0, ngi = 0;
        for (uint32_t f = f0; f < f1; ++f) {
            if (k3c_starts(f, P, T, heavy)) ++nst;
            ngi += (P[f + 1] - P[f] > p.cap) ? 1u : 0u;
        }
        uint32_t tot_items, tot_giant;
        const uint32_t ibase = block_exclusive_scan<kCutThreads>(nst, scratch, &tot_items);
        __syncthreads();
        const uint32_t gbase = block_exclusive_scan<kCutThreads>(ngi, scratch, &tot_giant);
        {
            uint32_t k = ibase, g = gbase;
            for (uint32_t f = f0; f < f1; ++f) {
                if (k3c_starts(f, P, T, heavy)) S[k++] = f;
                if (P[f + 1] - P[f] > p.cap && g < kMaxGiants) {
                    g_f[g] = f;
                    g_out[g] = S0 + P[f];
                    g_cur[g] = 0u;
                    g_min[g] = ~0ull;
                    g_max[g] = 0ull;
                    ++g;
                }
            }
        }
        if (tid == 0) {
            S[tot_items] = K;
            s_nitems = tot_items;
            s_ngiant = tot_giant;
            // too many giants for the per-bucket table, or no room left in the item list: the
            // whole coarse bucket becomes one segment for the radix pass
            s_whole = tot_giant > (uint32_t)kMaxGiants ? 1u : 0u;
            s_ovf = 0u;
            if (!s_whole) {
                const unsigned long long b = atomicAdd(&st->item_count, (unsigned long long)tot_items);
                if (b + tot_items > p.item_cap) {       // (the reserved slots below item_cap are
                    s_whole = 1u;                       //  still written, as empty items)
                    s_ovf = 1u;
                    atomicAdd(&st->item_overflow, 1ull);
                }
                s_base = (uint32_t)min(b, (unsigned long long)p.item_cap);
            }
        }
        __syncthreads();
        const uint32_t nitems = s_nitems;
        if (!s_whole || s_ovf) {
            // ---- emit the items (giant ones are copied below and written as empty items so
            // the list stays dense; the round pass skips empty items)
            for (uint32_t k = tid; k < nitems && s_base + k < p.item_cap; k += kCutThreads) {
                const uint32_t lo = S[k], hi = S[k + 1];
                const uint32_t cnt = P[hi] - P[lo];
                K3Item it;
                it.c = c;
                it.f_lo = lo << gs;
                it.f_hi = min(p.kfine, hi << gs);
                it.cnt = (s_ovf || (hi - lo == 1 && cnt > p.cap)) ? 0u : cnt;
                it.out = S0 + P[lo];
                items[s_base + k] = it;
            }
        }
        __syncthreads();
        const uint32_t ngiant = s_whole ? 0u : min(s_ngiant, (uint32_t)kMaxGiants);
        if (s_whole || ngiant > 0) {
            // ---- giant rank buckets (or the whole bucket): copy to the output range, min/max
            if (!s_whole) {
                for (uint32_t f = tid; f < K; f += kCutThreads) S[f] = 0u;   // giant map: f -> j + 1
                __syncthreads();
                for (uint32_t j = tid; j < ngiant; j += kCutThreads) S[g_f[j]] = j + 1;
            } else if (tid == 0) {
                g_out[0] = S0;
                g_cur[0] = 0u;
                g_min[0] = ~0ull;
                g_max[0] = 0ull;
            }
            __syncthreads();
            Bits lmin = ~(Bits)0, lmax = 0;
            int lj = -1;
            for (uint32_t i = tid; i < n; i += kCutThreads) {
                const uint32_t f = (uint32_t)reg_fine[rb + i] >> gs;
                int j;
                if (s_whole) j = 0;
                else j = (int)S[f] - 1;
                if (j < 0) continue;
                const KeyT key = reg_keys[rb + i];
                const Bits ob = KeyTraits<KeyT>::to_ord(key);
                const unsigned long long pos = g_out[j] + atomicAdd(&g_cur[j], 1u);
                out_keys[pos] = key;
                if (PERM) out_perm[pos] = reg_idx[rb + i];
                if (j != lj) {                        // flush the running min/max of the last run
                    if (lj >= 0) {
                        atomicMin(&g_min[lj], (unsigned long long)lmin);
                        atomicMax(&g_max[lj], (unsigned long long)lmax);
                    }
                    lj = j;
                    lmin = ~(Bits)0;
                    lmax = 0;
                }
                lmin = ob < lmin ? ob : lmin;
                lmax = ob > lmax ? ob : lmax;
            }
            if (lj >= 0) {
                atomicMin(&g_min[lj], (unsigned long long)lmin);
                atomicMax(&g_max[lj], (unsigned long long)lmax);
            }
            __syncthreads();
            const uint32_t nseg = s_whole ? 1u : ngiant;
            for (uint32_t j = tid; j < nseg; j += kCutThreads) {
                const bool equal = g_min[j] == g_max[j];
                const unsigned long long len = s_whole ? n : (unsigned long long)(P[g_f[j] + 1] - P[g_f[j]]);
                if (!equal || PERM) {                 // an all-equal key-only run is final
                    const unsigned long long k = atomicAdd(&st->seg_count, 1ull);
                    if (k < p.seg_cap) {
                        K3Seg sg;
                        sg.out = g_out[j];
                        sg.len = len;
                        sg.flags = equal ? 1u : 0u;
                        sg.pad = 0u;
                        segs[k] = sg;
                    } else {
                        atomicAdd(&st->item_overflow, 1ull);
                    }
                }
            }
        }
        __syncthreads();
    }
}

// Giant all-equal runs of a permutation sort (C5: 131072 copies of each of 4096 values): the
// keys are final, only the input indices of the run must become ascending (stability, reading
// A9).  One CTA (512 threads, three per SM) per run: min/max of the indices, a counting pass into nsb = len/32 index ranges
// (sub-buckets of ~32), a scatter into the scratch area, then every sub-bucket is ranked by
// one warp (<= 32: register shuffles; <= 224: shared memory) and written back, and the run is
// checked to be strictly ascending.  Runs longer than kIdxSortMax, or with a sub-bucket over
// 224 indices (a clustered index set), are flagged (seg.pad = 1) for the radix pass instead.
constexpr uint32_t kIdxSortMax = 1u << 21;
constexpr uint32_t kIdxSub = 4096;           // max sub-buckets per run
constexpr uint32_t kIdxWarpBuf = 224;

// Every element of the u32 run v[0, len) once, in 128-bit loads where aligned (scalar head and
// tail): fn(i, value) for the block's threads.
template <int NT, typename Fn>
__device__ __forceinline__ void for_each_u32(const uint32_t* v, uint32_t len, Fn&& fn) {
    const uint32_t head = min(len, (uint32_t)((16u - ((uint32_t)reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
    if (threadIdx.x < head) fn(threadIdx.x, v[threadIdx.x]);
    const uint32_t nv = (len - head) / 4u;
    const uint4* v4 = reinterpret_cast<const uint4*>(v + head);
    for (uint32_t k = threadIdx.x; k < nv; k += NT) {
        const uint4 q = v4[k];
        const uint32_t i = head + 4u * k;
        fn(i, q.x);
        fn(i + 1, q.y);
        fn(i + 2, q.z);
        fn(i + 3, q.w);
    }
    for (uint32_t i = head + 4u * nv + threadIdx.x; i < len; i += NT) fn(i, v[i]);
}

template <int NT>
__global__ void __launch_bounds__(NT, NT == 512 ? 3 : 1)
k3_index_sort(K3Seg* __restrict__ segs, uint32_t seg_cap, uint32_t* __restrict__ perm, uint32_t* __restrict__ tmp,
              DevStatus* __restrict__ st) {
    __shared__ uint32_t cnt[kIdxSub + 1];
    __shared__ uint32_t wbuf[NT / 32][kIdxWarpBuf];
    __shared__ uint32_t s_min, s_max, s_bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ns = (uint32_t)min(st->seg_count, (unsigned long long)seg_cap);
    for (uint32_t g = blockIdx.x; g < ns; g += gridDim.x) {
        const K3Seg sg = segs[g];
        if (!(sg.flags & 1u) || sg.len > kIdxSortMax || sg.len < 2) {
            if (tid == 0 && sg.len >= 2) segs[g].pad = 1u;          // radix pass
            continue;
        }
        const uint32_t len = (uint32_t)sg.len;
        uint32_t* pv = perm + sg.out;
        uint32_t* tv = tmp + sg.out;
        if (tid == 0) {
            s_min = 0xffffffffu;
            s_max = 0u;
            s_bad = 0u;
        }
        __syncthreads();
        uint32_t lmin = 0xffffffffu, lmax = 0u;
        for_each_u32<NT>(pv, len, [&](uint32_t, uint32_t v) {
            lmin = min(lmin, v);
            lmax = max(lmax, v);
        });
        lmin = __reduce_min_sync(0xffffffffu, lmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        if (lane == 0) {
            atomicMin(&s_min, lmin);
            atomicMax(&s_max, lmax);
        }
        uint32_t nsb = 1;
        while (nsb < kIdxSub && nsb * 32u < len) nsb <<= 1;
        for (uint32_t j = tid; j <= nsb; j += NT) cnt[j] = 0u;
        __syncthreads();
        const uint32_t vmin = s_min;
        const uint64_t range = (uint64_t)s_max - vmin + 1;
        uint32_t sh = 0;
        while ((range - 1) >> sh >= nsb) ++sh;
        for_each_u32<NT>(pv, len, [&](uint32_t, uint32_t v) { atomicAdd(&cnt[(v - vmin) >> sh], 1u); });
        __syncthreads();
        if (warp == 0) {                               // exclusive scan of nsb (<= 4096) counts
            const uint32_t per = (nsb + 31) / 32;
            const uint32_t j0 = min(nsb, lane * per), j1 = min(nsb, j0 + per);
            uint32_t loc = 0;
            for (uint32_t j = j0; j < j1; ++j) loc += cnt[j];
            uint32_t x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            uint32_t run = x - loc;
            for (uint32_t j = j0; j < j1; ++j) {
                const uint32_t c = cnt[j];
                cnt[j] = run;
                run += c;
            }
            if (lane == 31) cnt[nsb] = run;
        }
        __syncthreads();
        // scatter into sub-bucket order; afterwards cnt[j] = end of sub-bucket j
        for_each_u32<NT>(pv, len, [&](uint32_t, uint32_t v) { tv[atomicAdd(&cnt[(v - vmin) >> sh], 1u)] = v; });
        __syncthreads();
        for (uint32_t j = warp; j < nsb; j += NT / 32) {
            const uint32_t b = j ? cnt[j - 1] : 0u, e = cnt[j], sz = e - b;
            if (sz <= 32) {
                const uint32_t v = lane < sz ? tv[b + lane] : 0xffffffffu;
                uint32_t r = 0;
#pragma unroll
                for (int k = 0; k < 32; ++k) r += __shfl_sync(0xffffffffu, v, k) < v ? 1u : 0u;
                if (lane < sz) pv[b + r] = v;
            } else if (sz <= kIdxWarpBuf) {
                for (uint32_t k = lane; k < sz; k += 32) wbuf[warp][k] = tv[b + k];
                __syncwarp();
                for (uint32_t k = lane; k < sz; k += 32) {
                    const uint32_t v = wbuf[warp][k];
                    uint32_t r = 0;
                    for (uint32_t q = 0; q < sz; ++q) r += wbuf[warp][q] < v ? 1u : 0u;
                    pv[b + r] = v;
                }
                __syncwarp();
            } else if (lane == 0) {
                s_bad = 1u;
            }
        }
        __syncthreads();
        if (s_bad) {                                   // a clustered index set: radix pass
            for (uint32_t i = tid; i < len; i += NT) pv[i] = tv[i];   // (any order; re-sorted)
            if (tid == 0) segs[g].pad = 1u;
        } else {
            uint32_t viol = 0;                         // reading A14: strictly ascending indices
            for_each_u32<NT>(pv, len, [&](uint32_t i, uint32_t v) {
                if (i) viol += pv[i - 1] < v ? 0u : 1u;     // (the predecessor: L1-resident)
            });
            viol = __reduce_add_sync(0xffffffffu, viol);
            if (lane == 0 && viol) atomicAdd(&st->violations, (unsigned long long)viol);
            if (tid == 0) segs[g].pad = 0u;
        }
        __syncthreads();
    }
}

// K5 over the item and segment lists: the key before each item / segment start must not follow
// the key at it (the coarse-bucket starts are checked by k5_boundary_verify).
template <typename KeyT, bool PERM>
__global__ void k5_item_verify(const K3Item* __restrict__ items, const K3Seg* __restrict__ segs,
                               const KeyT* __restrict__ out_keys, const uint32_t* __restrict__ out_perm,
                               DevStatus* __restrict__ st, uint32_t item_cap, uint32_t seg_cap, uint64_t n) {
    const uint64_t ni = min((unsigned long long)item_cap, st->item_count);
    const uint64_t ns = min((unsigned long long)seg_cap, st->seg_count);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ni + ns;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = i < ni ? items[i].out : segs[i - ni].out;
        if (s == 0 || s >= n) continue;
        const auto a = KeyTraits<KeyT>::to_ord(out_keys[s - 1]);
        const auto b = KeyTraits<KeyT>::to_ord(out_keys[s]);
        const bool ok = PERM ? (a < b || (a == b && out_perm[s - 1] < out_perm[s])) : (a <= b);
        if (!ok) atomicAdd(&st->violations, 1ull);
    }
}

// K5 in one launch: every recorded coarse-bucket / K4-run start (range_start, the work of
// k5_boundary_verify) and every item / segment start (k5_item_verify), grid-stride.
template <typename KeyT, bool PERM>
__global__ void k5_verify_all(const unsigned long long* __restrict__ range_start, uint64_t nranges,
                              const K3Item* __restrict__ items, const K3Seg* __restrict__ segs,
                              const KeyT* __restrict__ out_keys, const uint32_t* __restrict__ out_perm,
                              DevStatus* __restrict__ st, uint32_t item_cap, uint32_t seg_cap, uint64_t n) {
    const uint64_t ni = min((unsigned long long)item_cap, st->item_count);
    const uint64_t ns = min((unsigned long long)seg_cap, st->seg_count);
    bool bad = false;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nranges + ni + ns;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = i < nranges ? range_start[i]
                                     : (i < nranges + ni ? items[i - nranges].out : segs[i - nranges - ni].out);
        if (s == ~0ull || s == 0 || s >= n) continue;
        const auto a = KeyTraits<KeyT>::to_ord(out_keys[s - 1]);
        const auto b = KeyTraits<KeyT>::to_ord(out_keys[s]);
        bad |= PERM ? !(a < b || (a == b && out_perm[s - 1] < out_perm[s])) : (b < a);
    }
    if (bad) atomicAdd(&st->violations, 1ull);
}

}  // namespace mlsort
