// k3_sort.cuh -- K3: gather one coarse bucket from every tile, place its keys into their
// rank buckets and sort inside each bucket (§2 l.86: "N numbers are put into their
// corresponding estimate ranking buckets ... only the numbers inside each bucket need to
// be sorted").
//
// A thread-block cluster of R CTAs (distributed shared memory) owns one coarse bucket c.
// CTA r gathers the pieces of c from tiles [rT/R, (r+1)T/R) (warp-cooperative, coalesced
// within each piece) and routes every element by its fine bucket to the owner CTA
// fine >> owner_shift, reserving slots with warp-aggregated remote shared-memory atomics.
// After a cluster barrier each CTA holds the keys of a contiguous fine range: a shared
// memory counting sort by fine bucket (the paper's placement), a stable-by-index
// insertion sort inside each fine bucket (the paper's fix-up), an adjacent-pair check
// (reading A14) and a coalesced store to its slice of the output.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mlsort {

constexpr int kK3Threads = 1024;
constexpr int kK3Warps = kK3Threads / 32;
constexpr int kTileK3 = 8192;   // must equal kTile (K1)

struct K3Params {
    uint32_t num_tiles;     // T
    uint32_t num_coarse;    // C
    uint32_t owner_shift;   // owner = fine >> owner_shift
    uint32_t kr;            // fine buckets per owner CTA = 2^owner_shift
    uint32_t cap;           // receive capacity (elements) per CTA
    uint32_t pad;
};

template <typename KeyT, bool PERM>
struct K3Layout {
    using Bits = typename KeyTraits<KeyT>::Bits;
    // [ctrl 256B][recv_key cap][sorted_key cap][hist kr][recv_idx cap][sorted_idx cap][recv_fine cap]
    static __host__ __device__ size_t bytes(uint32_t cap, uint32_t kr) {
        return 256 + (size_t)cap * sizeof(Bits) * 2 + (size_t)kr * 4 + (PERM ? (size_t)cap * 8 : 0) +
               (size_t)cap * 2 + 16;
    }
    static __host__ __device__ size_t elem_bytes() { return sizeof(Bits) * 2 + 2 + (PERM ? 8 : 0); }
};

template <typename KeyT, bool PERM>
__device__ __forceinline__ bool precedes(typename KeyTraits<KeyT>::Bits ka, uint32_t ia,
                                         typename KeyTraits<KeyT>::Bits kb, uint32_t ib) {
    if (PERM) return ka < kb || (ka == kb && ia < ib);
    return ka < kb;
}

template <typename KeyT, bool PERM, int R>
__global__ void __launch_bounds__(kK3Threads, 1)
k3_cluster_sort(K3Params p, const KeyT* __restrict__ part_keys, const uint16_t* __restrict__ part_fine,
                const uint32_t* __restrict__ part_idx, const uint16_t* __restrict__ matrix,
                const unsigned long long* __restrict__ starts, KeyT* __restrict__ out_keys,
                uint32_t* __restrict__ out_perm, unsigned long long* __restrict__ range_start,
                DevStatus* __restrict__ st, uint32_t* __restrict__ big_list) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* ctrl = reinterpret_cast<uint32_t*>(smem);            // [0] recv count
    uint32_t* scratch = ctrl + 16;
    Bits* recv_key = reinterpret_cast<Bits*>(smem + 256);
    Bits* sorted_key = recv_key + p.cap;
    uint32_t* hist = reinterpret_cast<uint32_t*>(sorted_key + p.cap);
    uint32_t* recv_idx = hist + p.kr;
    uint32_t* sorted_idx = recv_idx + (PERM ? p.cap : 0);
    uint16_t* recv_fine = reinterpret_cast<uint16_t*>(sorted_idx + (PERM ? p.cap : 0));

    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank();
    const uint32_t c = blockIdx.x / R;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const unsigned long long S0 = starts[c], S1 = starts[c + 1];
    const unsigned long long n_c = S1 - S0;
    if (n_c == 0) return;                                       // uniform across the cluster
    if (n_c > (unsigned long long)R * p.cap) {                  // overflow path (K4)
        if (r == 0 && tid == 0) {
            unsigned long long k = atomicAdd(&st->big_count, 1ull);
            big_list[k] = c;
            atomicAdd(&st->big_elems, n_c);
            atomicMax(&st->max_coarse, n_c);
        }
        return;
    }
    if (tid == 0) ctrl[0] = 0;
    cluster.sync();

    // ---------------- phase A: gather pieces of c from this CTA's tiles, route by owner
    const uint32_t T = p.num_tiles;
    const uint32_t t0 = (uint32_t)(((unsigned long long)r * T) / R);
    const uint32_t t1 = (uint32_t)(((unsigned long long)(r + 1) * T) / R);
    const uint16_t* colc = matrix + (size_t)c * T;
    const uint16_t* colc1 = matrix + (size_t)(c + 1) * T;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (uint32_t tb = t0 + warp * 32; tb < t1; tb += kK3Warps * 32) {
        const uint32_t t = tb + lane;
        uint32_t off = 0, len = 0;
        if (t < t1) {
            off = colc[t];
            len = (uint32_t)colc1[t] - off;
        }
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - len;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t b0 = 0; b0 < total; b0 += 32) {
            const uint32_t i = b0 + lane;
            // piece of element i: the largest lane l with excl_l <= i
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int cand = lo + step;
                const uint32_t v = __shfl_sync(0xffffffffu, excl, cand & 31);
                if (cand < 32 && v <= i) lo = cand;
            }
            const uint32_t poff = __shfl_sync(0xffffffffu, off, lo);
            const uint32_t pexc = __shfl_sync(0xffffffffu, excl, lo);
            const bool active = i < total;
            const unsigned amask = __ballot_sync(0xffffffffu, active);
            if (active) {
                const size_t src = (size_t)(tb + lo) * kTileK3 + poff + (i - pexc);
                const KeyT key = part_keys[src];
                const uint32_t fine = part_fine[src];
                const uint32_t idx = PERM ? part_idx[src] : 0u;
                const uint32_t owner = fine >> p.owner_shift;
                const unsigned peers = __match_any_sync(amask, owner);
                const int leader = __ffs(peers) - 1;
                uint32_t basepos = 0;
                uint32_t* rctrl = cluster.map_shared_rank(ctrl, (int)owner);
                if (lane == leader) basepos = atomicAdd(rctrl, (uint32_t)__popc(peers));
                basepos = __shfl_sync(peers, basepos, leader);
                const uint32_t slot = basepos + __popc(peers & lt_mask);
                if (slot < p.cap) {
                    cluster.map_shared_rank(recv_key, (int)owner)[slot] = KeyTraits<KeyT>::to_ord(key);
                    cluster.map_shared_rank(recv_fine, (int)owner)[slot] =
                        (uint16_t)(fine & (p.kr - 1u));
                    if (PERM) cluster.map_shared_rank(recv_idx, (int)owner)[slot] = idx;
                }
            }
        }
    }
    cluster.sync();

    // counts of every owner (remote reads), then a barrier so no CTA exits while others read
    uint32_t my_off = 0, cnt = 0;
    bool overflow = false;
    for (int o = 0; o < R; ++o) {
        const uint32_t co = *cluster.map_shared_rank(ctrl, o);
        overflow |= co > p.cap;
        if (o < r) my_off += co;
        if (o == r) cnt = co;
    }
    cluster.sync();
    if (overflow) {   // a skewed fine range overflowed one owner: whole bucket -> K4
        if (r == 0 && tid == 0) {
            unsigned long long k = atomicAdd(&st->big_count, 1ull);
            big_list[k] = c;
            atomicAdd(&st->big_elems, n_c);
            atomicMax(&st->max_coarse, n_c);
        }
        return;
    }
    if (r == 0 && tid == 0) atomicMax(&st->max_coarse, n_c);

    // ---------------- phase B: counting sort by fine bucket (placement)
    for (uint32_t f = tid; f < p.kr; f += kK3Threads) hist[f] = 0;
    __syncthreads();
    for (uint32_t e = tid; e < cnt; e += kK3Threads) atomicAdd(&hist[recv_fine[e]], 1u);
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
    for (uint32_t e = tid; e < cnt; e += kK3Threads) {
        const uint32_t pos = atomicAdd(&hist[recv_fine[e]], 1u);
        sorted_key[pos] = recv_key[e];
        if (PERM) sorted_idx[pos] = recv_idx[e];
    }
    __syncthreads();

    // ---------------- per-bucket fix-up: insertion sort by (key, index) (A9, A10)
    for (uint32_t f = tid; f < p.kr; f += kK3Threads) {
        const uint32_t s = f ? hist[f - 1] : 0u, e = hist[f];
        for (uint32_t i = s + 1; i < e; ++i) {
            const Bits kv = sorted_key[i];
            const uint32_t iv = PERM ? sorted_idx[i] : 0u;
            uint32_t j = i;
            while (j > s && precedes<KeyT, PERM>(kv, iv, sorted_key[j - 1], PERM ? sorted_idx[j - 1] : 0u)) {
                sorted_key[j] = sorted_key[j - 1];
                if (PERM) sorted_idx[j] = sorted_idx[j - 1];
                --j;
            }
            sorted_key[j] = kv;
            if (PERM) sorted_idx[j] = iv;
        }
    }
    __syncthreads();

    // ---------------- verify adjacent pairs inside this slice (reading A14)
    uint32_t viol = 0;
    for (uint32_t e = tid + 1; e < cnt; e += kK3Threads) {
        const Bits a = sorted_key[e - 1], b = sorted_key[e];
        const bool ok = PERM ? precedes<KeyT, true>(a, sorted_idx[e - 1], b, sorted_idx[e]) : (a <= b);
        viol += ok ? 0u : 1u;
    }
    viol = block_reduce_sum<kK3Threads>(viol, scratch);
    if (tid == 0 && viol) atomicAdd(&st->violations, (unsigned long long)viol);

    // ---------------- coalesced store of the slice
    const unsigned long long dst = S0 + my_off;
    if (tid == 0) range_start[(size_t)c * R + r] = cnt ? dst : ~0ull;
    for (uint32_t e = tid; e < cnt; e += kK3Threads) {
        out_keys[dst + e] = KeyTraits<KeyT>::from_ord(sorted_key[e]);
        if (PERM) out_perm[dst + e] = sorted_idx[e];
    }
}

}  // namespace mlsort
