// k1_partition.cuh -- K1: fused predict + bucket + tile-local coarse partition.
//
// One CTA per tile of kTile consecutive keys (§2: "the estimation of ranking of
// each number is independent of each other", l.94).  Per key: u = x - lo; the GVM forward
// pass (Eq. 3) on the SFU/FMA pipes; the rank bucket b = round(y*B) (l.65); the coarse id
// c = b >> fine_bits.  Per tile: a shared-memory histogram over the C coarse ids, a block
// scan, an shared-memory scatter that partitions the tile by c, and one coalesced store
// of the partitioned tile (keys, fine bits b & (2^fine_bits - 1), and the input index for
// stable/perm sorts).  The tile's exclusive coarse offsets go to a column-major matrix
// M[c][t] (uint16) so that K3 can find coarse bucket c's piece in every tile; the column
// sums of M are the global coarse-bucket starts.
#pragma once

#include "common.cuh"
#include "predict.cuh"

namespace mlsort {

constexpr int kTile = 8192;                   // keys per K1 tile
constexpr int kKeysPerThread = kTile / kThreads;   // 16
constexpr int kGroup = 8;                      // keys evaluated together (ILP)

struct K1Params {
    double lo_d, hi_d;       // input_lo / input_hi of the weights (tail diagnostic, f64 u)
    float lo_f;              // input_lo rounded to f32 (f32 u = x - lo_f)
    BucketMap bm;
    uint32_t fine_bits;      // b = c * 2^fine_bits + fine
    uint32_t num_coarse;     // C
    uint32_t num_tiles;      // T
    uint64_t n;
};

template <typename KeyT> __device__ __forceinline__ float key_to_u(KeyT x, const K1Params& p);
template <> __device__ __forceinline__ float key_to_u<float>(float x, const K1Params& p) {
    return x - p.lo_f;
}
template <> __device__ __forceinline__ float key_to_u<double>(double x, const K1Params& p) {
    return (float)(x - p.lo_d);
}

// Dynamic shared memory: stage_key[kTile] KeyT | stage_idx[kTile] u32 (PERM) | hist[C] u32
//                        | stage_fine[kTile] u16 | scratch.
template <typename KeyT, bool PERM>
__host__ __device__ constexpr size_t k1_smem_bytes(uint32_t num_coarse) {
    return (size_t)num_coarse * 4 + (size_t)kTile * sizeof(KeyT) + (PERM ? (size_t)kTile * 4 : 0) +
           (size_t)kTile * 2 + 512;
}

// GIVEN = true is the multi-GPU receive side (mlsort_sort_records): the bucket travels with
// the key, so no prediction is repeated; bucket_in holds global buckets, b_lo is this rank's
// first bucket and idx_in the global input indices.
template <typename KeyT, int MPAD, int PRED, bool PERM, bool GIVEN = false>
__global__ void __launch_bounds__(kThreads, 2)
k1_predict_partition(const KeyT* __restrict__ keys, FoldedWeights fw, K1Params p,
                     KeyT* __restrict__ part_keys, uint16_t* __restrict__ part_fine,
                     uint32_t* __restrict__ part_idx, uint16_t* __restrict__ matrix,
                     DevStatus* __restrict__ st, const uint32_t* __restrict__ bucket_in = nullptr,
                     const uint32_t* __restrict__ idx_in = nullptr, uint32_t b_lo = 0) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t C = p.num_coarse;
    // layout: stage_key[kTile] KeyT | stage_idx[kTile] u32 (PERM) | hist[C] u32 | stage_fine[kTile] u16 | scratch
    KeyT* stage_key = reinterpret_cast<KeyT*>(smem);
    uint32_t* stage_idx = reinterpret_cast<uint32_t*>(smem + (size_t)kTile * sizeof(KeyT));
    uint32_t* hist = stage_idx + (PERM ? kTile : 0);
    uint16_t* stage_fine = reinterpret_cast<uint16_t*>(hist + C);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(stage_fine + kTile);

    const int tid = threadIdx.x;
    const uint32_t tile = blockIdx.x;
    const uint64_t base = (uint64_t)tile * kTile;
    const uint32_t cnt = (uint32_t)min((uint64_t)kTile, p.n - base);

    for (uint32_t i = tid; i < C; i += kThreads) hist[i] = 0;

    // ---- predict (Eq. 3) and bucket (l.65) for this thread's 16 keys, 8 at a time
    // b of every key is parked in shared memory (u32 view of the key staging area, which is
    // not live yet) so the predict loop below can stay rolled without local-memory arrays.
    uint32_t* sb = reinterpret_cast<uint32_t*>(stage_key);
    uint32_t tail_lo = 0, tail_hi = 0;
    if (GIVEN) {
#pragma unroll
        for (int k = 0; k < kKeysPerThread; ++k) {
            const uint32_t e = tid + kThreads * k;
            uint32_t b = e < cnt ? bucket_in[base + e] - b_lo : 0u;
            sb[e] = b < p.bm.Bm1 ? b : p.bm.Bm1;
        }
    }
#pragma unroll 1
    for (int g = 0; g < (GIVEN ? 0 : kKeysPerThread / kGroup); ++g) {
        float u[kGroup], y[kGroup];
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
            const uint32_t e = tid + kThreads * (g * kGroup + q);
            KeyT x = e < cnt ? keys[base + e] : (KeyT)p.lo_d;
            if (!KeyTraits<KeyT>::finite(x)) {
                atomicMin(&st->bad_index, (unsigned long long)(base + e));
                x = (KeyT)p.lo_d;
            }
            if (e < cnt) {
                tail_lo += (double)x < p.lo_d;
                tail_hi += (double)x > p.hi_d;
            }
            u[q] = key_to_u<KeyT>(x, p);
        }
        gvm_forward_f32<MPAD, PRED, kGroup>(fw, u, y);
#pragma unroll
        for (int q = 0; q < kGroup; ++q) sb[tid + kThreads * (g * kGroup + q)] = bucket_of(y[q], p.bm);
    }
    uint32_t bk[kKeysPerThread];
#pragma unroll
    for (int k = 0; k < kKeysPerThread; ++k) bk[k] = sb[tid + kThreads * k];   // own entries only
    __syncthreads();   // hist zeroed

    // ---- tile histogram over coarse ids
#pragma unroll
    for (int k = 0; k < kKeysPerThread; ++k) {
        const uint32_t e = tid + kThreads * k;
        if (e < cnt) atomicAdd(&hist[bk[k] >> p.fine_bits], 1u);
    }
    __syncthreads();

    // ---- exclusive scan of hist; write this tile's column of M (uint16, <= kTile)
    const uint32_t per = (C + kThreads - 1) / kThreads;
    const uint32_t c0 = min(C, tid * per), c1 = min(C, c0 + per);
    uint32_t local = 0;
    for (uint32_t c = c0; c < c1; ++c) local += hist[c];
    uint32_t total;
    uint32_t run = block_exclusive_scan<kThreads>(local, scratch, &total);
    for (uint32_t c = c0; c < c1; ++c) {
        uint32_t h = hist[c];
        hist[c] = run;
        matrix[(size_t)c * p.num_tiles + tile] = (uint16_t)run;
        run += h;
    }
    if (tid == 0) matrix[(size_t)C * p.num_tiles + tile] = (uint16_t)cnt;   // sentinel row
    __syncthreads();

    // ---- scatter into the shared staging area, partitioned by coarse id
    const uint32_t fmask = (1u << p.fine_bits) - 1u;
#pragma unroll
    for (int k = 0; k < kKeysPerThread; ++k) {
        const uint32_t e = tid + kThreads * k;
        if (e < cnt) {
            const uint32_t pos = atomicAdd(&hist[bk[k] >> p.fine_bits], 1u);
            stage_key[pos] = keys[base + e];            // L2-resident re-read
            stage_fine[pos] = (uint16_t)(bk[k] & fmask);
            if (PERM) stage_idx[pos] = GIVEN ? idx_in[base + e] : (uint32_t)(base + e);
        }
    }
    // tail counters (reduce while the scatter drains)
    uint32_t tl = block_reduce_sum<kThreads>(tail_lo, scratch);
    uint32_t th = block_reduce_sum<kThreads>(tail_hi, scratch + 64);
    if (tid == 0) {
        if (tl) atomicAdd(&st->tail_lo, (unsigned long long)tl);
        if (th) atomicAdd(&st->tail_hi, (unsigned long long)th);
    }
    __syncthreads();

    // ---- coalesced store of the partitioned tile
    for (uint32_t e = tid; e < cnt; e += kThreads) {
        part_keys[base + e] = stage_key[e];
        part_fine[base + e] = stage_fine[e];
        if (PERM) part_idx[base + e] = stage_idx[e];
    }
}

// Column sums of M: S[c] = sum_t M[c][t] = number of keys with coarse id < c, i.e. the
// global start of coarse bucket c (its length is S[c+1] - S[c]).  One CTA per row.
__global__ void __launch_bounds__(kThreads)
k2_coarse_starts(const uint16_t* __restrict__ matrix, uint32_t num_tiles,
                 unsigned long long* __restrict__ starts) {
    __shared__ unsigned long long wsum[kWarps];
    const uint32_t c = blockIdx.x;
    const uint16_t* row = matrix + (size_t)c * num_tiles;
    unsigned long long s = 0;
    for (uint32_t t = threadIdx.x; t < num_tiles; t += kThreads) s += row[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kWarps; ++w) t += wsum[w];
        starts[c] = t;
    }
}

}  // namespace mlsort
