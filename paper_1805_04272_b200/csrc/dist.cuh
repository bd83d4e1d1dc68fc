// dist.cuh -- multi-GPU send side: every rank predicts the GLOBAL rank
// bucket b of its keys (Eq. 3 + l.65 with the global B) and partitions its records by the
// owner rank floor(b*G/B), so rank g receives exactly the rank range [gB/G, (g+1)B/G)
// (BASELINE north_star).  Records of one destination stay in input order (stable), so after
// the all-to-all a receiver sees equal keys in increasing global index.
#pragma once

#include "common.cuh"
#include "predict.cuh"
#include "k1_partition.cuh"
#include "k4_overflow.cuh"

namespace mlsort {

constexpr uint32_t kMaxRanks = 64;

__device__ __forceinline__ uint32_t owner_of(uint32_t b, uint64_t B, uint32_t G) {
    return (uint32_t)(((uint64_t)b * G) / B);
}

// Ownership rule of one exchange.  Monotone model (Eq. 4): owner = floor(b*G/B), the rank
// range of BJ:5.  A model that fails Eq. 4 does not order the buckets, so its keys are routed
// by key value instead -- owner = clamp(floor((x - lo) G / (hi - lo)), 0, G-1), monotone in x
// by construction -- and each receiver sorts whatever buckets it gets (reading A14).
struct OwnerRule {
    uint64_t B;
    uint32_t G;
    uint32_t keyspace;      // 1: route by key value
    double lo, scale;       // keyspace: owner = floor((x - lo) * scale), scale = G / (hi - lo)
};

template <typename KeyT>
__device__ __forceinline__ uint32_t owner_rule(const OwnerRule& r, KeyT x, uint32_t b) {
    if (!r.keyspace) return owner_of(b, r.B, r.G);
    const double t = ((double)x - r.lo) * r.scale;
    if (!(t > 0.0)) return 0u;
    return t >= (double)(r.G - 1) ? r.G - 1 : (uint32_t)t;
}

template <typename KeyT, int MPAD, int PRED>
__global__ void __launch_bounds__(kRadixThreads)
k_dist_predict(const KeyT* __restrict__ keys, uint64_t n, FoldedWeights fw, K1Params p, OwnerRule orl,
               uint32_t nchunks, uint32_t* __restrict__ bucket_out, uint32_t* __restrict__ ghist,
               DevStatus* __restrict__ st) {
    __shared__ uint32_t h[kMaxRanks];
    __shared__ uint32_t scratch[128];
    const int tid = threadIdx.x;
    for (int i = tid; i < (int)kMaxRanks; i += kRadixThreads) h[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kRadixChunk;
    uint32_t tl = 0, th = 0;
    constexpr int G8 = 8;
    KeyT xs[G8];
#pragma unroll 1
    for (int g = 0; g < kRadixItems / G8; ++g) {
        float u[G8], ul[G8];
        int32_t y[G8];
#pragma unroll
        for (int q = 0; q < G8; ++q) {
            const uint64_t e = base + tid + (uint64_t)kRadixThreads * (g * G8 + q);
            KeyT x = e < n ? keys[e] : (KeyT)p.lo_d;
            if (!KeyTraits<KeyT>::finite(x)) {
                atomicMin(&st->bad_index, (unsigned long long)e);
                x = (KeyT)p.lo_d;
            }
            if (e < n) {
                tl += (double)x < p.lo_d;
                th += (double)x > p.hi_d;
            }
            xs[q] = x;
            key_to_u<KeyT>(x, p, u[q], ul[q]);
        }
        gvm_forward_dense<MPAD, PRED, G8>(fw, u, ul, y);
#pragma unroll
        for (int q = 0; q < G8; ++q) {
            const uint64_t e = base + tid + (uint64_t)kRadixThreads * (g * G8 + q);
            if (e < n) {
                const uint32_t b = bucket_of_fxp(y[q], p.bm);
                bucket_out[e] = b;
                atomicAdd(&h[owner_rule<KeyT>(orl, xs[q], b)], 1u);
            }
        }
    }
    tl = block_reduce_sum<kRadixThreads>(tl, scratch);
    th = block_reduce_sum<kRadixThreads>(th, scratch + 64);
    __syncthreads();
    if (tid == 0) {
        if (tl) atomicAdd(&st->tail_lo, (unsigned long long)tl);
        if (th) atomicAdd(&st->tail_hi, (unsigned long long)th);
    }
    for (uint32_t d = tid; d < orl.G; d += kRadixThreads) ghist[(size_t)d * nchunks + blockIdx.x] = h[d];
}

// stable scatter by owner (warp w owns elements [w*512, (w+1)*512) of the chunk, lane order)
template <typename KeyT>
__global__ void __launch_bounds__(kRadixThreads)
k_dist_scatter(const KeyT* __restrict__ keys, const uint32_t* __restrict__ bucket, uint64_t n, uint64_t gofs,
               OwnerRule orl, uint32_t nchunks, const uint32_t* __restrict__ ghist,
               KeyT* __restrict__ rkeys, uint32_t* __restrict__ rbucket, uint32_t* __restrict__ ridx) {
    constexpr int W = kRadixThreads / 32;
    __shared__ uint16_t wcnt[W][kMaxRanks];
    __shared__ uint32_t goff[kMaxRanks];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < W * (int)kMaxRanks; i += kRadixThreads) (&wcnt[0][0])[i] = 0;
    const uint32_t G = orl.G;
    for (uint32_t d = threadIdx.x; d < G; d += kRadixThreads) goff[d] = ghist[(size_t)d * nchunks + blockIdx.x];
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kRadixChunk + (uint64_t)warp * 32 * kRadixItems;
    uint32_t rank[kRadixItems], dig[kRadixItems];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t e = base + (uint64_t)r * 32 + lane;
        const bool ok = e < n;
        dig[r] = ok ? owner_rule<KeyT>(orl, keys[e], bucket[e]) : kMaxRanks + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
        const uint32_t before = ok ? wcnt[warp][dig[r]] : 0u;
        rank[r] = before + __popc(peers & lt);
        __syncwarp();
        if (ok && (peers & lt) == 0) wcnt[warp][dig[r]] = (uint16_t)(before + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < G; d += kRadixThreads) {
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
            rkeys[dst] = keys[e];
            rbucket[dst] = bucket[e];
            if (ridx) ridx[dst] = (uint32_t)(gofs + e);
        }
    }
}

template <typename KeyT>
int dist_partition(const KeyT* keys, uint64_t n, uint64_t gofs, const OwnerRule& orl, uint32_t mpad, int pred,
                   const FoldedWeights& fw, const K1Params& kp, KeyT* rkeys, uint32_t* rbucket, uint32_t* ridx,
                   uint32_t* bucket_tmp, uint32_t* ghist, DevStatus* st, uint64_t* h_counts, cudaStream_t s) {
    const uint32_t nchunks = (uint32_t)((n + kRadixChunk - 1) / kRadixChunk);
    const uint32_t G = orl.G;
#define DCASE(M)                                                                                          \
    if (mpad == M) {                                                                                      \
        if (pred == kPredMufu)                                                                            \
            k_dist_predict<KeyT, M, kPredMufu><<<nchunks, kRadixThreads, 0, s>>>(keys, n, fw, kp, orl, nchunks, \
                                                                                  bucket_tmp, ghist, st); \
        else if (pred == kPredMixed)                                                                      \
            k_dist_predict<KeyT, M, kPredMixed><<<nchunks, kRadixThreads, 0, s>>>(keys, n, fw, kp, orl, nchunks, \
                                                                                   bucket_tmp, ghist, st); \
        else                                                                                              \
            k_dist_predict<KeyT, M, kPredPacked><<<nchunks, kRadixThreads, 0, s>>>(keys, n, fw, kp, orl, nchunks, \
                                                                                    bucket_tmp, ghist, st); \
    }
    DCASE(16) DCASE(32) DCASE(64)
#undef DCASE
    if (cudaGetLastError() != cudaSuccess) return MLSORT_ERR_CUDA;
    // per-destination totals (before the scan): column sums of ghist
    std::vector<uint32_t> h((size_t)G * nchunks);
    if (cudaMemcpyAsync(h.data(), ghist, h.size() * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return MLSORT_ERR_CUDA;
    k_radix_scan<<<1, 1024, 0, s>>>(ghist, (uint64_t)G * nchunks);
    k_dist_scatter<KeyT><<<nchunks, kRadixThreads, 0, s>>>(keys, bucket_tmp, n, gofs, orl, nchunks, ghist, rkeys,
                                                            rbucket, ridx);
    if (cudaGetLastError() != cudaSuccess) return MLSORT_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return MLSORT_ERR_CUDA;
    for (uint32_t g = 0; g < G; ++g) {
        uint64_t t = 0;
        for (uint32_t c = 0; c < nchunks; ++c) t += h[(size_t)g * nchunks + c];
        h_counts[g] = t;
    }
    return MLSORT_OK;
}

}  // namespace mlsort
