// k0_sample.cuh -- K0: region sizes from a sample of the predicted coarse buckets.
//
// K1 stores each coarse bucket contiguously in its own region ("put into their
// corresponding estimate ranking buckets").  For large inputs a fixed region of kRegionFactor x
// the average bucket wastes memory and still overflows on skewed data (the lognormal C3), which
// costs a second K1 pass.  K0 predicts every S-th key with the same network (Eq. 3, l.65),
// counts the coarse buckets of that sample, and lays the regions out with the expected size
// S k_c plus a 6-sigma binomial margin 6 S sqrt(k_c + 1) + 64.  The sum is bounded by
// n + 6 sqrt(S C (n + S C)) + 72 C (Cauchy-Schwarz), which is how the workspace is sized; a
// region that still overflows sends the call to the exact-layout retry as before.
#pragma once

#include "common.cuh"
#include "predict.cuh"
#include "k1_partition.cuh"

namespace mlsort {

template <typename KeyT, int MPAD>
__global__ void __launch_bounds__(256)
k0_sample(const KeyT* __restrict__ keys, uint64_t n, uint64_t stride, FoldedWeights fw, K1Params p,
          uint32_t* __restrict__ est) {
    extern __shared__ uint32_t h[];          // [C] sampled coarse counts of this CTA
    const uint32_t C = p.num_coarse;
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) h[c] = 0u;
    __syncthreads();
    constexpr int G = 8;
    const uint64_t ns = (n + stride - 1) / stride;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t s0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s0 < ns; s0 += step * G) {
        float u[G], ul[G];
        int32_t y[G];
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const uint64_t s = s0 + (uint64_t)q * step;
            KeyT x = s < ns ? keys[s * stride] : (KeyT)p.lo_d;
            if (!KeyTraits<KeyT>::finite(x)) x = (KeyT)p.lo_d;
            key_to_u<KeyT>(x, p, u[q], ul[q]);
        }
        gvm_forward_dense<MPAD, kPredPacked, G>(fw, u, ul, y);
#pragma unroll
        for (int q = 0; q < G; ++q)
            if (s0 + (uint64_t)q * step < ns) atomicAdd(&h[bucket_of_fxp(y[q], p.bm) >> p.fine_bits], 1u);
    }
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x)
        if (h[c]) atomicAdd(&est[c], h[c]);
}

// One CTA: rbase[c] = exclusive prefix of the region capacities, rbase[C] = their sum (<= area;
// if the bound were ever exceeded the regions fall back to equal shares and K1's overflow
// check sends the call to the exact-layout retry).
static __global__ void __launch_bounds__(1024)
k0_regions(const uint32_t* __restrict__ est, uint32_t C, uint64_t stride, unsigned long long area,
           unsigned long long* __restrict__ rbase) {
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (C + 1023) / 1024;
    const uint32_t c0 = min(C, (uint32_t)tid * per), c1 = min(C, c0 + per);
    auto capc = [&](uint32_t c) {
        const double k = (double)est[c];
        unsigned long long v = (unsigned long long)(k * (double)stride + 6.0 * (double)stride * sqrt(k + 1.0)) + 64ull;
        return (v + 7ull) & ~7ull;
    };
    unsigned long long loc = 0;
    for (uint32_t c = c0; c < c1; ++c) loc += capc(c);
    unsigned long long x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = wsum[lane], z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        wsum[lane] = z - w;
        if (lane == 31) total = z;
    }
    __syncthreads();
    unsigned long long run = wsum[warp] + x - loc;
    const bool fits = total <= area;
    const unsigned long long share = (area / max(C, 1u)) & ~7ull;
    for (uint32_t c = c0; c < c1; ++c) {
        rbase[c] = fits ? run : (unsigned long long)c * share;
        run += capc(c);
    }
    if (tid == 0) rbase[C] = fits ? total : (unsigned long long)C * share;
}

}  // namespace mlsort
