// selftest.cuh -- exhaustive on-device monotonicity sweeps of the predictor's primitives
// (reading A14; SURVEY.md §8(c) "predictor y (GPU side)": K8).
//
// PAPER.md Eq. 4 (l.76-84) makes the network monotone in exact arithmetic; the f32 predictor
// (predict.cuh) is monotone too if every primitive it composes is: FFMA/FADD with round-to-
// nearest are monotone in each operand (IEEE), the fixed-point sum is exact, so what remains
// to be shown are the approximate instructions -- MUFU.EX2 (ex2.approx.ftz.f32), MUFU.RCP
// (rcp.approx.ftz.f32, MUFU/MIXED predictors) -- and the packed FMA-pipe reciprocal chain.
// Each sweep below evaluates one of them on EVERY input of its domain in ascending order and
// counts the adjacent pairs whose outputs go the wrong way.  The sort does not depend on the
// result for correctness (K3/K5 verify every adjacent pair), only on speed.
#pragma once

#include <cstdint>
#include "predict.cuh"

namespace mlsort {

enum {
    kSweepEx2 = 0,          // ex2.approx.ftz.f32 over all non-NaN f32: non-decreasing
    kSweepRcpChain = 1,     // packed chain -1/d over every f32 d in [1, 2^61]: r non-increasing
    kSweepRcpMufu = 2,      // rcp.approx.ftz.f32 over every positive f32: non-increasing
    kSweepLogistic = 3,     // packed-predictor term r(1 + ex2(min(a, 60))) over all non-NaN a
};

struct SweepOut {
    unsigned long long descents;    // adjacent inputs whose outputs go the wrong way
    unsigned long long evaluated;   // inputs evaluated
    unsigned int max_rel_err_bits;  // kSweepRcpChain: max |r d - 1| (f32 bits, >= 0)
    unsigned int pad;
};

// input number o of the sweep's ascending sequence -> f32 bits
__device__ __forceinline__ uint32_t sweep_bits(int what, uint64_t o) {
    if (what == kSweepRcpChain) return 0x3F800000u + (uint32_t)o;          // 1 .. 2^61
    if (what == kSweepRcpMufu) return 1u + (uint32_t)o;                    // +denormal_min .. FLT_MAX
    const uint32_t ob = (uint32_t)o;                                       // order-preserving index
    return (ob & 0x80000000u) ? (ob & 0x7fffffffu) : ~ob;
}

__device__ __forceinline__ uint64_t sweep_count(int what) {
    if (what == kSweepRcpChain) return 0x5E000000ull - 0x3F800000ull + 1ull;
    if (what == kSweepRcpMufu) return 0x7F7FFFFFull;
    return 1ull << 32;
}

// value whose sequence must be NON-DECREASING along the sweep (decreasing primitives negated)
__device__ __forceinline__ float sweep_eval(int what, float x, f32x2 k1_2, f32x2 one2, float& rel) {
    rel = 0.0f;
    if (what == kSweepEx2) return ex2_approx(x);
    if (what == kSweepRcpMufu) return -rcp_approx(x);
    float d = x;
    if (what == kSweepLogistic) d = ex2_approx(fminf(x, kAClamp)) + 1.0f;
    const f32x2 nr2 = neg_rcp_packed(pk2(d, d), k1_2, one2);
    float nr, nr_b;
    upk2(nr2, nr, nr_b);
    if (what == kSweepRcpChain) rel = (float)fabs(-(double)nr * (double)d - 1.0);
    return nr;          // -r: non-decreasing when r is non-increasing
}

// one thread per chunk of kSweepChunk consecutive inputs (+ the first input of the next chunk)
constexpr uint32_t kSweepChunk = 2048;

static __global__ void __launch_bounds__(256)
k_sweep_monotone(int what, f32x2 k1_2, f32x2 one2, SweepOut* out) {
    const uint64_t total = sweep_count(what);
    const uint64_t nchunks = (total + kSweepChunk - 1) / kSweepChunk;
    unsigned long long desc = 0, evals = 0;
    float maxrel = 0.0f;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o0 = c * kSweepChunk;
        const uint64_t o1 = min(total, o0 + kSweepChunk + 1);     // overlap one input with the next chunk
        bool have = false;
        float prev = 0.0f;
        for (uint64_t o = o0; o < o1; ++o) {
            const float x = __uint_as_float(sweep_bits(what, o));
            if (x != x) continue;                                   // NaN inputs are not in the domain
            float rel;
            const float v = sweep_eval(what, x, k1_2, one2, rel);
            if (o < o0 + kSweepChunk) {
                ++evals;
                maxrel = fmaxf(maxrel, rel);
            }
            if (have && v < prev) ++desc;
            prev = v;
            have = true;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        desc += __shfl_down_sync(0xffffffffu, desc, o);
        evals += __shfl_down_sync(0xffffffffu, evals, o);
        maxrel = fmaxf(maxrel, __shfl_down_sync(0xffffffffu, maxrel, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (desc) atomicAdd(&out->descents, desc);
        atomicAdd(&out->evaluated, evals);
        atomicMax(&out->max_rel_err_bits, __float_as_uint(maxrel));
    }
}

}  // namespace mlsort
