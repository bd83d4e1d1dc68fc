// predict.cuh -- the GVM forward pass (§2 Eq. 3, l.73-76) in f32 on the SFU/FMA
// pipes, and the rank-bucket map r = round(y*B) (l.65).
//
// Folding: with u = x - lo and
// x^ = 2u/(hi-lo) - 1, the logistic argument satisfies
//     exp(-t_j) = 2^(A_j*u + C_j),   A_j = -2 beta_j w1_j log2(e)/(hi-lo),
//                                    C_j =  beta_j (w1_j + b_j) log2(e),
// so one activation is  a = FFMA(A_j, u, C_j); e = ex2(a); d = 1 + e; r = 1/d;
// y = FFMA(w2_j, r, y).  u is formed in the key's own precision (an f64 subtract for
// f64 keys) and then rounded to f32, so y depends on x only through a monotone map.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mlsort {

constexpr int kMaxM = 64;

// Passed by value: lives in the kernel-parameter constant bank, so every FFMA reads its
// weight operand straight from constant memory (warp-uniform, no LDS).
struct FoldedWeights {
    float A[kMaxM];
    float C[kMaxM];
    float W[kMaxM];
};

struct BucketMap {
    float Bf;          // (float)B
    uint32_t Bm1;      // B - 1
};

__device__ __forceinline__ float ex2_approx(float a) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a));
    return e;
}
__device__ __forceinline__ float rcp_approx(float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return r;
}
// Reciprocal on the FMA pipe for d in [1, 2^61]: bit-trick seed (|rel err| < 0.125)
// and three Newton steps r <- r + r(1 - d r) (error squares each step, < 1e-7 after 3).
__device__ __forceinline__ float rcp_newton(float d) {
    float r = __int_as_float(0x7EF311C3 - __float_as_int(d));
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    return r;
}

enum { kPredMufu = 1, kPredMixed = 2 };

// Evaluate Eq. 3 for KG keys at once (independent chains give the SFU/FMA pipes ILP).
// MPAD is the padded neuron count (pad neurons have W = 0).  PRED selects the reciprocal
// formulation; in kPredMixed one neuron in four uses MUFU.RCP and three use the Newton
// reciprocal, balancing MUFU (ex2) load against FMA-pipe issue.
template <int MPAD, int PRED, int KG>
__device__ __forceinline__ void gvm_forward_f32(const FoldedWeights& fw, const float (&u)[KG],
                                                float (&y)[KG]) {
#pragma unroll
    for (int q = 0; q < KG; ++q) y[q] = 0.0f;
#pragma unroll
    for (int j = 0; j < MPAD; ++j) {
        const float A = fw.A[j], C = fw.C[j], W = fw.W[j];
        const bool use_mufu_rcp = (PRED == kPredMufu) || ((j & 3) == 0);
#pragma unroll
        for (int q = 0; q < KG; ++q) {
            float a = fmaf(A, u[q], C);
            float r;
            if (use_mufu_rcp) {
                r = rcp_approx(1.0f + ex2_approx(a));
            } else {
                a = fminf(a, 60.0f);             // keeps d = 1 + 2^a inside Newton's range
                r = rcp_newton(1.0f + ex2_approx(a));
            }
            y[q] = fmaf(W, r, y[q]);
        }
    }
}

// r = clamp(round_half_up(y * B), 0, B - 1) (S:232, S:297-S:298).  For y >= 0
// round-half-up equals round-half-away-from-zero (reading A6); negative y saturate to 0.
__device__ __forceinline__ uint32_t bucket_of(float y, const BucketMap& bm) {
    uint32_t r = __float2uint_rd(fmaf(y, bm.Bf, 0.5f));
    return r < bm.Bm1 ? r : bm.Bm1;
}

}  // namespace mlsort
