// predict.cuh -- the GVM forward pass (§2 Eq. 3, l.73-76) in f32 on the SFU/FMA
// pipes, and the rank-bucket map r = round(y*B) (l.65).
//
// Folding: with u = x - x0 and
// x^ = 2(u + x0 - lo)/(hi-lo) - 1, the logistic argument satisfies
//     exp(-t_j) = 2^(A_j*u + C_j),   A_j = -2 beta_j w1_j log2(e)/(hi-lo),
//                                    C_j =  beta_j (w1_j + b_j) log2(e) + A_j (x0 - lo),
// so one activation is  a = FFMA(A_j, u, C_j); e = ex2(a); d = 1 + e; r = 1/d; then the
// w2_j-weighted term is accumulated.  The origin x0 is 0 for f32 keys whose range is near 0
// (then u = x exactly and no key resolution is lost to a subtraction), else input_lo.  f64 keys
// form u in f64 and round it once to f32, so y depends on x only through the monotone map
// x -> fl32(x - x0) (k1_partition.cuh key_to_u).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mlsort {

constexpr int kMaxM = 64;

// Passed by value: lives in the kernel-parameter constant bank, so every FFMA reads its
// weight operand straight from constant memory (warp-uniform, no LDS).
struct __align__(16) FoldedWeights {
    // (c, c) pairs of the packed predictor's constants, read from the parameter bank (uniform
    // registers) instead of occupying vector register pairs: 1, k1, 1.5*2^23, 2^-kAShift.
    // The hot members come first: the whole struct is a kernel parameter and only the first
    // 4 KB of the parameter bank are addressed directly by the instructions that read them.
    unsigned long long one2, k1_2, magic2, dofs2;
    float A[kMaxM];
    // packed predictor, exponent-shifted (see kAShift): Cs_j = C_j - kAShift, Wns_j = -W_j 2^-kAShift
    float Cs[kMaxM];
    float Wns[kMaxM];
    // Per-pair lower clamp of the packed predictor (pair_clamp != 0; DESIGN.md "K1 per-pair
    // clamp"): for models whose neurons all have A_j < 0 the host orders the neurons by their left
    // saturation bound and checks, for every pair p, that L_p = max_j (119 - Cs_j)/A_j (every
    // argument <= 119 for u >= L_p) lies below both neurons' left saturation bound (a_j >= 24.5,
    // where the computed term is the exact constant 0).  Then u_p = max(u, L_p) changes no term
    // and no argument can overflow the reciprocal chain: one FMNMX per pair and key instead of one
    // per activation.
    float Lp[kMaxM / 2];
    uint32_t pair_clamp;
    // u in [u_safe_lo, u_safe_hi] keeps every shifted argument A_j u + Cs_j <= kAClamp, so the
    // packed predictor may skip its per-activation clamp for such keys (CLAMP = false).  When
    // u_cl_lo/hi are finite, keys clamp u into [u_cl_lo, u_cl_hi] (K1Params), every argument
    // there is <= kANoClamp and u_safe spans everything.
    float u_safe_lo, u_safe_hi, u_cl_lo, u_cl_hi;
    // Saturated-pair skipping.  Neurons are stored sorted by
    // centre.  For u < lo2[p] both neurons of pair p have a > 24.5 or a < -26.5 on their left
    // side, and for u > hi2[p] on their right side; there the computed fixed-point terms are
    // EXACT constants (a >= 24: |W r| < 1/4 rounds to 0; a <= -26: 1 + 2^a rounds to 1, so the
    // reciprocal chain returns its value at d = 1), whose float bits are tl2[p] / tr2[p].
    float lo2[kMaxM / 2], hi2[kMaxM / 2];
    uint32_t tl2[kMaxM / 2], tr2[kMaxM / 2];
    float C[kMaxM];
    float W[kMaxM];    // w2_j * 2^S (fixed-point accumulation scale, see below)
    float Wn[kMaxM];   // -W_j
    // class of a key for the value grouping in k1_ws: lut[ordered_bits(u) >> 21], 64 classes
    unsigned char lut[2048];
};

struct BucketMap {
    float Bf;          // (float)B
    uint32_t Bm1;      // B - 1
    unsigned long long B;
    uint32_t S;        // y = acc * 2^-S
    uint32_t pow2;     // B = 2^k: the bucket is a shift of acc (sh = S - k, half = 2^(sh-1) or 0)
    int32_t sh, half;
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

// kPredSkip: the packed arithmetic with saturated-pair skipping (bit-identical to kPredPacked;
// k1_ws runs it on value-grouped tiles)
enum { kPredMufu = 1, kPredMixed = 2, kPredPacked = 3, kPredSkip = 4 };

// ---- packed-pair (f32x2) formulation --------------------
// Blackwell's FFMA2/FMUL2 evaluate two neurons per instruction; their B operand can be a
// uniform register, so neuron constants are read as (A_j, A_j+1) pairs straight from the
// kernel-parameter bank.  The reciprocal 1/d, d = 1 + 2^a in [1, 2^61], is computed on the FMA
// pipe as
//     r0 = bits trick  (0x7EF33400 - bits(d); the chain carries -r, whose bits are
//                       0xFEF33400 - bits(d), so no negation is ever issued)
//     r1 = r0 (k1 - d r0)               k1 = 2.001281198  (modified Newton step, |rel| <= 1.3e-3)
//     r2 = r1 (1 + e + e^2), e = 1 - d r1   (cubic step, |rel| <= (1.3e-3)^3 + rounding)
// and the term is FFMA2(-r2, -W, magic).  Every f32x2 constant is a kernel parameter, so the
// FFMA2s read it from a uniform register instead of a vector register pair (the f32x2 chain is
// bound by vector-register reads; scripts/k9_pipes.cu measures the variants).
// Host emulation (IEEE fma semantics, scripts/k9_pipes.cu notes): max |r2 d - 1| = 6.2e-8
// (~1 ulp) and r2 is non-increasing in d over every f32 of [1, 2) (the bit trick is
// scale-invariant, so that binade covers all of them).
#ifndef MLSORT_RCP_NEWTON2
#define MLSORT_RCP_NEWTON2 0     // 1: Newton instead of the cubic second step (A/B experiments)
#endif
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 r, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
constexpr uint32_t kSeedNeg = 0xFEF33400u;
// Optional exponent shift of the packed predictor: 1/(1 + 2^a) = 2^-s / (2^-s + 2^(a-s)).
// With s > 0 the chain evaluates d = 2^-s + 2^(a - s) (W scaled by 2^-s), so d stays normal up
// to a = s + 119 and far fewer warps need the per-activation clamp; but a - s is then rounded
// at |a - s| ~ s (ulp 2^-17 for s = 100 instead of <= 2^-19), which coarsens y at the steep
// neurons by about one rank bucket and made K3 slower (0.44 -> 0.58 ms on C2) than K1 got
// faster (1.044 -> 1.021 ms).  Measured and kept off (s = 0, clamp at 59 -> d <= 2^60).
constexpr float kAShift = 0.0f;
constexpr float kAClamp = 60.0f;             // 0x7EF33400 + 0x80000000: bits of -r0 from bits(d)
// Largest argument the chain takes without a clamp: d = 1 + 2^a <= 2^120 keeps the seed
// 0xFEF33400 - bits(d) a negative NORMAL float and every intermediate finite; for a >= 24 the
// term W r + magic rounds to magic exactly (|W r| < 1/4), so nothing depends on the chain's
// accuracy there.
constexpr float kANoClamp = 120.0f;

// -1/d for both lanes of d2 (d in [1, 2^61]) by the packed chain above; shared by the predictor
// and the exhaustive monotonicity sweep (selftest.cuh), so the swept instructions are the
// shipped ones.
__device__ __forceinline__ f32x2 neg_rcp_packed(f32x2 d2, f32x2 k1_2, f32x2 one2) {
    float d0, d1;
    upk2(d2, d0, d1);
    // the seed's bit trick yields -r0 directly (sign bit folded into the constant)
    f32x2 nr2 = pk2(__uint_as_float(kSeedNeg - __float_as_uint(d0)), __uint_as_float(kSeedNeg - __float_as_uint(d1)));
    nr2 = fmul2(nr2, ffma2(d2, nr2, k1_2));                 // -r1 = -r0 (k1 - d r0)
    const f32x2 e2 = ffma2(d2, nr2, one2);                  // e = 1 - d r1
#if MLSORT_RCP_NEWTON2
    return ffma2(nr2, e2, nr2);                             // -r1 (1 + e): |rel| <= 1.7e-6
#else
    return ffma2(nr2, ffma2(e2, e2, e2), nr2);              // -r1 (1 + e + e^2)
#endif
}

// Fixed-point accumulation of Eq. 3: every term w2_j * sigma_j is scaled
// by 2^S (folded into W_j) and rounded to an integer by one FFMA against the magic constant
// 1.5 * 2^23, whose float bits are then summed in a 32-bit integer:
//     acc = sum_j bits(FFMA(sigma_j, W_j, 1.5*2^23)) - M * bits(1.5*2^23)  =  sum_j round(w2_j sigma_j 2^S).
// The sum is exact, every rounding is monotone, so y = acc * 2^-S is monotone in u whenever
// the MUFU results are; and its resolution 2^-S (S = 21 - floor(log2 max|w2|), typically
// 2^-26..2^-27) is much finer than an f32 sum near y = 1 (2^-24), which keeps the rank
// buckets Poisson-like instead of merging up to 2^-24 * B of them.
constexpr float kFxpMagic = 12582912.0f;            // 1.5 * 2^23
constexpr int32_t kFxpMagicBits = 0x4B400000;

// Evaluate Eq. 3 for KG keys at once (independent chains give the SFU/FMA pipes ILP).
// MPAD is the padded neuron count (pad neurons have W = 0).  PRED selects the reciprocal
// formulation; in kPredMixed one neuron in four uses MUFU.RCP and three use the Newton
// reciprocal, balancing MUFU (ex2) load against FMA-pipe issue.
// Overflow guard of the reciprocal chain (d = 1 + 2^a must stay <= 2^120):
//   kClampNone: none -- valid only when every key of the group has u in [u_safe_lo, u_safe_hi]
//               (then a_j <= 59 for every neuron);
//   kClampAct:  a_j = min(a_j, 60) per activation (any model);
//   kClampPair: u_p = max(u, Lp[p]) per neuron pair (packed predictor, fw.pair_clamp != 0).
enum { kClampNone = 0, kClampAct = 1, kClampPair = 2 };
template <int MPAD, int PRED, int KG, int CLAMP = kClampAct>
__device__ __forceinline__ void gvm_forward_fxp(const FoldedWeights& fw, const float (&uh)[KG],
                                                const float (&ul)[KG], int32_t (&acc)[KG]) {
#pragma unroll
    // modular (uint32) arithmetic: the partial sums wrap, the final value fits an int32
    for (int q = 0; q < KG; ++q) acc[q] = (int32_t)(0u - (uint32_t)MPAD * (uint32_t)kFxpMagicBits);
    if (PRED == kPredPacked) {
        const f32x2* A2 = reinterpret_cast<const f32x2*>(fw.A);
        const f32x2* C2 = reinterpret_cast<const f32x2*>(fw.Cs);
        const f32x2* Wn2 = reinterpret_cast<const f32x2*>(fw.Wns);
#pragma unroll
        for (int j = 0; j < MPAD / 2; ++j) {
#pragma unroll
            for (int q = 0; q < KG; ++q) {
                const float up = CLAMP == kClampPair ? fmaxf(uh[q], fw.Lp[j]) : uh[q];
                const f32x2 a2 = ffma2(pk2(up, up), A2[j], C2[j]);     // a - s
                float a0, a1;
                upk2(a2, a0, a1);
                if (CLAMP == kClampAct) {
                    a0 = fminf(a0, kAClamp);         // d stays finite and normal
                    a1 = fminf(a1, kAClamp);
                }
                const f32x2 d2 = fadd2(pk2(ex2_approx(a0), ex2_approx(a1)), fw.dofs2);   // d = 2^-s + e
                const f32x2 nr2 = neg_rcp_packed(d2, fw.k1_2, fw.one2);
                const f32x2 t2 = ffma2(nr2, Wn2[j], fw.magic2);         // W 2^-s r + magic
                float t0, t1;
                upk2(t2, t0, t1);
                acc[q] = (int32_t)((uint32_t)acc[q] + __float_as_uint(t0) + __float_as_uint(t1));
            }
        }
    } else {
#pragma unroll
    for (int j = 0; j < MPAD; j += 2) {          // neuron pairs: one IADD3 accumulates two terms
        int32_t t[2][KG];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float A = fw.A[j + h], C = fw.C[j + h], W = fw.W[j + h];
            const bool use_mufu_rcp = (PRED == kPredMufu) || (((j + h) & 3) == 0);
#pragma unroll
            for (int q = 0; q < KG; ++q) {
                float a = fmaf(A, uh[q], C);
                float r;
                if (use_mufu_rcp) {
                    r = rcp_approx(1.0f + ex2_approx(a));
                } else {
                    a = fminf(a, 60.0f);             // keeps d = 1 + 2^a inside Newton's range (any CLAMP)
                    r = rcp_newton(1.0f + ex2_approx(a));
                }
                t[h][q] = __float_as_int(fmaf(r, W, kFxpMagic));
            }
        }
#pragma unroll
        for (int q = 0; q < KG; ++q) acc[q] = (int32_t)((uint32_t)acc[q] + (uint32_t)t[0][q] + (uint32_t)t[1][q]);
    }
    }
}

// The dense evaluation every kernel outside k1_ws's per-warp choice uses: the per-pair clamp when
// the host established it for these weights (packed predictor), else the per-activation clamp.
// For keys the clamps do not move, both give the bits of the clamp-free chain.
template <int MPAD, int PRED, int KG>
__device__ __forceinline__ void gvm_forward_dense(const FoldedWeights& fw, const float (&uh)[KG],
                                                  const float (&ul)[KG], int32_t (&acc)[KG]) {
    if (PRED == kPredPacked && fw.pair_clamp)
        gvm_forward_fxp<MPAD, PRED, KG, kClampPair>(fw, uh, ul, acc);
    else
        gvm_forward_fxp<MPAD, PRED, KG, kClampAct>(fw, uh, ul, acc);
}

// Packed predictor with saturated-pair skipping for a group of KG keys per lane whose u lie in
// [umin, umax] across the warp (warp-uniform): a pair whose active interval misses
// [umin, umax] contributes its exact constant bits; the others are evaluated.  The result is
// bit-identical to gvm_forward_fxp<MPAD, kPredPacked, KG, CLAMP>.
template <int MPAD, int KG, bool CLAMP>
__device__ __forceinline__ void gvm_forward_skip(const FoldedWeights& fw, const float (&uh)[KG], float umin,
                                                 float umax, int32_t (&acc)[KG]) {
    uint32_t acc_c = 0u - (uint32_t)MPAD * (uint32_t)kFxpMagicBits;
    uint32_t accv[KG];
#pragma unroll
    for (int q = 0; q < KG; ++q) accv[q] = 0u;
    const f32x2* A2 = reinterpret_cast<const f32x2*>(fw.A);
    const f32x2* C2 = reinterpret_cast<const f32x2*>(fw.Cs);
    const f32x2* Wn2 = reinterpret_cast<const f32x2*>(fw.Wns);
#pragma unroll 1
    for (int j = 0; j < MPAD / 2; ++j) {
        if (umax < fw.lo2[j]) {
            acc_c += fw.tl2[j];
            continue;
        }
        if (umin > fw.hi2[j]) {
            acc_c += fw.tr2[j];
            continue;
        }
        const f32x2 Aj = A2[j], Cj = C2[j], Wj = Wn2[j];
#pragma unroll
        for (int q = 0; q < KG; ++q) {
            const f32x2 a2 = ffma2(pk2(uh[q], uh[q]), Aj, Cj);
            float a0, a1;
            upk2(a2, a0, a1);
            if (CLAMP) {
                a0 = fminf(a0, kAClamp);
                a1 = fminf(a1, kAClamp);
            }
            const f32x2 d2 = fadd2(pk2(ex2_approx(a0), ex2_approx(a1)), fw.dofs2);
            const f32x2 nr2 = neg_rcp_packed(d2, fw.k1_2, fw.one2);
            const f32x2 t2 = ffma2(nr2, Wj, fw.magic2);
            float t0, t1;
            upk2(t2, t0, t1);
            accv[q] += __float_as_uint(t0) + __float_as_uint(t1);
        }
    }
#pragma unroll
    for (int q = 0; q < KG; ++q) acc[q] = (int32_t)(accv[q] + acc_c);
}

// order-preserving unsigned bits of an f32 (IEEE totalOrder)
__device__ __forceinline__ uint32_t f32_ordbits(float x) {
    const uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// r = clamp(round_half_up(y * B), 0, B - 1) with y = acc * 2^-S, in exact integer arithmetic
// (S:232, S:297-S:298).  For y >= 0 round-half-up equals round-half-away-
// from-zero (reading A6); negative y map to bucket 0.
__device__ __forceinline__ uint32_t bucket_of_fxp(int32_t acc, const BucketMap& bm) {
    if (bm.pow2 && bm.sh >= 0) {
        // B = 2^k, sh = S - k >= 0: (acc * 2^k + 2^(S-1)) >> S == (acc + 2^(sh-1)) >> sh (half = 0
        // for sh = 0), exactly, in 32-bit arithmetic: |acc| < M * 2^22 <= 2^28 (fxp_shift), so
        // acc + half cannot overflow; the arithmetic shift keeps negative sums negative
        const int32_t r = (acc + bm.half) >> bm.sh;
        return (uint32_t)min(max(r, 0), (int32_t)bm.Bm1);
    }
    if (bm.pow2) {
        // sh < 0: acc * 2^-sh (the 1/2 floors away), exactly
        long long r = (long long)acc << (-bm.sh);
        r = r < 0 ? 0 : r;
        return r < (long long)bm.Bm1 ? (uint32_t)r : bm.Bm1;
    }
    const long long v = (long long)acc * (long long)bm.B + (1ll << (bm.S - 1));
    if (v < 0) return 0u;
    const unsigned long long r = (unsigned long long)v >> bm.S;
    return r < bm.Bm1 ? (uint32_t)r : bm.Bm1;
}

__device__ __forceinline__ float fxp_to_float(int32_t acc, const BucketMap& bm) {
    return (float)acc * __int_as_float((127 - (int)bm.S) << 23);
}

}  // namespace mlsort
