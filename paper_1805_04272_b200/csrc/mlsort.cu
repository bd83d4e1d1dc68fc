// mlsort.cu -- libmlsort.so device entry points: plan selection, workspace layout, kernel
// dispatch and the one host synchronisation per sort.
//
// Pipeline of mlsort_sort:
//   K1 predict + bucket + tile partition + region store (Eq. 3 l.73-76, l.65)
//   K2 coarse-bucket starts (scan of the exact bucket sizes left in the region cursors)
//   K3 cluster gather + rank-bucket placement + per-bucket fix-up (l.86)
//   K4 overflow path for coarse buckets K3 cannot hold (l.121 tails)
//   K5 boundary verify (reading A14) -> conventional-sort fallback on violation
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.h"
#include "common.cuh"
#include "predict.cuh"
#include "k1_partition.cuh"
#include "k1_ws.cuh"
#include "k3_sort.cuh"
#include "k3_local.cuh"
#include "k4_overflow.cuh"
#include "dist.cuh"
#include "selftest.cuh"
#include "k0_sample.cuh"

using namespace mlsort;

// Internal helpers live in a namespace named per translation-unit slice (see the split below):
// the same file is compiled several times, and nvcc gives an anonymous namespace the same
// external name in every one of those objects.
#ifndef MLSORT_TU
#define MLSORT_TU_NAME all
#else
#define MLSORT_TU_NAME MLSORT_TU
#endif
#define MLSORT_CAT2(a, b) a##b
#define MLSORT_CAT(a, b) MLSORT_CAT2(a, b)
#define MLSORT_LOCAL MLSORT_CAT(mlsort_local_tu, MLSORT_TU_NAME)
namespace MLSORT_LOCAL {}
using namespace MLSORT_LOCAL;

// NVTX phase ranges (nvtx3 is header-only: no cost unless a profiler injects itself)
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, size): a driver call per
// launch would add host time in front of every sort
template <typename F>
cudaError_t set_smem(F* kern, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> done;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const void* key = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(kern) ^ ((uintptr_t)dev << 56));
    for (auto& d : done)
        if (d.first == key && d.second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
        bool found = false;
        for (auto& d : done)
            if (d.first == key) {
                d.second = bytes;
                found = true;
            }
        if (!found) done.emplace_back(key, bytes);
    }
    return e;
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "mlsort: CUDA error %s at %s:%d: %s\n", cudaGetErrorName(e_),       \
                    __FILE__, __LINE__, cudaGetErrorString(e_));                                \
            return MLSORT_ERR_CUDA;                                                             \
        }                                                                                       \
    } while (0)

namespace MLSORT_LOCAL {

constexpr size_t kAlign = 256;
constexpr double kRegionFactor = 4.0;        // region capacity / average coarse-bucket size
constexpr size_t kK3SmemBudget = 74752;      // three K3 CTAs (256 threads each) per SM
constexpr size_t kK3LSmemMax = 232448;       // K3 secondary pass: one 1024-thread CTA per SM (227 KB)
constexpr size_t kK3LSmemPrimary = 115712;   // K3 primary pass: two 512-thread CTAs per SM (113 KB each)
constexpr size_t kK1SmemMax = 110 * 1024;    // K1: keep two 512-thread CTAs per SM
constexpr int kSMs = 148;

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline uint32_t ceil_log2(uint64_t x) {
    uint32_t r = 0;
    while ((1ull << r) < x) ++r;
    return r;
}

// ---------------------------------------------------------------- folded weights (A1 item 1)
// Fixed-point scale of the y accumulator: |w2_j| 2^S < 2^22 for every neuron (so each
// rounded term stays in the magic constant's binade) -> S = 21 - floor(log2 max|w2|).
uint32_t fxp_shift(const Weights& w) {
    double mx = 0;
    for (uint32_t j = 0; j < w.m; ++j) mx = std::max(mx, std::fabs(w.w2[j]));
    if (mx <= 0) return 30;
    int e = (int)std::floor(std::log2(mx));
    int S = 21 - e;
    return (uint32_t)std::max(1, std::min(30, S));
}

// Origin of u = x - x0 (predict.cuh "Folding"): 0 for f32 keys whose range straddles or is
// near 0 (u = x exactly), otherwise input_lo.
double origin_of(const Weights& w, bool f32) {
    if (!f32) return w.lo;
    const double span = w.hi - w.lo;
    if ((w.lo <= 0.0 && w.hi >= 0.0) || std::max(std::fabs(w.lo), std::fabs(w.hi)) <= 4.0 * span) return 0.0;
    return (double)(float)w.lo;
}

// Device reciprocal chain of the packed predictor evaluated at d = 1 (host emulation with IEEE
// fma / multiply, bit-identical to FFMA2 / FMUL2): -r(1), the value every a <= -26 produces.
float neg_rcp_at_one() {
    auto bits_f = [](uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; };
    const float d = 1.0f, k1 = 2.001281198f;
    const float nr0 = bits_f(0xFEF33400u - 0x3F800000u);
    const float t = std::fmaf(d, nr0, k1);
    const float nr1 = nr0 * t;
    const float e = std::fmaf(d, nr1, 1.0f);
    const float pp = std::fmaf(e, e, e);
    return std::fmaf(nr1, pp, nr1);
}

uint32_t f32_bits(float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    return b;
}

FoldedWeights fold(const Weights& w, uint32_t mpad, bool f32) {
    FoldedWeights f;
    std::memset(&f, 0, sizeof(f));
    const double log2e = 1.4426950408889634;
    const double span = w.hi - w.lo;
    const double scale = std::ldexp(1.0, (int)fxp_shift(w));
    const double x0 = origin_of(w, f32);
    // neurons sorted by the centre of their logistic (u where a_j = 0), so that the two neurons
    // of a pair saturate together and a warp's narrow u range skips whole pairs; the sum of
    // Eq. 3 is order-independent (exact integer accumulation)
    std::vector<uint32_t> order(w.m);
    for (uint32_t j = 0; j < w.m; ++j) order[j] = j;
    auto centre = [&](uint32_t j) {
        const double A = -2.0 * w.beta[j] * w.w1[j] * log2e / span;
        const double C = w.beta[j] * (w.w1[j] + w.b[j]) * log2e + A * (x0 - w.lo);
        return A != 0.0 ? -C / A : 0.0;
    };
    // Models whose neurons all have A_j < 0 (every monotone increasing net the trainer emits) are
    // ordered by the left saturation bound instead (a_j = 24.5), which pairs neurons whose
    // per-pair clamp interval is non-empty (predict.cuh FoldedWeights::Lp; checked below).
    auto coefA = [&](uint32_t j) { return -2.0 * w.beta[j] * w.w1[j] * log2e / span; };
    bool all_neg = w.m > 0;
    for (uint32_t j = 0; j < w.m; ++j) all_neg &= coefA(j) < 0.0;
    auto left_bound = [&](uint32_t j) {
        const double A = coefA(j);
        const double C = w.beta[j] * (w.w1[j] + w.b[j]) * log2e + A * (x0 - w.lo);
        return (24.5 - C) / A;
    };
    if (all_neg && !std::getenv("MLSORT_NO_PAIR_CLAMP"))
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return left_bound(a) < left_bound(b); });
    else
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return centre(a) < centre(b); });
    for (uint32_t j = 0; j < mpad; ++j) {
        if (j < w.m) {
            const uint32_t o = order[j];
            const double A = -2.0 * w.beta[o] * w.w1[o] * log2e / span;
            f.A[j] = (float)A;
            f.C[j] = (float)(w.beta[o] * (w.w1[o] + w.b[o]) * log2e + A * (x0 - w.lo));
            f.W[j] = (float)(w.w2[o] * scale);
            f.Wn[j] = -f.W[j];
            f.Cs[j] = (float)((double)f.C[j] - (double)kAShift);
            f.Wns[j] = std::ldexp(f.Wn[j], -(int)kAShift);
        } else {
            f.A[j] = 0.0f;
            f.C[j] = 0.0f;
            f.W[j] = 0.0f;   // pad neurons contribute nothing
            f.Wn[j] = 0.0f;
            f.Cs[j] = -kAShift;
            f.Wns[j] = 0.0f;
        }
    }
    // ---- saturated-pair skipping bounds and constants (predict.cuh gvm_forward_skip)
    const float nr_one = neg_rcp_at_one();
    const uint32_t kMagicBits = 0x4B400000u;
    for (uint32_t pp = 0; pp < mpad / 2; ++pp) {
        double lo2 = INFINITY, hi2 = -INFINITY;
        uint32_t tl = 0, tr = 0;
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t j = 2 * pp + h;
            const double A = f.A[j], C = f.C[j];
            const uint32_t tzero = kMagicBits;
            const uint32_t tsat = f32_bits(std::fmaf(nr_one, f.Wn[j], 12582912.0f));
            double lo, hi;
            uint32_t left, right;
            if (A < 0) {            // u -> -inf: a -> +inf (term 0); u -> +inf: saturated
                lo = (24.5 - C) / A;
                hi = (-26.5 - C) / A;
                left = tzero;
                right = tsat;
            } else if (A > 0) {     // u -> -inf: saturated; u -> +inf: term 0
                lo = (-26.5 - C) / A;
                hi = (24.5 - C) / A;
                left = tsat;
                right = tzero;
            } else if (f.W[j] == 0.0f) {   // pad: a constant zero term everywhere
                lo = INFINITY;
                hi = -INFINITY;
                left = right = tzero;
            } else {                // a constant argument: never skipped
                lo = -INFINITY;
                hi = INFINITY;
                left = right = tzero;
            }
            lo2 = std::min(lo2, lo);
            hi2 = std::max(hi2, hi);
            tl += left;
            tr += right;
        }
        // round outwards so a skip decision on f32 u is always safe
        float flo = (float)lo2, fhi = (float)hi2;
        if (std::isfinite(flo) && (double)flo > lo2) flo = std::nextafter(flo, -INFINITY);
        if (std::isfinite(fhi) && (double)fhi < hi2) fhi = std::nextafter(fhi, INFINITY);
        f.lo2[pp] = flo;
        f.hi2[pp] = fhi;
        f.tl2[pp] = tl;
        f.tr2[pp] = tr;
    }
    // ---- value classes for k1_ws's grouping: class = floor(64 y(u)) on a log-like grid of u
    // (the top 11 order-preserving bits of the f32 u); only performance depends on it
    for (uint32_t i = 0; i < 2048; ++i) {
        const uint32_t ob = (i << 21) | (1u << 20);
        const uint32_t bits = (ob & 0x80000000u) ? (ob & 0x7fffffffu) : ~ob;
        float u;
        std::memcpy(&u, &bits, 4);
        int cls;
        if (!std::isfinite(u)) {
            cls = (ob & 0x80000000u) ? 63 : 0;
        } else {
            const double x = (double)u + x0;
            const double xh = 2.0 * (x - w.lo) / span - 1.0;
            double y = 0;
            for (uint32_t j = 0; j < w.m; ++j) {
                const double t = w.beta[j] * (w.w1[j] * xh - w.b[j]);
                y += w.w2[j] / (1.0 + std::exp(-t));
            }
            cls = (int)std::floor(y * 64.0);
            cls = std::max(0, std::min(63, cls));
        }
        f.lut[i] = (unsigned char)cls;
    }
    // safe range of u for the clamp-free packed predictor: A_j u + Cs_j <= kAClamp - 1 for every
    // neuron (the f32 FFMA's rounding is far below the margin of the reciprocal chain, whose d
    // stays normal up to a - s = 125)
    double ulo = -INFINITY, uhi = INFINITY;
    const double amax = (double)kAClamp - 1.0;
    for (uint32_t j = 0; j < mpad; ++j) {
        const double A = f.A[j], C = f.Cs[j];
        if (A < 0) ulo = std::max(ulo, (amax - C) / A);
        else if (A > 0) uhi = std::min(uhi, (amax - C) / A);
        else if (C > amax) { ulo = INFINITY; uhi = -INFINITY; }
    }
    f.u_safe_lo = ulo == -INFINITY ? -INFINITY : (float)std::nextafter((float)ulo, INFINITY);
    f.u_safe_hi = uhi == INFINITY ? INFINITY : (float)std::nextafter((float)uhi, -INFINITY);
    if (!(f.u_safe_lo <= f.u_safe_hi)) { f.u_safe_lo = INFINITY; f.u_safe_hi = -INFINITY; }
    // ---- key-side clamp (K1Params u_cl_lo/hi): below min_p lo2[p] every pair is in its left
    // saturation and above max_p hi2[p] in its right one, where each term is an exact constant;
    // clamping u just inside those bounds changes no output bit.  If no argument can exceed
    // kANoClamp inside them, every warp runs the clamp-free chain.
    f.u_cl_lo = -INFINITY;
    f.u_cl_hi = INFINITY;
    {
        float lo = INFINITY, hi = -INFINITY;
        for (uint32_t pp = 0; pp < mpad / 2; ++pp) {
            if (std::isfinite(f.lo2[pp])) lo = std::min(lo, f.lo2[pp]);
            if (std::isfinite(f.hi2[pp])) hi = std::max(hi, f.hi2[pp]);
        }
        bool ok = std::isfinite(lo) && std::isfinite(hi) && lo <= hi;
        if (ok) {
            lo = std::nextafter(lo, -INFINITY);
            hi = std::nextafter(hi, INFINITY);
            for (uint32_t j = 0; j < mpad && ok; ++j) {
                const double a1 = (double)f.A[j] * lo + (double)f.Cs[j], a2 = (double)f.A[j] * hi + (double)f.Cs[j];
                ok = std::max(a1, a2) <= (double)kANoClamp - 1.0;
            }
        }
        if (ok && !std::getenv("MLSORT_NO_UCLAMP")) {
            f.u_cl_lo = lo;
            f.u_cl_hi = hi;
            f.u_safe_lo = -INFINITY;
            f.u_safe_hi = INFINITY;
        }
    }
    // ---- per-pair lower clamp (predict.cuh FoldedWeights::Lp): for u >= L_p every argument of
    // the pair is <= 119 (the chain's d stays <= 2^120), and L_p lies below both neurons' left
    // saturation bound (a >= 24.5: the computed term is the exact constant 0, as for every u < L_p),
    // so max(u, L_p) changes no output bit.  Pad neurons (A = 0, a = 0) accept any L_p.
    // Not needed when the key-side clamp already keeps every argument <= 119 (u_safe spans
    // everything: the clamp-free chain for every warp, e.g. C1).
    f.pair_clamp = 0;
    const bool clamp_free = f.u_safe_lo == -INFINITY && f.u_safe_hi == INFINITY;
    if (all_neg && !clamp_free && !std::getenv("MLSORT_NO_PAIR_CLAMP")) {
        bool ok = true;
        for (uint32_t pp = 0; pp < mpad / 2 && ok; ++pp) {
            double thr = -INFINITY, lob = INFINITY;
            for (uint32_t h = 0; h < 2; ++h) {
                const uint32_t j = 2 * pp + h;
                const double A = f.A[j], C = f.Cs[j];
                if (A < 0.0) {
                    thr = std::max(thr, ((double)kANoClamp - 1.0 - C) / A);
                    lob = std::min(lob, (24.5 - C) / A);
                } else if (A > 0.0 || C > (double)kANoClamp - 1.0) {
                    ok = false;
                }
            }
            float L = thr == -INFINITY ? -INFINITY : (float)thr;
            if (std::isfinite(L) && (double)L < thr) L = std::nextafter(L, INFINITY);   // round up
            ok = ok && (double)L <= lob - 1e-6 * std::max(1.0, std::fabs(lob));
            f.Lp[pp] = L;
        }
        f.pair_clamp = ok ? 1u : 0u;
    }
    auto pair = [](float v) {
        uint32_t bb;
        std::memcpy(&bb, &v, 4);
        return ((unsigned long long)bb << 32) | bb;
    };
    f.one2 = pair(1.0f);
    f.k1_2 = pair(2.001281198f);
    f.magic2 = pair(12582912.0f);
    f.dofs2 = pair(std::ldexp(1.0f, -(int)kAShift));
    return f;
}

// Folding costs ~1 ms of host time (the 2048-entry class table evaluates the network); it is
// done once per (weights handle, key dtype) and cached.
const FoldedWeights& fold_cached(const Weights& w, uint32_t mpad, bool f32) {
    struct Entry {
        uint64_t serial;
        uint32_t mpad;
        bool f32;
        FoldedWeights fw;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;     // small, most recent last
    thread_local FoldedWeights result;
    std::lock_guard<std::mutex> lock(mu);
    for (size_t i = 0; i < cache.size(); ++i)
        if (cache[i].serial == w.serial && cache[i].mpad == mpad && cache[i].f32 == f32) {
            result = cache[i].fw;
            return result;
        }
    if (cache.size() >= 16) cache.erase(cache.begin());
    cache.push_back(Entry{w.serial, mpad, f32, fold(w, mpad, f32)});
    result = cache.back().fw;
    return result;
}

uint32_t mpad_of(uint32_t m);

// Public predictor choice -> internal variant.  MLSORT_PRED_DEFAULT is the packed predictor,
// with value grouping + saturated-pair skipping when M > 32: measured on B200, M = 64 (C3) K1
// 14.9 -> 5.3 ms with it, M = 32 (C2) 1.01 -> 1.23 ms.  MLSORT_GROUP=1/0 overrides the default
// (experiments).  Skipping is exact, so every variant of the packed family gives the same bits.
int resolve_pred(int32_t predictor, uint32_t m) {
    if (predictor == MLSORT_PRED_MUFU) return kPredMufu;
    if (predictor == MLSORT_PRED_MIXED) return kPredMixed;
    if (predictor == MLSORT_PRED_PACKED) return kPredPacked;
    if (predictor == MLSORT_PRED_SKIP) return kPredSkip;
    const char* e = std::getenv("MLSORT_GROUP");
    if (e) return std::atoi(e) != 0 ? kPredSkip : kPredPacked;
    return mpad_of(m) >= 64 ? kPredSkip : kPredPacked;
}

uint32_t mpad_of(uint32_t m) { return m <= 16 ? 16 : m <= 32 ? 32 : 64; }

// ---------------------------------------------------------------- plan
struct Plan {
    uint64_t n = 0, B = 0;
    uint32_t tile = kTileSmall;
    uint32_t T = 0, fb = 0, C = 0, R = 1, kr = 1, cap = 0, capc = 0;
    size_t k1_smem = 0, k3_smem = 0;
    size_t ks = 4;
    bool perm = false;
    bool local = false;      // K3 = one CTA per coarse bucket (k3_local_sort), else clusters
    uint32_t cap1 = 0;       // local plan: primary-pass capacity (two CTAs per SM)
    size_t k3_smem1 = 0;     // local plan: primary-pass shared memory
    bool ws = false;         // K1 = warp-specialized persistent k1_ws (tile = ws tile), else k1_predict_partition
    bool ws_stage = true;    // k1_ws stages the keys in shared memory (else re-reads them from L2)
    bool ws_group = false;   // k1_ws with value grouping + saturated-pair skipping
    uint32_t kfine = 0;      // rank buckets per coarse bucket (local plan)
    uint32_t item_cap = 0;   // local plan: k3_cut item list / segment list capacities (k3_big.cuh)
    uint32_t seg_cap = 0;
    bool sampled = false;    // regions sized from a sample of the predicted buckets (K0)
    uint64_t stride = 1;     // K0: every stride-th key is predicted
    uint64_t area = 0;       // region slots (all coarse buckets)
};

// Regions sized by K0 (k0_sample.cuh) for inputs large enough that fixed 4x regions waste GBs
// and skewed data overflows them (one more K1 pass); small inputs keep the fixed layout.
constexpr uint64_t kSampledMinN = 1ull << 27;
constexpr uint64_t kSampleTarget = 1ull << 22;     // sampled keys per call

void set_region_area(Plan& p) {
    if (p.sampled) {
        const double S = (double)p.stride, C = (double)p.C, n = (double)p.n;
        p.area = (uint64_t)(n + 6.0 * std::sqrt(S * C * (n + S * C)) + 72.0 * C) + 64;
        p.area = (p.area + 7) & ~7ull;
    } else {
        p.area = (uint64_t)p.C * p.capc;
    }
}

size_t k3_elem_bytes(size_t ks, bool perm) { return ks * 2 + 4 + (perm ? 8 : 0); }

constexpr size_t kK1WsSmemMax = 232448;      // 227 KB, the sm_100 per-block maximum

uint32_t ws_tile_of(size_t ks, bool group = false) {
    return ks == 4 ? (uint32_t)ws_tile<float>(group) : (uint32_t)ws_tile<double>(group);
}

Plan make_plan_base(uint64_t n, uint64_t B, size_t ks, bool perm, bool allow_ws);

// Choose the K1 variant after the coarse partition is fixed: the warp-specialized kernel when
// its shared memory fits (and the caller predicts), else the phase-alternating one.
Plan make_plan(uint64_t n, uint64_t B, size_t ks, bool perm, bool allow_ws = true, bool group = false) {
    Plan p = make_plan_base(n, B, ks, perm, allow_ws);
    // K0-sized regions: predicting sorts only (the records path has no network to sample)
    p.sampled = allow_ws && n >= kSampledMinN && !std::getenv("MLSORT_NO_SAMPLE");
    p.stride = std::max<uint64_t>(1, n / kSampleTarget);
    set_region_area(p);
    // the value-grouped variant when asked for and its shared memory fits, else the plain one
    for (int gi = group ? 0 : 1; allow_ws && gi < 2 && !p.ws; ++gi) {
        const bool g = gi == 0;
        const uint32_t wt = ws_tile_of(ks, g);
        size_t sm = k1ws_smem_bytes(ks, wt, p.C, g, true);
        p.ws_stage = sm <= kK1WsSmemMax && !std::getenv("MLSORT_NO_STAGE");
        if (!p.ws_stage) sm = k1ws_smem_bytes(ks, wt, p.C, g, false);
        // k1_ws keeps 32-bit region slots (+ tile) with 0xFFFFFFFF reserved
        const bool slots32 = p.area + p.tile + (uint64_t)wt + 8 < 0xFFFFFFFFull;
        if (sm <= kK1WsSmemMax && slots32) {
            p.ws = true;
            p.ws_group = g;
            p.tile = wt;
            p.T = (uint32_t)((n + wt - 1) / wt);
            p.k1_smem = sm;
        }
    }
    return p;
}

// k3_cut emits at most 2 n_c / (cap/2) + 2 items per coarse bucket plus one empty item per giant
// rank bucket, and at most n / cap + 1 segments per ... (k3_big.cuh): bounded by the totals
void set_item_caps(Plan& p) {
    const uint64_t cap = std::max<uint32_t>(p.cap, 2);
    p.item_cap = (uint32_t)std::min<uint64_t>(0x7FFFFFFFull, 8 * p.n / cap + 4ull * p.C + 64);
    p.seg_cap = (uint32_t)std::min<uint64_t>(0x7FFFFFFFull, 2 * p.n / cap + p.C + 64);
}

Plan make_plan_base(uint64_t n, uint64_t B, size_t ks, bool perm, bool allow_ws) {
    Plan p;
    p.n = n;
    p.B = B;
    p.ks = ks;
    p.perm = perm;
    p.tile = kTileSmall;
    p.T = (uint32_t)((n + p.tile - 1) / p.tile);
    const uint32_t lb = ceil_log2(B);
    const uint32_t fb_max = std::min<uint32_t>(16, lb);
    const uint32_t fb_min = lb > 14 ? lb - 14 : 0;   // C <= 16384
    // Local plan (preferred): the fewest coarse buckets such that one CTA holds a coarse bucket
    // of 2x the average size in shared memory next to its rank-bucket histogram.
    // MLSORT_FINE_BITS=<fb> forces the rank-bucket bits of the local plan (experiments only)
    const char* fb_env = std::getenv("MLSORT_FINE_BITS");
    const int fb_force = fb_env ? std::atoi(fb_env) : -1;
    for (int fb = (int)fb_max; fb >= (int)fb_min; --fb) {
        if (fb_force >= 0 && fb != fb_force) continue;
        const uint64_t C = (B + (1ull << fb) - 1) >> fb;
        const size_t k1 = k1_smem_bytes(ks, perm, p.tile, (uint32_t)C);
        const bool ws_fits = allow_ws && k1ws_smem_bytes(ks, ws_tile_of(ks), (uint32_t)C, false, false) <= kK1WsSmemMax;
        if (k1 > kK1SmemMax && !ws_fits) continue;
        const uint32_t kfine = 1u << fb;
        const uint64_t cap = k3l_cap_for(kK3LSmemMax, ks, perm, kfine, kL3ThreadsBig);
        const double avg = (double)n * (double)kfine / (double)B;
        if ((double)cap < 2.0 * avg + 64.0) continue;
        p.local = true;
        p.fb = (uint32_t)fb;
        p.C = (uint32_t)C;
        p.R = 1;
        p.kr = kfine;
        p.kfine = kfine;
        p.cap = (uint32_t)cap;
        p.k1_smem = k1;
        p.k3_smem = k3l_smem_bytes(ks, perm, kfine, (uint32_t)cap, kL3ThreadsBig);
        // two-CTA primary pass only when it holds the average bucket with margin
        // (the primary pass keeps kfine counters although it merges rank-bucket pairs: sizing it
        // for the merged buckets -- cap1 18432 -> 22528 on C2 -- moved buckets from the
        // 1024-thread secondary pass into it and made K3 slower, 0.389 -> 0.396 ms,
        // profiles/r02/ab_k3_cap1_finebits13_rejected.log)
        p.cap1 = k3l_cap_for(kK3LSmemPrimary, ks, perm, kfine, kL3Threads);
        if ((double)p.cap1 < 1.1 * avg + 64.0 || std::getenv("MLSORT_K3_NO_PRIMARY")) p.cap1 = 0;
        p.k3_smem1 = p.cap1 ? k3l_smem_bytes(ks, perm, kfine, p.cap1, kL3Threads) : 0;
        uint64_t cc = (uint64_t)std::ceil(kRegionFactor * avg) + 64;
        cc = (cc + 7) & ~7ull;
        p.capc = (uint32_t)std::min<uint64_t>(cc, 0xFFFFFFF0ull);
        set_item_caps(p);
        return p;
    }
    // No rank-bucket split gives an average coarse bucket that one CTA holds with margin (large
    // f64 inputs, a CTA's shared memory being the limit): the most coarse buckets K1 allows,
    // and k3_cut splits every coarse bucket that does not fit into items that do (k3_big.cuh).
    for (int fb = (int)std::max(fb_min, 0u); fb <= (int)fb_max; ++fb) {
        const uint64_t C = (B + (1ull << fb) - 1) >> fb;
        const bool k1_ok = k1_smem_bytes(ks, perm, p.tile, (uint32_t)C) <= kK1SmemMax ||
                           (allow_ws && k1ws_smem_bytes(ks, ws_tile_of(ks), (uint32_t)C, false, false) <= kK1WsSmemMax);
        if (!k1_ok && fb < (int)fb_max) continue;
        const uint32_t kfine = 1u << fb;
        p.local = true;
        p.fb = (uint32_t)fb;
        p.C = (uint32_t)C;
        p.R = 1;
        p.kr = kfine;
        p.kfine = kfine;
        p.cap = k3l_cap_for(kK3LSmemMax, ks, perm, kfine, kL3ThreadsBig);
        p.k1_smem = k1_smem_bytes(ks, perm, p.tile, p.C);
        p.k3_smem = k3l_smem_bytes(ks, perm, kfine, p.cap, kL3ThreadsBig);
        p.cap1 = 0;
        p.k3_smem1 = 0;
        break;
    }
    set_item_caps(p);
    {   // region capacity: kRegionFactor x the average coarse bucket, multiple of 8 (16 B rows)
        const double avg = (double)n * (double)(1ull << p.fb) / (double)B;
        uint64_t cc = (uint64_t)std::ceil(kRegionFactor * avg) + 64;
        cc = (cc + 7) & ~7ull;
        p.capc = (uint32_t)std::min<uint64_t>(cc, 0xFFFFFFF0ull);
    }
    return p;
}

// ---------------------------------------------------------------- workspace layout
struct Layout {
    size_t status = 0, reg_keys = 0, reg_fine = 0, reg_idx = 0, cursor = 0, starts = 0,
           range_start = 0, big_list = 0, flags = 0, big_mark = 0, radix = 0, mid_list = 0, segs = 0, rbase = 0,
           items = 0, k3segs = 0, est = 0, total = 0;
    size_t radix_bytes = 0;
};

size_t radix_area(uint64_t n, size_t bits_bytes, bool payload) {
    const uint64_t nchunks = (n + kRadixChunk - 1) / kRadixChunk;
    return align_up(n * bits_bytes) * 2 + (payload ? align_up(n * 4) * 2 : 0) + align_up(nchunks * 256 * 4) +
           align_up((nchunks * 256 / kScanTile + 1) * 4);
}

Layout make_layout(const Plan& p) {
    Layout L;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align_up(bytes);
        return o;
    };
    L.status = take(sizeof(DevStatus));
    // regions (K1 -> K3/K4) and the radix area (K4 radix / fallback) are never live together
    // C regions of capc slots, plus one tile of trash rows for pieces that overflow a region
    const uint64_t slots = p.area + p.tile;
    const size_t reg_bytes = align_up(slots * p.ks) + align_up(slots * 2) + (p.perm ? align_up(slots * 4) : 0);
    const size_t rad = radix_area(p.n, p.ks, p.perm);
    const size_t shared_area = std::max(reg_bytes, rad);
    const size_t area = take(shared_area);
    L.reg_keys = area;
    L.reg_fine = area + align_up(slots * p.ks);
    L.reg_idx = L.reg_fine + align_up(slots * 2);
    L.radix = area;
    L.radix_bytes = shared_area;
    L.cursor = take((size_t)p.C * 4);
    L.starts = take((size_t)(p.C + 1) * 8);
    L.range_start = take((size_t)p.C * p.R * 8);
    L.big_list = take((size_t)p.C * 4);
    L.flags = take((size_t)p.C * 4);
    L.big_mark = take((size_t)p.C * 4);
    L.mid_list = take((size_t)p.C * 4);
    L.segs = take((size_t)std::max<uint32_t>(p.C, p.seg_cap) * 24);
    L.rbase = take((size_t)(p.C + 1) * 8);
    L.items = take((size_t)p.item_cap * sizeof(K3Item));
    L.k3segs = take((size_t)p.seg_cap * sizeof(K3Seg));
    L.est = take((size_t)p.C * 4);
    L.total = off;
    return L;
}

template <typename T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

struct HostStatusBuf {
    DevStatus* h = nullptr;
    std::mutex mu;
};
thread_local DevStatus* tl_status = nullptr;
DevStatus* host_status() {
    if (!tl_status) {
        if (cudaMallocHost(&tl_status, sizeof(DevStatus)) != cudaSuccess) {
            tl_status = nullptr;
            static DevStatus fallback;
            return &fallback;
        }
    }
    return tl_status;
}

int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = kSMs;
    }
    return g_num_sms;
}

// ---------------------------------------------------------------- launch helpers
struct Launches {
    uint64_t count = 0;
};

template <typename KeyT, int MPAD, int PRED, bool PERM, bool GIVEN>
cudaError_t launch_k1_t(const Plan& p, const KeyT* keys, const FoldedWeights& fw, const K1Params& kp,
                        void* ws, const Layout& L, cudaStream_t s, const uint32_t* bucket_in,
                        const uint32_t* idx_in, uint32_t b_lo, const unsigned long long* rbase) {
    auto kern = k1_predict_partition<KeyT, MPAD, PRED, PERM, GIVEN, kTileSmall>;
    cudaError_t e = set_smem(kern, p.k1_smem);
    if (e != cudaSuccess) return e;
    kern<<<kp.num_tiles, kThreads, p.k1_smem, s>>>(keys, fw, kp, at<KeyT>(ws, L.reg_keys), at<uint16_t>(ws, L.reg_fine),
                                          PERM ? at<uint32_t>(ws, L.reg_idx) : nullptr,
                                          at<uint32_t>(ws, L.cursor), at<DevStatus>(ws, L.status), bucket_in,
                                          idx_in, b_lo, rbase);
    return cudaGetLastError();
}

#ifndef MLSORT_K1_KG
#define MLSORT_K1_KG 8
#endif
constexpr int kK1Kg = MLSORT_K1_KG;   // keys per predictor lane in flight (k1_ws KGW)

template <typename KeyT, int MPAD, int PRED, bool PERM>
cudaError_t launch_k1_ws_t(const Plan& p, const KeyT* keys, const FoldedWeights& fw, const K1Params& kp, void* ws,
                           const Layout& L, cudaStream_t s, const unsigned long long* rbase) {
    const bool group = PRED == kPredPacked && p.ws_group;
    auto kern = group ? k1_ws<KeyT, MPAD, PRED, PERM, 8, true, PRED == kPredPacked>
                      : k1_ws<KeyT, MPAD, PRED, PERM, kK1Kg, true, false>;
    cudaError_t e = set_smem(kern, p.k1_smem);
    if (e != cudaSuccess) return e;
    const int grid = std::min<int>(num_sms(), (int)kp.num_tiles);
    kern<<<grid, ws_threads(group), p.k1_smem, s>>>(keys, kp, at<KeyT>(ws, L.reg_keys), at<uint16_t>(ws, L.reg_fine),
                                             PERM ? at<uint32_t>(ws, L.reg_idx) : nullptr, at<uint32_t>(ws, L.cursor),
                                             at<DevStatus>(ws, L.status), rbase, fw);
    return cudaGetLastError();
}

template <typename KeyT, bool PERM, bool GIVEN>
cudaError_t launch_k1(const Plan& p, const KeyT* keys, uint32_t mpad, int pred, const FoldedWeights& fw,
                      const K1Params& kp, void* ws, const Layout& L, cudaStream_t s,
                      const uint32_t* bucket_in = nullptr, const uint32_t* idx_in = nullptr, uint32_t b_lo = 0,
                      const unsigned long long* rbase = nullptr) {
    if (GIVEN)
        return launch_k1_t<KeyT, 16, kPredMufu, PERM, GIVEN>(p, keys, fw, kp, ws, L, s, bucket_in, idx_in, b_lo, rbase);
    if (!GIVEN && p.ws) {
#define K1WS(M)                                                                                            \
        if (mpad == M) {                                                                                   \
            if (pred == kPredMufu) return launch_k1_ws_t<KeyT, M, kPredMufu, PERM>(p, keys, fw, kp, ws, L, s, rbase);   \
            if (pred == kPredMixed) return launch_k1_ws_t<KeyT, M, kPredMixed, PERM>(p, keys, fw, kp, ws, L, s, rbase); \
            return launch_k1_ws_t<KeyT, M, kPredPacked, PERM>(p, keys, fw, kp, ws, L, s, rbase);                   \
        }
        K1WS(16) K1WS(32) K1WS(64)
#undef K1WS
        return cudaErrorInvalidValue;
    }
#define K1CASE(M)                                                                                          \
    if (mpad == M) {                                                                                       \
        if (pred == kPredMufu)                                                                             \
            return launch_k1_t<KeyT, M, kPredMufu, PERM, GIVEN>(p, keys, fw, kp, ws, L, s, bucket_in, idx_in, b_lo, rbase); \
        if (pred == kPredPacked)                                                                           \
            return launch_k1_t<KeyT, M, kPredPacked, PERM, GIVEN>(p, keys, fw, kp, ws, L, s, bucket_in, idx_in, b_lo, rbase); \
        return launch_k1_t<KeyT, M, kPredMixed, PERM, GIVEN>(p, keys, fw, kp, ws, L, s, bucket_in, idx_in, b_lo, rbase);    \
    }
    K1CASE(16) K1CASE(32) K1CASE(64)
#undef K1CASE
    return cudaErrorInvalidValue;
}

template <typename KeyT, bool PERM, int NT, bool ITEMS = false>
cudaError_t launch_k3_pass(const Plan& p, void* ws, const Layout& L, KeyT* out_keys, uint32_t* out_perm, cudaStream_t s,
                           bool secondary, bool to_mid, uint32_t cap, size_t smem, int grid,
                           const unsigned long long* rbase, bool premid = false) {
    auto kern = k3_local_sort<KeyT, PERM, NT, ITEMS>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    K3LParams kp;
    kp.capc = p.capc;
    kp.num_coarse = p.C;
    kp.kfine = p.kfine;
    kp.cap = cap;
    kp.secondary = secondary ? 1u : 0u;
    kp.to_mid = to_mid ? 1u : 0u;
    kp.item_cap = p.item_cap;
    kp.premid = premid ? 1u : 0u;
    {   // the coarse-bucket passes merge rank-bucket pairs (fine id >> 1: ~2 keys per rank bucket
        // at B = N): C2 K3 0.416 -> 0.390 ms (>> 2: 0.508, >> 3: 0.731; profiles/r02/k3_fshift.log).
        // MLSORT_K3_FSHIFT=k overrides (experiments).
        const char* e = std::getenv("MLSORT_K3_FSHIFT");
        kp.fshift = e ? (uint32_t)std::atoi(e) : (p.kfine >= 4096 ? 1u : 0u);
    }
    {   // key-only f32, primary pass, at most ~1 key per rank bucket: position-based fix-up (step 4p
        // of k3_local.cuh) on unmerged rank buckets, in both passes (the secondary pass holds the
        // overloaded coarse buckets, whose longer rank buckets fall back to the walk more often;
        // still faster: profiles/r02/ab_k3_posfix.log).  MLSORT_K3_POSFIX=0/1/2 overrides.
        const char* e = std::getenv("MLSORT_K3_POSFIX");
        const bool fit = !PERM && !ITEMS && sizeof(KeyT) == 4 &&
                         (double)p.n <= 1.001 * (double)p.C * (double)p.kfine;
        const int pv = e ? std::atoi(e) : 2;       // 1: the primary pass only (experiments)
        kp.posfix = fit && (pv >= 2 || (pv == 1 && !secondary)) ? 1u : 0u;
        kp.tails_first = !ITEMS && !secondary && !std::getenv("MLSORT_K3_NO_TAILS_FIRST") ? 1u : 0u;
        if (kp.posfix && !std::getenv("MLSORT_K3_FSHIFT")) kp.fshift = 0u;
    }
    DevStatus* st = at<DevStatus>(ws, L.status);
    unsigned long long* ticket = ITEMS ? &st->ticket3d : (secondary ? &st->ticket3b : &st->ticket3);
    kern<<<grid, NT, smem, s>>>(kp, at<KeyT>(ws, L.reg_keys), at<uint16_t>(ws, L.reg_fine),
                                PERM ? at<uint32_t>(ws, L.reg_idx) : nullptr, at<unsigned long long>(ws, L.starts),
                                out_keys, out_perm, at<unsigned long long>(ws, L.range_start), st,
                                at<uint32_t>(ws, L.big_list), at<uint32_t>(ws, L.big_mark), at<uint32_t>(ws, L.mid_list),
                                ticket, rbase, at<K3Item>(ws, L.items));
    return cudaGetLastError();
}

// Coarse buckets too large for the K3 passes: k3_cut splits them into items (and copies giant
// rank buckets to their output ranges), then the round pass sorts the items (k3_big.cuh).
template <typename KeyT, bool PERM>
cudaError_t launch_k3_big(const Plan& p, void* ws, const Layout& L, KeyT* out_keys, uint32_t* out_perm,
                          cudaStream_t s, const unsigned long long* rbase) {
    auto cut = k3_cut<KeyT, PERM>;
    uint32_t gshift = 0;
    while ((p.kfine >> gshift) > kCutGroups) ++gshift;
    const size_t smem = (size_t)(2 * (p.kfine >> gshift) + 2) * 4;
    cudaError_t e = set_smem(cut, smem);
    if (e != cudaSuccess) return e;
    K3CutParams cp;
    cp.capc = p.capc;
    cp.kfine = p.kfine;
    cp.cap = p.cap;
    cp.item_cap = p.item_cap;
    cp.seg_cap = p.seg_cap;
    cp.gshift = gshift;
    cut<<<std::min<int>(num_sms(), (int)p.C), kCutThreads, smem, s>>>(
        cp, at<KeyT>(ws, L.reg_keys), at<uint16_t>(ws, L.reg_fine), PERM ? at<uint32_t>(ws, L.reg_idx) : nullptr,
        at<unsigned long long>(ws, L.starts), at<uint32_t>(ws, L.big_list), at<DevStatus>(ws, L.status),
        at<K3Item>(ws, L.items), at<K3Seg>(ws, L.k3segs), out_keys, out_perm, at<unsigned long long>(ws, L.range_start),
        rbase);
    e = cudaGetLastError();
    if (std::getenv("MLSORT_SYNC_DEBUG")) {
        e = cudaStreamSynchronize(s);
        fprintf(stderr, "mlsort: k3_cut -> %s\n", cudaGetErrorString(e));
    }
    if (e != cudaSuccess) return e;
    e = launch_k3_pass<KeyT, PERM, kL3ThreadsBig, true>(p, ws, L, out_keys, out_perm, s, false, false, p.cap,
                                                         p.k3_smem, num_sms(), rbase);
    if (std::getenv("MLSORT_SYNC_DEBUG")) {
        e = cudaStreamSynchronize(s);
        fprintf(stderr, "mlsort: k3 rounds -> %s\n", cudaGetErrorString(e));
    }
    return e;
}

// Auxiliary stream and fork/join events of the concurrent K3 passes, per (thread, device).
struct ForkStreams {
    int dev = -1;
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
ForkStreams& fork_streams() {
    thread_local std::vector<ForkStreams> all;
    int dev = 0;
    cudaGetDevice(&dev);
    for (auto& f : all)
        if (f.dev == dev) return f;
    ForkStreams f;
    f.dev = dev;
    if (cudaStreamCreateWithFlags(&f.aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming) != cudaSuccess)
        f.aux = nullptr;
    all.push_back(f);
    return all.back();
}

// K3 local plan: primary pass (two 512-thread CTAs per SM, capacity cap1) over every coarse
// bucket, then the secondary pass (one 1024-thread CTA per SM, capacity cap) over the buckets
// the primary pass handed over.
template <typename KeyT, bool PERM>
cudaError_t launch_k3_local(const Plan& p, void* ws, const Layout& L, KeyT* out_keys, uint32_t* out_perm,
                            cudaStream_t s, const unsigned long long* rbase) {
    cudaError_t e;
    if (p.cap1 > 0) {
        // K2 listed the coarse buckets above cap1, so the secondary pass (one 1024-thread CTA per
        // SM) runs on a forked stream concurrently with the primary pass: the large buckets
        // start first and the primary pass's CTAs fill every SM they free, instead of the
        // secondary pass running alone after the primary pass's tail
        ForkStreams& fk = fork_streams();
        if (!fk.aux) return cudaErrorNotReady;
        e = cudaEventRecord(fk.fork, s);
        if (e != cudaSuccess) return e;
        e = cudaStreamWaitEvent(fk.aux, fk.fork, 0);
        if (e != cudaSuccess) return e;
        e = launch_k3_pass<KeyT, PERM, kL3ThreadsBig>(p, ws, L, out_keys, out_perm, fk.aux, true, false,
                                                      p.cap, p.k3_smem, num_sms(), rbase);
        if (e != cudaSuccess) return e;
        e = cudaEventRecord(fk.join, fk.aux);
        if (e != cudaSuccess) return e;
        e = launch_k3_pass<KeyT, PERM, kL3Threads>(p, ws, L, out_keys, out_perm, s, false, true, p.cap1,
                                                   p.k3_smem1, std::min<int>(2 * num_sms(), (int)p.C), rbase,
                                                   true);
        if (e != cudaSuccess) return e;
        e = cudaStreamWaitEvent(s, fk.join, 0);
    } else {
        e = launch_k3_pass<KeyT, PERM, kL3ThreadsBig>(p, ws, L, out_keys, out_perm, s, false, false,
                                                      p.cap, p.k3_smem, std::min<int>(num_sms(), (int)p.C), rbase);
    }
    if (std::getenv("MLSORT_SYNC_DEBUG")) {
        e = cudaStreamSynchronize(s);
        fprintf(stderr, "mlsort: k3 passes -> %s\n", cudaGetErrorString(e));
    }
    if (e != cudaSuccess) return e;
    return launch_k3_big<KeyT, PERM>(p, ws, L, out_keys, out_perm, s, rbase);
}

template <typename KeyT, bool PERM>
cudaError_t launch_k3(const Plan& p, void* ws, const Layout& L, KeyT* out_keys, uint32_t* out_perm, cudaStream_t s,
                      const unsigned long long* rbase) {
    return launch_k3_local<KeyT, PERM>(p, ws, L, out_keys, out_perm, s, rbase);
}

// Stable LSD radix sort of (ord bits, payload) pairs, n elements, in the radix area.
// Passes over the payload digits first when `payload_first` (restores input order),
// then over the key digits.  Returns the buffer index (0/1) holding the result.
template <typename Bits>
int radix_sort_pairs(Bits* k0, uint32_t* v0, Bits* k1, uint32_t* v1, uint32_t* ghist, uint64_t n,
                     bool payload_first, cudaStream_t s, Launches& nl, cudaError_t& err, bool skip_keys = false,
                     int key_bits = (int)(sizeof(Bits) * 8)) {
    const uint32_t nchunks = (uint32_t)((n + kRadixChunk - 1) / kRadixChunk);
    int cur = 0;
    err = set_smem(k_radix_scatter<Bits>, radix_scatter_smem<Bits>());
    if (err != cudaSuccess) return 0;
    auto pass = [&](int field, int shift) {
        Bits* ki = cur ? k1 : k0;
        uint32_t* vi = cur ? v1 : v0;
        Bits* ko = cur ? k0 : k1;
        uint32_t* vo = cur ? v0 : v1;
        k_radix_hist<Bits><<<nchunks, kRadixThreads, 0, s>>>(ki, vi, n, field, shift, nchunks, ghist);
        {   // digit-major exclusive scan of the chunk histograms
            const uint64_t m = (uint64_t)nchunks * 256;
            const uint32_t nt = (uint32_t)((m + kScanTile - 1) / kScanTile);
            if (nt <= 1) {
                k_radix_scan<<<1, 1024, 0, s>>>(ghist, m);
            } else {
                uint32_t* tot = ghist + m;                 // scratch after the histograms
                k_scan_blocks<<<nt, 1024, 0, s>>>(ghist, m, tot);
                k_radix_scan<<<1, 1024, 0, s>>>(tot, nt);
                k_scan_add<<<nt, 256, 0, s>>>(ghist, m, tot);
                nl.count += 2;
            }
        }
        k_radix_scatter<Bits><<<nchunks, kRadixThreads, radix_scatter_smem<Bits>(), s>>>(ki, vi, ko, vo, n, field, shift,
                                                                                        nchunks, ghist);
        nl.count += 3;
        cur ^= 1;
    };
    if (payload_first && v0)
        for (int sh = 0; sh < 32; sh += 8) pass(1, sh);
    if (!skip_keys)
        for (int sh = 0; sh < key_bits; sh += 8) pass(0, sh);
    err = cudaGetLastError();
    return cur;
}

int grid_for(uint64_t n, int threads) {
    uint64_t g = (n + threads - 1) / threads;
    return (int)std::min<uint64_t>(std::max<uint64_t>(g, 1), (uint64_t)num_sms() * 16);
}

// Sort segment [S0, S0+len) of (out_keys, out_perm) by (key, index) with the radix area.
template <typename KeyT, bool PERM>
int radix_segment(KeyT* out_keys, uint32_t* out_perm, uint64_t S0, uint64_t len, bool keys_equal,
                  void* ws, const Layout& L, cudaStream_t s, Launches& nl) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    char* base = at<char>(ws, L.radix);
    Bits* k0 = reinterpret_cast<Bits*>(base);
    Bits* k1 = reinterpret_cast<Bits*>(base + align_up(len * sizeof(Bits)));
    uint32_t* v0 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(len * sizeof(Bits))) : nullptr;
    uint32_t* v1 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(len * sizeof(Bits)) + align_up(len * 4)) : nullptr;
    uint32_t* gh = reinterpret_cast<uint32_t*>(base + 2 * align_up(len * sizeof(Bits)) + (PERM ? 2 * align_up(len * 4) : 0));
    k_to_ord<KeyT><<<grid_for(len, 256), 256, 0, s>>>(out_keys + S0, k0, nullptr, len, 0);
    if (PERM) CK(cudaMemcpyAsync(v0, out_perm + S0, len * 4, cudaMemcpyDeviceToDevice, s));
    cudaError_t err;
    int cur = radix_sort_pairs<Bits>(k0, v0, k1, v1, gh, len, PERM, s, nl, err, keys_equal);
    if (err != cudaSuccess) return MLSORT_ERR_CUDA;
    k_from_ord<KeyT><<<grid_for(len, 256), 256, 0, s>>>(cur ? k1 : k0, out_keys + S0, len);
    if (PERM) CK(cudaMemcpyAsync(out_perm + S0, cur ? v1 : v0, len * 4, cudaMemcpyDeviceToDevice, s));
    nl.count += 2;
    CK(cudaGetLastError());
    return MLSORT_OK;
}

// Whole-input conventional sort (fallback): stable radix sort of (key, iota).
template <typename KeyT, bool PERM>
int fallback_sort(const KeyT* keys, uint64_t n, KeyT* out_keys, uint32_t* out_perm, void* ws, const Layout& L,
                  cudaStream_t s, Launches& nl) {
    using Bits = typename KeyTraits<KeyT>::Bits;
    char* base = at<char>(ws, L.radix);
    Bits* k0 = reinterpret_cast<Bits*>(base);
    Bits* k1 = reinterpret_cast<Bits*>(base + align_up(n * sizeof(Bits)));
    uint32_t* v0 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits))) : nullptr;
    uint32_t* v1 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits)) + align_up(n * 4)) : nullptr;
    uint32_t* gh = reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits)) + (PERM ? 2 * align_up(n * 4) : 0));
    k_to_ord<KeyT><<<grid_for(n, 256), 256, 0, s>>>(keys, k0, v0, n, 0);
    cudaError_t err;
    int cur = radix_sort_pairs<Bits>(k0, v0, k1, v1, gh, n, false, s, nl, err);
    if (err != cudaSuccess) return MLSORT_ERR_CUDA;
    k_from_ord<KeyT><<<grid_for(n, 256), 256, 0, s>>>(cur ? k1 : k0, out_keys, n);
    if (PERM) CK(cudaMemcpyAsync(out_perm, cur ? v1 : v0, n * 4, cudaMemcpyDeviceToDevice, s));
    nl.count += 2;
    CK(cudaGetLastError());
    return MLSORT_OK;
}

K1Params k1_params(const Weights& w, const Plan& p, uint64_t B, bool f32, const FoldedWeights* fw = nullptr) {
    K1Params kp;
    kp.u_cl_lo = fw ? fw->u_cl_lo : -INFINITY;
    kp.u_cl_hi = fw ? fw->u_cl_hi : INFINITY;
    kp.lo_d = w.lo;
    kp.hi_d = w.hi;
    kp.x0_d = origin_of(w, f32);
    kp.x0_f = (float)kp.x0_d;
    {   // f32 tail thresholds: smallest float >= lo, largest float <= hi
        float lf = (float)w.lo, hf = (float)w.hi;
        if ((double)lf < w.lo) lf = std::nextafter(lf, INFINITY);
        if ((double)hf > w.hi) hf = std::nextafter(hf, -INFINITY);
        kp.lo_tf = lf;
        kp.hi_tf = hf;
    }
    kp.bm.Bf = (float)B;
    kp.bm.Bm1 = (uint32_t)(B - 1);
    kp.bm.B = B;
    kp.bm.S = fxp_shift(w);
    kp.bm.pow2 = (B & (B - 1)) == 0 && B <= (1ull << 32) ? 1u : 0u;
    kp.bm.sh = (int32_t)kp.bm.S - (int32_t)ceil_log2(B);
    kp.bm.half = kp.bm.sh > 0 ? (1 << (kp.bm.sh - 1)) : 0;
    kp.fine_bits = p.fb;
    kp.num_coarse = p.C;
    kp.num_tiles = p.T;
    kp.tile0 = 0;
    kp.flags = p.ws_stage ? kK1StageKeys : 0u;
    kp.capc = p.capc;
    kp.n = p.n;
    return kp;
}

// Chunked input arrival (mlsort_sort_host): K1 is launched per chunk of tiles after the chunk's
// host-to-device copy has completed (event), so the copy of chunk i+1 overlaps K1 on chunk i.
struct ChunkPlan {
    int n = 0;
    uint32_t tile_begin[16] = {}, tile_end[16] = {};
    cudaEvent_t ready[16] = {};
};

// The core pipeline shared by mlsort_sort (predict) and mlsort_sort_records (GIVEN buckets).
struct PhaseTimer {
    // events are created once per (thread, device) and reused: creating and destroying them per
    // call would put ~12 driver calls of host time into every timed sort
    bool on = false;
    cudaEvent_t* ev = nullptr;
    int n = 0;
    cudaStream_t s = nullptr;
    void start(bool enable, cudaStream_t st) {
        on = false;
        if (!enable) return;
        struct Pool {
            int dev;
            cudaEvent_t ev[6];
        };
        thread_local std::vector<Pool> pools;
        int dev = 0;
        cudaGetDevice(&dev);
        for (auto& p : pools)
            if (p.dev == dev) ev = p.ev;
        if (!ev) {
            Pool p;
            p.dev = dev;
            for (auto& e : p.ev)
                if (cudaEventCreate(&e) != cudaSuccess) return;
            pools.push_back(p);
            ev = pools.back().ev;
        }
        on = true;
        s = st;
        cudaEventRecord(ev[0], s);
        n = 1;
    }
    void mark() {
        if (on && n < 6) cudaEventRecord(ev[n++], s);
    }
    void finish(mlsort_info* info) {   // after the stream was synchronised
        if (!on) return;
        if (info) {
            for (int i = 1; i < n; ++i) cudaEventElapsedTime(&info->phase_ms[i - 1], ev[i - 1], ev[i]);
            cudaEventElapsedTime(&info->phase_ms[5], ev[0], ev[n - 1]);
        }
        on = false;
    }
};

template <typename KeyT>
cudaError_t launch_k0(const Plan& p, const KeyT* keys, uint32_t mpad, const FoldedWeights& fw, const K1Params& kp,
                      void* ws, const Layout& L, cudaStream_t s) {
    const size_t smem = (size_t)p.C * 4;
    const uint64_t ns = (p.n + p.stride - 1) / p.stride;
    const int grid = (int)std::min<uint64_t>((uint64_t)num_sms() * 2, (ns + 2047) / 2048 + 1);
    cudaError_t e = cudaSuccess;
#define K0CASE(M)                                                                                          \
    if (mpad == M) {                                                                                       \
        e = set_smem(k0_sample<KeyT, M>, smem);                                                            \
        if (e != cudaSuccess) return e;                                                                    \
        k0_sample<KeyT, M><<<grid, 256, smem, s>>>(keys, p.n, p.stride, fw, kp, at<uint32_t>(ws, L.est));  \
    }
    K0CASE(16) K0CASE(32) K0CASE(64)
#undef K0CASE
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k0_regions<<<1, 1024, 0, s>>>(at<uint32_t>(ws, L.est), p.C, p.stride, (unsigned long long)p.area,
                                  at<unsigned long long>(ws, L.rbase));
    return cudaGetLastError();
}

// ---------------------------------------------------------------- CUDA graph of one call
// Key of a captured launch sequence: every argument the kernels of the first attempt see.
struct GraphKey {
    const void* keys;
    const void* out_keys;
    const void* out_perm;
    const void* ws;
    uint64_t n, B, wserial;
    int pred;
    uint32_t mpad;
    int dev;
    bool operator==(const GraphKey& o) const {
        return keys == o.keys && out_keys == o.out_keys && out_perm == o.out_perm && ws == o.ws && n == o.n &&
               B == o.B && wserial == o.wserial && pred == o.pred && mpad == o.mpad && dev == o.dev;
    }
};

// Replay the graph captured for key k on stream s, capturing it first (on a private stream: the
// caller's may be the legacy default stream, which cannot capture) when it is new.  Per thread
// (the captured status read targets this thread's pinned status word) and per template
// instantiation; a small LRU.  *done = false leaves the work to the direct launches (graphs
// disabled by MLSORT_NO_GRAPH, or a capture that failed, remembered per key).
template <typename Enqueue>
int graph_run(GraphKey k, cudaStream_t s, Enqueue&& enqueue, uint64_t* launches, bool* done) {
    *done = false;
    static const bool disabled = std::getenv("MLSORT_NO_GRAPH") != nullptr;
    if (disabled) return MLSORT_OK;
    struct Entry {
        GraphKey k;
        cudaGraphExec_t exec;     // nullptr: capture failed, launch directly
        uint64_t launches;
    };
    struct Cap {
        int dev;
        cudaStream_t cs;
    };
    thread_local std::vector<Entry> cache;
    thread_local std::vector<Cap> caps;
    cudaGetDevice(&k.dev);
    for (size_t i = 0; i < cache.size(); ++i) {
        if (cache[i].k == k) {
            Entry e = cache[i];
            cache.erase(cache.begin() + i);
            cache.push_back(e);                               // most recent last
            if (!e.exec) return MLSORT_OK;
            CK(cudaGraphLaunch(e.exec, s));
            *launches += e.launches;
            *done = true;
            return MLSORT_OK;
        }
    }
    cudaStream_t cs = nullptr;
    for (auto& c : caps)
        if (c.dev == k.dev) cs = c.cs;
    if (!cs) {
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        caps.push_back(Cap{k.dev, cs});
    }
    Entry e{k, nullptr, 0};
    cudaGraph_t g = nullptr;
    uint64_t before = *launches;
    bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        ok = enqueue(cs) == MLSORT_OK;
        ok = (cudaStreamEndCapture(cs, &g) == cudaSuccess) && ok && g;
    }
    if (ok) ok = cudaGraphInstantiate(&e.exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();                                        // clear a failed capture's error
    e.launches = *launches - before;
    *launches = before;
    if (!ok) e.exec = nullptr;
    if (cache.size() >= 8) {
        if (cache.front().exec) cudaGraphExecDestroy(cache.front().exec);
        cache.erase(cache.begin());
    }
    cache.push_back(e);
    if (!e.exec) return MLSORT_OK;
    CK(cudaGraphLaunch(e.exec, s));
    *launches += e.launches;
    *done = true;
    return MLSORT_OK;
}

template <typename KeyT, bool PERM, bool GIVEN>
int run_pipeline(const KeyT* keys, uint64_t n, uint64_t B, const Weights* w, int pred, KeyT* out_keys,
                 uint32_t* out_perm, void* ws, uint64_t ws_bytes, cudaStream_t s, mlsort_info* info,
                 const uint32_t* bucket_in, const uint32_t* idx_in, uint32_t b_lo, bool timing = false,
                 bool verify_all = false, const ChunkPlan* chunks = nullptr) {
    NvtxRange nvtx_call("mlsort_sort");
    Launches nl;
    PhaseTimer tm;
    const bool group = !GIVEN && pred == kPredSkip;
    const Plan p = make_plan(n, B, sizeof(KeyT), PERM, !GIVEN, group);
    const Layout L = make_layout(p);
    if (ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) % kAlign)) return MLSORT_ERR_WORKSPACE;
    FoldedWeights fw;
    uint32_t mpad = 16;
    K1Params kp;
    if (!GIVEN) {
        mpad = mpad_of(w->m);
        fw = fold_cached(*w, mpad, sizeof(KeyT) == 4);
        kp = k1_params(*w, p, B, sizeof(KeyT) == 4, &fw);
    } else {
        std::memset(&fw, 0, sizeof(fw));
        Weights dummy;
        dummy.lo = 0;
        dummy.hi = 1;
        kp = k1_params(dummy, p, B, sizeof(KeyT) == 4);
        kp.lo_d = -INFINITY;
        kp.hi_d = INFINITY;
    }
    if (pred != kPredMufu && pred != kPredMixed) pred = kPredPacked;
    tm.start(timing, s);
    DevStatus* dst = at<DevStatus>(ws, L.status);
    DevStatus* hs = host_status();
    DevStatus st;
    const unsigned long long* rbase = nullptr;   // regions at c * capc; K0-sized or exact (retry) layouts
    const uint64_t nranges = (uint64_t)p.C * p.R;
    if (p.local && p.cap1 > 0) fork_streams();       // (created outside any graph capture)
    // One attempt's device work, from the status reset to the status read, enqueued on q (the
    // caller's stream, or the capture stream of the graph path below).
    auto enqueue = [&](cudaStream_t q, int attempt) -> int {
        // one launch resets the status word, the range starts, the big marks and the cursors
        k0_init<<<(unsigned)std::max<uint64_t>(1, (std::max<uint64_t>(nranges, p.C) + 255) / 256), 256, 0, q>>>(
            dst, at<unsigned long long>(ws, L.range_start), nranges, at<uint32_t>(ws, L.big_mark),
            at<uint32_t>(ws, L.cursor), p.C, (p.sampled && attempt == 0) ? at<uint32_t>(ws, L.est) : nullptr);
        CK(cudaGetLastError());
        if (!GIVEN && p.sampled && attempt == 0) {        // K0: regions from a sample of the buckets
            if (chunks)                                   // (the sample spans every chunk)
                for (int i = 0; i < chunks->n; ++i) CK(cudaStreamWaitEvent(q, chunks->ready[i], 0));
            CK((launch_k0<KeyT>(p, keys, mpad, fw, kp, ws, L, q)));
            rbase = at<unsigned long long>(ws, L.rbase);
            nl.count += 2;
        }

        if (chunks && chunks->n > 0) {
            for (int i = 0; i < chunks->n; ++i) {
                CK(cudaStreamWaitEvent(q, chunks->ready[i], 0));
                K1Params kc = kp;
                kc.tile0 = chunks->tile_begin[i];
                kc.num_tiles = chunks->tile_end[i] - chunks->tile_begin[i];
                if (kc.num_tiles == 0) continue;
                CK((launch_k1<KeyT, PERM, GIVEN>(p, keys, mpad, pred, fw, kc, ws, L, q, bucket_in, idx_in, b_lo, rbase)));
                nl.count += 1;
            }
            nl.count -= 1;   // counted once below
        } else {
            NvtxRange r("mlsort K1 predict + partition");
            CK((launch_k1<KeyT, PERM, GIVEN>(p, keys, mpad, pred, fw, kp, ws, L, q, bucket_in, idx_in, b_lo, rbase)));
        }
        tm.mark();
        k2_coarse_starts<<<1, 1024, 0, q>>>(at<uint32_t>(ws, L.cursor), p.C, at<unsigned long long>(ws, L.starts),
                                            n < (1ull << 31), p.local ? p.cap1 : 0u, at<uint32_t>(ws, L.mid_list),
                                            dst);
        CK(cudaGetLastError());
        tm.mark();
        // K3 checks the adjacent order of every coarse bucket it sorts (reading A14) for every
        // model, fused with its store; K5 checks every coarse-bucket boundary.
        {
            NvtxRange r("mlsort K3 (passes, cut, rounds)");
            CK((launch_k3<KeyT, PERM>(p, ws, L, out_keys, out_perm, q, rbase)));
        }
        if (PERM) {     // giant all-equal runs: order their indices (k3_big.cuh; regions are dead now)
            k3_index_sort<512><<<num_sms() * 3, 512, 0, q>>>(at<K3Seg>(ws, L.k3segs), p.seg_cap, out_perm,
                                                     at<uint32_t>(ws, L.radix), dst);
            CK(cudaGetLastError());
        }
        tm.mark();
        tm.mark();
        k5_verify_all<KeyT, PERM><<<(unsigned)std::max<uint64_t>(num_sms() * 2, std::min<uint64_t>((nranges + 255) / 256,
                                                                                              num_sms() * 8)),
                                    256, 0, q>>>(at<unsigned long long>(ws, L.range_start), nranges,
                                                 at<K3Item>(ws, L.items), at<K3Seg>(ws, L.k3segs), out_keys,
                                                 out_perm, dst, p.item_cap, p.seg_cap, n);
        CK(cudaGetLastError());
        tm.mark();
        nl.count += 6 + (p.cap1 > 0 ? 1 : 0) + (PERM ? 1 : 0);

        CK(cudaMemcpyAsync(hs, dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, q));
        return MLSORT_OK;
    };
    for (int attempt = 0;; ++attempt) {
        // The first attempt of an untimed call runs as a CUDA graph captured once per launch
        // configuration (pointers, sizes, weights): one graph launch instead of ~8 kernel launches
        // and their host-side latency in front of the device work (graph_run).
        bool done = false;
        if (attempt == 0 && !timing && !chunks && !GIVEN) {
            const GraphKey gk{keys, out_keys, out_perm, ws, n, B, GIVEN ? 0ull : w->serial, pred, mpad, 0};
            const int rc = graph_run(gk, s, [&](cudaStream_t q) { return enqueue(q, 0); }, &nl.count, &done);
            if (rc != MLSORT_OK) return rc;
            if (done && p.sampled) rbase = at<unsigned long long>(ws, L.rbase);
        }
        if (!done) {
            const int rc = enqueue(s, attempt);
            if (rc != MLSORT_OK) return rc;
        }
        CK(cudaStreamSynchronize(s));
        st = *hs;
        if (info) {
            info->num_coarse = p.C;
            info->tail_lo = st.tail_lo;
            info->tail_hi = st.tail_hi;
            info->max_coarse = st.max_coarse;
            info->big_buckets = st.big_count;
        }
        // A region overflowed (the data's coarse-bucket sizes are more skewed than the region
        // capacity allows): the cursors now hold the exact bucket sizes, so lay the regions out
        // exactly (16-B aligned starts) and run the pipeline once more.
        if (st.region_overflow > 0 && attempt == 0 && st.bad_index == ~0ull) {
            std::vector<uint32_t> sizes(p.C);
            CK(cudaMemcpy(sizes.data(), at<uint32_t>(ws, L.cursor), (size_t)p.C * 4, cudaMemcpyDeviceToHost));
            std::vector<unsigned long long> rb(p.C + 1);
            unsigned long long off = 0;
            for (uint32_t c = 0; c < p.C; ++c) {
                rb[c] = off;
                off += ((unsigned long long)sizes[c] + 7ull) & ~7ull;
            }
            rb[p.C] = off;
            if (off <= p.area) {
                unsigned long long* d_rb = at<unsigned long long>(ws, L.rbase);
                CK(cudaMemcpyAsync(d_rb, rb.data(), (size_t)(p.C + 1) * 8, cudaMemcpyHostToDevice, s));
                CK(cudaStreamSynchronize(s));          // (the host vectors die at scope end)
                rbase = d_rb;
                continue;
            }
        }
        break;
    }
    tm.finish(info);
    if (st.bad_index != ~0ull) {
        if (info) info->bad_index = (int64_t)st.bad_index;
        return MLSORT_ERR_NONFINITE_KEY;
    }
    // K5 boundary violations plus violations found inside cluster-K3 slices
    uint64_t violations = st.violations + st.k3_violations;
    if (st.region_overflow > 0) violations += 1;   // a region was full: use the conventional sort
    if (st.item_overflow > 0) violations += 1;     // (lists sized for the worst case: not expected)
    std::vector<K3Seg> ks;
    if (st.region_overflow == 0 && st.seg_count > 0) {
        // segments left for the radix pass: distinct keys, or runs k3_index_sort flagged (pad)
        const uint64_t nseg_dev = std::min<uint64_t>(st.seg_count, p.seg_cap);
        ks.resize(nseg_dev);
        CK(cudaMemcpyAsync(ks.data(), at<K3Seg>(ws, L.k3segs), nseg_dev * sizeof(K3Seg), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ks.erase(std::remove_if(ks.begin(), ks.end(), [](const K3Seg& g) { return PERM && g.pad == 0u && (g.flags & 1u); }),
                 ks.end());
    }
    const bool need_radix = !ks.empty();
    if (need_radix) {   // the stable radix pass over the runs K3 could not sort (k3_cut segments)
        NvtxRange r("mlsort radix segments");
        std::vector<unsigned long long> seg;
        uint64_t tot = 0;
        bool all_equal = true;
        std::sort(ks.begin(), ks.end(), [](const K3Seg& a, const K3Seg& b) { return a.out < b.out; });
        for (const K3Seg& g : ks) {
            all_equal &= (g.flags & 1u) != 0;
            seg.push_back(g.out);
            seg.push_back(tot);
            seg.push_back(g.len);
            tot += g.len;
        }
        if (tot > 0) {
            using Bits = typename KeyTraits<KeyT>::Bits;
            const uint32_t nseg = (uint32_t)(seg.size() / 3);
            unsigned long long* d_seg = at<unsigned long long>(ws, L.segs);
            CK(cudaMemcpyAsync(d_seg, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, s));
            char* rbase = at<char>(ws, L.radix);
            Bits* k0 = reinterpret_cast<Bits*>(rbase);
            Bits* k1 = reinterpret_cast<Bits*>(rbase + align_up(tot * sizeof(Bits)));
            uint32_t* v0 = PERM ? reinterpret_cast<uint32_t*>(rbase + 2 * align_up(tot * sizeof(Bits))) : nullptr;
            uint32_t* v1 = PERM ? reinterpret_cast<uint32_t*>(rbase + 2 * align_up(tot * sizeof(Bits)) + align_up(tot * 4)) : nullptr;
            uint32_t* gh = reinterpret_cast<uint32_t*>(rbase + 2 * align_up(tot * sizeof(Bits)) + (PERM ? 2 * align_up(tot * 4) : 0));
            const int sg = (int)std::min<uint32_t>(nseg, (uint32_t)num_sms() * 8);
            cudaError_t err;
            if (PERM && all_equal && nseg > 1) {
                // every run is all-equal: only the indices inside each run need ordering, so the
                // radix key is the run's ordinal (its keys are already in place) -- 4 index passes
                // plus ceil(log2(runs)/8) ordinal passes instead of 4 + 8*sizeof(key) / 8
                k_seg_gather_ordinal<Bits><<<sg, 256, 0, s>>>(d_seg, nseg, out_perm, k0, v0);
                int bits = 0;
                while ((1ull << bits) < nseg) ++bits;
                int cur = radix_sort_pairs<Bits>(k0, v0, k1, v1, gh, tot, true, s, nl, err, false, bits);
                if (err != cudaSuccess) return MLSORT_ERR_CUDA;
                k_seg_scatter_perm<<<sg, 256, 0, s>>>(d_seg, nseg, cur ? v1 : v0, out_perm);
            } else {
                k_seg_gather<KeyT><<<sg, 256, 0, s>>>(d_seg, nseg, out_keys, out_perm, k0, v0);
                // a single all-equal perm run only needs its indices ordered
                const bool skip_keys = all_equal && nseg == 1;
                int cur = radix_sort_pairs<Bits>(k0, v0, k1, v1, gh, tot, PERM, s, nl, err, skip_keys);
                if (err != cudaSuccess) return MLSORT_ERR_CUDA;
                k_seg_scatter<KeyT><<<sg, 256, 0, s>>>(d_seg, nseg, cur ? k1 : k0, cur ? v1 : v0, out_keys, out_perm);
            }
            CK(cudaGetLastError());
            nl.count += 2;
        }
        // re-verify every boundary now that all ranges are final
        CK(cudaMemsetAsync(&dst->violations, 0, 8, s));
        k5_boundary_verify<KeyT, PERM><<<(unsigned)((nranges + 255) / 256), 256, 0, s>>>(
            at<unsigned long long>(ws, L.range_start), nranges, out_keys, out_perm, dst);
        k5_item_verify<KeyT, PERM><<<num_sms() * 2, 256, 0, s>>>(at<K3Item>(ws, L.items), at<K3Seg>(ws, L.k3segs),
                                                                 out_keys, out_perm, dst, p.item_cap, p.seg_cap, n);
        CK(cudaMemcpyAsync(hs, dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        // the first K5 pass ran before the overflow buckets were sorted: only the fresh boundary
        // check counts, together with the slice-internal K3 violations
        violations = st.k3_violations + hs->violations + (st.region_overflow > 0 ? 1 : 0) +
                     (st.item_overflow > 0 ? 1 : 0);
    }
    if (std::getenv("MLSORT_DEBUG"))
        fprintf(stderr, "mlsort: plan C=%u fb=%u R=%u local=%d ws=%d group=%d cap=%u cap1=%u | k5=%llu k3=%llu "
                "region_overflow=%llu overflow=%llu big=%llu local_repairs=%llu posfix_fallbacks=%llu -> violations=%llu\n",
                p.C, p.fb, p.R, (int)p.local, (int)p.ws, (int)p.ws_group, p.cap, p.cap1, st.violations,
                st.k3_violations, st.region_overflow, st.overflow, st.big_count, st.local_repairs, st.posfix_fallbacks,
                (unsigned long long)violations);
    if (info) info->repairs = violations + st.local_repairs;
    if (violations > 0) {   // reading A14: escalate to the conventional sort
        if (GIVEN) {
            // records path: sort (key, global index) pairs of the received records
            using Bits = typename KeyTraits<KeyT>::Bits;
            char* base = at<char>(ws, L.radix);
            Bits* k0 = reinterpret_cast<Bits*>(base);
            Bits* k1 = reinterpret_cast<Bits*>(base + align_up(n * sizeof(Bits)));
            uint32_t* v0 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits))) : nullptr;
            uint32_t* v1 = PERM ? reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits)) + align_up(n * 4)) : nullptr;
            uint32_t* gh = reinterpret_cast<uint32_t*>(base + 2 * align_up(n * sizeof(Bits)) + (PERM ? 2 * align_up(n * 4) : 0));
            k_to_ord<KeyT><<<grid_for(n, 256), 256, 0, s>>>(keys, k0, nullptr, n, 0);
            if (PERM) CK(cudaMemcpyAsync(v0, idx_in, n * 4, cudaMemcpyDeviceToDevice, s));
            cudaError_t err;
            int cur = radix_sort_pairs<Bits>(k0, v0, k1, v1, gh, n, PERM, s, nl, err);
            if (err != cudaSuccess) return MLSORT_ERR_CUDA;
            k_from_ord<KeyT><<<grid_for(n, 256), 256, 0, s>>>(cur ? k1 : k0, out_keys, n);
            if (PERM) CK(cudaMemcpyAsync(out_perm, cur ? v1 : v0, n * 4, cudaMemcpyDeviceToDevice, s));
        } else {
            int rc = fallback_sort<KeyT, PERM>(keys, n, out_keys, out_perm, ws, L, s, nl);
            if (rc) return rc;
        }
        CK(cudaStreamSynchronize(s));
        if (info) info->fallback_used = 1;
    }
    if (info) info->kernel_launches = nl.count;
    return MLSORT_OK;
}

// Large enough for both plan flavours (predicting sorts may use k1_ws, the records path not).
uint64_t workspace_bytes(uint64_t n, mlsort_dtype dt, uint64_t B, bool perm) {
    const size_t ks = dt == MLSORT_F32 ? 4 : 8;
    return std::max(make_layout(make_plan(n, B, ks, perm, true)).total,
                    make_layout(make_plan(n, B, ks, perm, false)).total);
}

}  // namespace MLSORT_LOCAL

// ==================================================================== translation-unit split
// run_pipeline<KeyT, PERM, GIVEN> holds almost all kernel instantiations; build.py compiles this
// file several times with -DMLSORT_TU=k so each variant is instantiated in exactly one object,
// in parallel (MLSORT_TU = 0: the C ABI and the remaining entry points).  Without MLSORT_TU the
// file is one self-contained translation unit.
#ifndef MLSORT_TU
#define MLSORT_TU (-1)
#endif
#define MLSORT_IN_TU(k) (MLSORT_TU == -1 || MLSORT_TU == (k))

#define MLSORT_RUN_ARGS(K)                                                                                     \
    const K *keys, uint64_t n, uint64_t B, const mlsort::Weights *w, int pred, K *out_keys, uint32_t *out_perm, \
        void *ws, uint64_t ws_bytes, cudaStream_t s, mlsort_info *info, const uint32_t *bucket_in,            \
        const uint32_t *idx_in, uint32_t b_lo, bool timing, bool verify_all, const void *chunks
#define MLSORT_RUN_CALL                                                                                         \
    keys, n, B, w, pred, out_keys, out_perm, ws, ws_bytes, s, info, bucket_in, idx_in, b_lo, timing, verify_all, \
        static_cast<const ChunkPlan*>(chunks)

namespace mlsort_tu {
template <typename KeyT, bool PERM, bool GIVEN>
int run(MLSORT_RUN_ARGS(KeyT));
#define MLSORT_RUN_VARIANT(TU, K, P, G)                                                        \
    template <> int run<K, P, G>(MLSORT_RUN_ARGS(K));
MLSORT_RUN_VARIANT(1, float, false, false)
MLSORT_RUN_VARIANT(2, float, true, false)
MLSORT_RUN_VARIANT(3, double, false, false)
MLSORT_RUN_VARIANT(3, double, true, false)
MLSORT_RUN_VARIANT(4, float, false, true)
MLSORT_RUN_VARIANT(4, float, true, true)
MLSORT_RUN_VARIANT(4, double, false, true)
MLSORT_RUN_VARIANT(4, double, true, true)
#undef MLSORT_RUN_VARIANT
}  // namespace mlsort_tu

#define MLSORT_RUN_DEFINE(K, P, G)                                                              \
    template <> int mlsort_tu::run<K, P, G>(MLSORT_RUN_ARGS(K)) { return run_pipeline<K, P, G>(MLSORT_RUN_CALL); }
#if MLSORT_IN_TU(1)
MLSORT_RUN_DEFINE(float, false, false)
#endif
#if MLSORT_IN_TU(2)
MLSORT_RUN_DEFINE(float, true, false)
#endif
#if MLSORT_IN_TU(3)
MLSORT_RUN_DEFINE(double, false, false)
MLSORT_RUN_DEFINE(double, true, false)
#endif
#if MLSORT_IN_TU(4)
MLSORT_RUN_DEFINE(float, false, true)
MLSORT_RUN_DEFINE(float, true, true)
MLSORT_RUN_DEFINE(double, false, true)
MLSORT_RUN_DEFINE(double, true, true)
#endif

#if MLSORT_IN_TU(0)
// ==================================================================== C ABI

extern "C" int mlsort_sort_workspace_size(uint64_t n, mlsort_dtype dt, const mlsort_opts* o, int want_perm,
                                          uint64_t* bytes) {
    if (!bytes || (dt != MLSORT_F32 && dt != MLSORT_F64)) return MLSORT_ERR_INVALID_ARG;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n;
    if (n == 0) {
        *bytes = 0;
        return MLSORT_OK;
    }
    if (B > (1ull << 30) || B < 1) return MLSORT_ERR_INVALID_ARG;
    *bytes = workspace_bytes(n, dt, B, want_perm != 0) + 2 * kAlign;
    return MLSORT_OK;
}

namespace MLSORT_LOCAL {
int sort_impl(const void* d_keys, const uint32_t* d_payload, uint64_t n, mlsort_dtype dt, const mlsort_weights* wh,
              const mlsort_opts* o, void* d_out_keys, uint32_t* d_out_perm, uint32_t* d_out_payload, void* d_ws,
              uint64_t ws_bytes, void* stream, mlsort_info* info, const ChunkPlan* chunks) {
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->bad_index = -1;
    }
    if (dt != MLSORT_F32 && dt != MLSORT_F64) return MLSORT_ERR_INVALID_ARG;
    if (n == 0) return MLSORT_OK;
    if (!d_keys || !wh || !d_out_keys || d_keys == d_out_keys) return MLSORT_ERR_INVALID_ARG;
    if (d_out_payload && (!d_payload || !d_out_perm)) return MLSORT_ERR_INVALID_ARG;
    if (d_out_perm && n >= (1ull << 32)) return MLSORT_ERR_INVALID_ARG;
    if (n >= (1ull << 32)) return MLSORT_ERR_INVALID_ARG;
    if (o && (o->reserved[0] || o->reserved[1] || o->reserved[2])) return MLSORT_ERR_INVALID_ARG;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n;
    if (B > (1ull << 30)) return MLSORT_ERR_INVALID_ARG;
    const Weights* w = reinterpret_cast<const Weights*>(wh);
    const int pred = resolve_pred(o ? o->predictor : 0, w->m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // align the workspace base
    uintptr_t wsp = reinterpret_cast<uintptr_t>(d_ws);
    uintptr_t aligned = (wsp + kAlign - 1) / kAlign * kAlign;
    if (!d_ws || ws_bytes < (aligned - wsp)) return MLSORT_ERR_WORKSPACE;
    void* ws = reinterpret_cast<void*>(aligned);
    ws_bytes -= (aligned - wsp);
    const bool perm = d_out_perm != nullptr;
    const bool timing = o && o->timing;
    const bool verify_all = o && o->verify == 2;
    int rc;
    if (dt == MLSORT_F32) {
        rc = perm ? mlsort_tu::run<float, true, false>((const float*)d_keys, n, B, w, pred, (float*)d_out_keys, d_out_perm,
                                                     ws, ws_bytes, s, info, nullptr, nullptr, 0, timing, verify_all, chunks)
                  : mlsort_tu::run<float, false, false>((const float*)d_keys, n, B, w, pred, (float*)d_out_keys, nullptr,
                                                      ws, ws_bytes, s, info, nullptr, nullptr, 0, timing, verify_all, chunks);
    } else {
        rc = perm ? mlsort_tu::run<double, true, false>((const double*)d_keys, n, B, w, pred, (double*)d_out_keys,
                                                      d_out_perm, ws, ws_bytes, s, info, nullptr, nullptr, 0, timing, verify_all, chunks)
                  : mlsort_tu::run<double, false, false>((const double*)d_keys, n, B, w, pred, (double*)d_out_keys,
                                                       nullptr, ws, ws_bytes, s, info, nullptr, nullptr, 0, timing, verify_all, chunks);
    }
    if (rc == MLSORT_OK && d_out_payload) {
        k_gather_payload<float><<<grid_for(n, 256), 256, 0, s>>>(d_out_perm, d_payload, d_out_payload, n);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        if (info) info->kernel_launches += 1;
    }
    return rc;
}
}  // namespace MLSORT_LOCAL

extern "C" int mlsort_sort(const void* d_keys, const uint32_t* d_payload, uint64_t n, mlsort_dtype dt,
                           const mlsort_weights* wh, const mlsort_opts* o, void* d_out_keys, uint32_t* d_out_perm,
                           uint32_t* d_out_payload, void* d_ws, uint64_t ws_bytes, void* stream, mlsort_info* info) {
    return sort_impl(d_keys, d_payload, n, dt, wh, o, d_out_keys, d_out_perm, d_out_payload, d_ws, ws_bytes, stream,
                     info, nullptr);
}

extern "C" int mlsort_sort_host_workspace_size(uint64_t n, mlsort_dtype dt, const mlsort_opts* o, int want_perm,
                                               uint64_t* bytes) {
    uint64_t b = 0;
    int rc = mlsort_sort_workspace_size(n, dt, o, want_perm, &b);
    if (rc) return rc;
    const size_t ks = dt == MLSORT_F32 ? 4 : 8;
    *bytes = b + 2 * align_up(n * ks) + (want_perm ? align_up(n * 4) : 0) + kAlign;
    return MLSORT_OK;
}

extern "C" int mlsort_sort_host(const void* h_keys, uint64_t n, mlsort_dtype dt, const mlsort_weights* w,
                                const mlsort_opts* o, void* h_out_keys, uint32_t* h_out_perm, void* d_ws,
                                uint64_t ws_bytes, void* stream, mlsort_info* info) {
    if (dt != MLSORT_F32 && dt != MLSORT_F64) return MLSORT_ERR_INVALID_ARG;
    if (n == 0) {
        if (info) {
            std::memset(info, 0, sizeof(*info));
            info->bad_index = -1;
        }
        return MLSORT_OK;
    }
    if (!h_keys || !h_out_keys || !d_ws) return MLSORT_ERR_INVALID_ARG;
    const size_t ks = dt == MLSORT_F32 ? 4 : 8;
    uintptr_t wsp = reinterpret_cast<uintptr_t>(d_ws);
    uintptr_t aligned = (wsp + kAlign - 1) / kAlign * kAlign;
    const uint64_t need_io = 2 * align_up(n * ks) + (h_out_perm ? align_up(n * 4) : 0);
    if (ws_bytes < (aligned - wsp) + need_io) return MLSORT_ERR_WORKSPACE;
    char* base = reinterpret_cast<char*>(aligned);
    void* d_in = base;
    void* d_out = base + align_up(n * ks);
    uint32_t* d_perm = h_out_perm ? reinterpret_cast<uint32_t*>(base + 2 * align_up(n * ks)) : nullptr;
    void* rest = base + need_io;
    const uint64_t rest_bytes = ws_bytes - (aligned - wsp) - need_io;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // The host-to-device copy is split into chunks of whole K1 tiles on a copy stream; K1 is
    // launched per chunk as soon as that chunk has arrived, so prediction overlaps the copy.
    // copy stream + chunk events, cached per (thread, device): a later call on another device
    // must not record events against a stream of the first one
    struct CopyCtx {
        int dev = -1;
        cudaStream_t cs = nullptr;
        cudaEvent_t evs[16] = {};
    };
    thread_local std::vector<CopyCtx> ctxs;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CopyCtx* cx = nullptr;
    for (auto& c : ctxs)
        if (c.dev == dev) cx = &c;
    if (!cx) {
        CopyCtx c;
        c.dev = dev;
        CK(cudaStreamCreateWithFlags(&c.cs, cudaStreamNonBlocking));
        for (auto& e : c.evs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctxs.push_back(c);
        cx = &ctxs.back();
    }
    cudaStream_t cs = cx->cs;
    cudaEvent_t* evs = cx->evs;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n;
    ChunkPlan cp;
    if (B <= (1ull << 30) && n < (1ull << 32)) {
        const Weights* wh = reinterpret_cast<const Weights*>(w);
        const bool group = wh && resolve_pred(o ? o->predictor : 0, wh->m) == kPredSkip;
        const Plan pl = make_plan(n, B, ks, h_out_perm != nullptr, true, group);
        const uint32_t nchunk = std::min<uint32_t>(8, pl.T);
        const uint32_t per = (pl.T + nchunk - 1) / nchunk;
        cudaEvent_t start_ev = evs[15];
        CK(cudaEventRecord(start_ev, s));                 // the copy stream follows earlier work on s
        CK(cudaStreamWaitEvent(cs, start_ev, 0));
        for (uint32_t i = 0; i < nchunk; ++i) {
            const uint32_t tb = i * per, te = std::min<uint32_t>(pl.T, tb + per);
            if (tb >= te) break;
            const uint64_t k0 = (uint64_t)tb * pl.tile, k1 = std::min<uint64_t>(n, (uint64_t)te * pl.tile);
            CK(cudaMemcpyAsync(static_cast<char*>(d_in) + k0 * ks, static_cast<const char*>(h_keys) + k0 * ks,
                               (k1 - k0) * ks, cudaMemcpyHostToDevice, cs));
            CK(cudaEventRecord(evs[i], cs));
            cp.tile_begin[cp.n] = tb;
            cp.tile_end[cp.n] = te;
            cp.ready[cp.n] = evs[i];
            ++cp.n;
        }
        // (stream s waits on every chunk's event before that chunk's K1 launch, so everything
        // after K1 -- K2..K5, fallbacks -- is ordered after the whole copy)
    } else {
        CK(cudaMemcpyAsync(d_in, h_keys, n * ks, cudaMemcpyHostToDevice, s));
    }
    int rc = sort_impl(d_in, nullptr, n, dt, w, o, d_out, d_perm, nullptr, rest, rest_bytes, stream, info,
                       cp.n ? &cp : nullptr);
    if (rc) {
        // the chunked copies may still be in flight on cs (e.g. an argument error before any
        // K1 launch waited on them): they must not outlive the call
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(s);
        return rc;
    }
    CK(cudaMemcpyAsync(h_out_keys, d_out, n * ks, cudaMemcpyDeviceToHost, s));
    if (h_out_perm) CK(cudaMemcpyAsync(h_out_perm, d_perm, n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return MLSORT_OK;
}

// ---------------------------------------------------------------- approximate ranking
namespace MLSORT_LOCAL {
// Each warp evaluates 32 x G consecutive keys (lane + 32 q), so on sorted input a warp spans a
// narrow value range and the skipping variant (SKIP) drops whole saturated pairs, exactly as on
// k1_ws's value-grouped tiles.  The clamped chain is used throughout: for keys inside the safe
// range the clamp is the identity, so the bits equal the sort's clamp-free evaluation.
template <typename KeyT, int MPAD, int PRED, bool SKIP>
__global__ void __launch_bounds__(256)
k_predict(const KeyT* __restrict__ keys, uint64_t n, FoldedWeights fw, K1Params p, float* __restrict__ y_out,
          uint32_t* __restrict__ b_out) {
    constexpr int G = 8;
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t wb = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 * G); wb < n;
         wb += nwarps * 32 * G) {
        float u[G], ul[G];
        int32_t y[G];
        float mn = INFINITY, mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const uint64_t i = wb + (uint64_t)q * 32 + lane;
            KeyT x = i < n ? keys[i] : (KeyT)p.lo_d;
            if (!KeyTraits<KeyT>::finite(x)) x = (KeyT)p.lo_d;
            key_to_u<KeyT>(x, p, u[q], ul[q]);
            if (i < n) {
                mn = fminf(mn, u[q]);
                mx = fmaxf(mx, u[q]);
            }
        }
        if (SKIP) {
            const uint32_t omn = __reduce_min_sync(0xffffffffu, f32_ordbits(mn));
            const uint32_t omx = __reduce_max_sync(0xffffffffu, f32_ordbits(mx));
            const float umin = __uint_as_float((omn & 0x80000000u) ? (omn & 0x7fffffffu) : ~omn);
            const float umax = __uint_as_float((omx & 0x80000000u) ? (omx & 0x7fffffffu) : ~omx);
            gvm_forward_skip<MPAD, G, true>(fw, u, umin, umax, y);
        } else {
            gvm_forward_dense<MPAD, PRED, G>(fw, u, ul, y);
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const uint64_t i = wb + (uint64_t)q * 32 + lane;
            if (i < n) {
                if (y_out) y_out[i] = fxp_to_float(y[q], p.bm);
                if (b_out) b_out[i] = bucket_of_fxp(y[q], p.bm);
            }
        }
    }
}

template <typename KeyT>
int launch_predict(const KeyT* keys, uint64_t n, const Weights& w, uint64_t B, int pred, float* y, uint32_t* b,
                   cudaStream_t s) {
    const uint32_t mpad = mpad_of(w.m);
    FoldedWeights fw = fold_cached(w, mpad, sizeof(KeyT) == 4);
    Plan p;
    p.n = n;
    K1Params kp = k1_params(w, p, B, sizeof(KeyT) == 4, &fw);
    const uint64_t warps = (n + 32 * 8 - 1) / (32 * 8);
    const int grid = (int)std::min<uint64_t>((uint64_t)num_sms() * 8, (warps + 7) / 8);
#define PCASE(M)                                                                                    \
    if (mpad == M) {                                                                                \
        if (pred == kPredMufu) k_predict<KeyT, M, kPredMufu, false><<<grid, 256, 0, s>>>(keys, n, fw, kp, y, b); \
        else if (pred == kPredMixed) k_predict<KeyT, M, kPredMixed, false><<<grid, 256, 0, s>>>(keys, n, fw, kp, y, b); \
        else if (pred == kPredSkip) k_predict<KeyT, M, kPredPacked, true><<<grid, 256, 0, s>>>(keys, n, fw, kp, y, b); \
        else k_predict<KeyT, M, kPredPacked, false><<<grid, 256, 0, s>>>(keys, n, fw, kp, y, b);   \
    }
    PCASE(16) PCASE(32) PCASE(64)
#undef PCASE
    CK(cudaGetLastError());
    return MLSORT_OK;
}
}  // namespace MLSORT_LOCAL

extern "C" int mlsort_predict(const void* d_keys, uint64_t n, mlsort_dtype dt, const mlsort_weights* wh,
                              uint64_t num_buckets, int32_t predictor, float* d_y, uint32_t* d_bucket, void* stream) {
    if (dt != MLSORT_F32 && dt != MLSORT_F64) return MLSORT_ERR_INVALID_ARG;
    if (n == 0) return MLSORT_OK;
    if (!d_keys || !wh) return MLSORT_ERR_INVALID_ARG;
    const uint64_t B = num_buckets ? num_buckets : n;
    if (B > (1ull << 32)) return MLSORT_ERR_INVALID_ARG;
    const Weights* w = reinterpret_cast<const Weights*>(wh);
    const int pred = resolve_pred(predictor, w->m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return dt == MLSORT_F32 ? launch_predict<float>((const float*)d_keys, n, *w, B, pred, d_y, d_bucket, s)
                            : launch_predict<double>((const double*)d_keys, n, *w, B, pred, d_y, d_bucket, s);
}

// ---------------------------------------------------------------- multi-GPU building blocks
extern "C" int mlsort_dist_partition_workspace_size(uint64_t n_local, mlsort_dtype dt, uint32_t nranks,
                                                    uint64_t* bytes) {
    if (!bytes || nranks < 1 || nranks > kMaxRanks || (dt != MLSORT_F32 && dt != MLSORT_F64)) return MLSORT_ERR_INVALID_ARG;
    const uint64_t nchunks = (n_local + kRadixChunk - 1) / kRadixChunk;
    *bytes = align_up(sizeof(DevStatus)) + align_up(n_local * 4) + align_up(nchunks * kMaxRanks * 4) + 2 * kAlign;
    return MLSORT_OK;
}

extern "C" int mlsort_dist_partition(const void* d_shard, uint64_t n_local, uint64_t global_offset, uint64_t n_global,
                                     mlsort_dtype dt, const mlsort_weights* wh, const mlsort_opts* o, uint32_t nranks,
                                     void* d_rec_keys, uint32_t* d_rec_bucket, uint32_t* d_rec_index,
                                     uint64_t* h_send_counts, void* d_ws, uint64_t ws_bytes, void* stream,
                                     mlsort_info* info) {
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->bad_index = -1;
    }
    if (dt != MLSORT_F32 && dt != MLSORT_F64) return MLSORT_ERR_INVALID_ARG;
    if (!wh || !h_send_counts || nranks < 1 || nranks > kMaxRanks) return MLSORT_ERR_INVALID_ARG;
    if (n_global >= (1ull << 32) || global_offset + n_local > n_global) return MLSORT_ERR_INVALID_ARG;
    for (uint32_t g = 0; g < nranks; ++g) h_send_counts[g] = 0;
    if (n_local == 0) return MLSORT_OK;
    if (!d_shard || !d_rec_keys || !d_rec_bucket) return MLSORT_ERR_INVALID_ARG;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n_global;
    if (B > (1ull << 30)) return MLSORT_ERR_INVALID_ARG;
    const Weights* w = reinterpret_cast<const Weights*>(wh);
    int pred = resolve_pred(o ? o->predictor : 0, w->m);
    if (pred == kPredSkip) pred = kPredPacked;   // (same bits; the owner partition does not group)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uintptr_t wsp = reinterpret_cast<uintptr_t>(d_ws);
    uintptr_t aligned = (wsp + kAlign - 1) / kAlign * kAlign;
    uint64_t need = 0;
    mlsort_dist_partition_workspace_size(n_local, dt, nranks, &need);
    if (!d_ws || ws_bytes < need) return MLSORT_ERR_WORKSPACE;
    char* base = reinterpret_cast<char*>(aligned);
    DevStatus* dst = reinterpret_cast<DevStatus*>(base);
    uint32_t* bucket_tmp = reinterpret_cast<uint32_t*>(base + align_up(sizeof(DevStatus)));
    uint32_t* ghist = reinterpret_cast<uint32_t*>(base + align_up(sizeof(DevStatus)) + align_up(n_local * 4));
    DevStatus init;
    std::memset(&init, 0, sizeof(init));
    init.bad_index = ~0ull;
    CK(cudaMemcpyAsync(dst, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    const uint32_t mpad = mpad_of(w->m);
    FoldedWeights fw = fold_cached(*w, mpad, dt == MLSORT_F32);
    Plan p;
    p.n = n_local;
    K1Params kp = k1_params(*w, p, B, dt == MLSORT_F32, &fw);
    OwnerRule orl;
    orl.B = B;
    orl.G = nranks;
    orl.keyspace = monotone(*w) ? 0u : 1u;    // reading A14: no bucket order without Eq. 4
    orl.lo = w->lo;
    orl.scale = (double)nranks / (w->hi - w->lo);
    int rc = dt == MLSORT_F32
                 ? dist_partition<float>((const float*)d_shard, n_local, global_offset, orl, mpad, pred, fw, kp,
                                         (float*)d_rec_keys, d_rec_bucket, d_rec_index, bucket_tmp, ghist, dst,
                                         h_send_counts, s)
                 : dist_partition<double>((const double*)d_shard, n_local, global_offset, orl, mpad, pred, fw,
                                          kp, (double*)d_rec_keys, d_rec_bucket, d_rec_index, bucket_tmp, ghist, dst,
                                          h_send_counts, s);
    if (rc) return rc;
    DevStatus* hs = host_status();
    CK(cudaMemcpyAsync(hs, dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (info) {
        info->tail_lo = hs->tail_lo;
        info->tail_hi = hs->tail_hi;
        info->kernel_launches = 3;
        info->fallback_used = (int32_t)orl.keyspace;
    }
    if (hs->bad_index != ~0ull) {
        if (info) info->bad_index = (int64_t)hs->bad_index;
        return MLSORT_ERR_NONFINITE_KEY;
    }
    return MLSORT_OK;
}

extern "C" int mlsort_sort_records_workspace_size(uint64_t n, mlsort_dtype dt, uint64_t bucket_lo, uint64_t bucket_hi,
                                                  uint64_t* bytes) {
    if (!bytes || bucket_hi <= bucket_lo) return MLSORT_ERR_INVALID_ARG;
    mlsort_opts o;
    std::memset(&o, 0, sizeof(o));
    o.num_buckets = bucket_hi - bucket_lo;
    if (n == 0) {
        *bytes = 0;
        return MLSORT_OK;
    }
    return mlsort_sort_workspace_size(n, dt, &o, 1, bytes);
}

extern "C" int mlsort_sort_records(const void* d_keys, const uint32_t* d_bucket, const uint32_t* d_index, uint64_t n,
                                   mlsort_dtype dt, uint64_t bucket_lo, uint64_t bucket_hi, void* d_out_keys,
                                   uint32_t* d_out_index, void* d_ws, uint64_t ws_bytes, void* stream,
                                   mlsort_info* info) {
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->bad_index = -1;
    }
    if (dt != MLSORT_F32 && dt != MLSORT_F64) return MLSORT_ERR_INVALID_ARG;
    if (n == 0) return MLSORT_OK;
    if (!d_keys || !d_bucket || !d_out_keys || bucket_hi <= bucket_lo) return MLSORT_ERR_INVALID_ARG;
    if ((d_index == nullptr) != (d_out_index == nullptr)) return MLSORT_ERR_INVALID_ARG;
    if (n >= (1ull << 32) || bucket_hi - bucket_lo > (1ull << 30)) return MLSORT_ERR_INVALID_ARG;
    uintptr_t wsp = reinterpret_cast<uintptr_t>(d_ws);
    uintptr_t aligned = (wsp + kAlign - 1) / kAlign * kAlign;
    if (!d_ws || ws_bytes < (aligned - wsp)) return MLSORT_ERR_WORKSPACE;
    void* ws = reinterpret_cast<void*>(aligned);
    ws_bytes -= (aligned - wsp);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t B = bucket_hi - bucket_lo;
    const uint32_t blo = (uint32_t)bucket_lo;
    if (dt == MLSORT_F32)
        return d_index ? mlsort_tu::run<float, true, true>((const float*)d_keys, n, B, nullptr, kPredMixed,
                                                         (float*)d_out_keys, d_out_index, ws, ws_bytes, s, info,
                                                         d_bucket, d_index, blo, false, false, nullptr)
                       : mlsort_tu::run<float, false, true>((const float*)d_keys, n, B, nullptr, kPredMixed,
                                                          (float*)d_out_keys, nullptr, ws, ws_bytes, s, info,
                                                          d_bucket, nullptr, blo, false, false, nullptr);
    return d_index ? mlsort_tu::run<double, true, true>((const double*)d_keys, n, B, nullptr, kPredMixed,
                                                      (double*)d_out_keys, d_out_index, ws, ws_bytes, s, info,
                                                      d_bucket, d_index, blo, false, false, nullptr)
                   : mlsort_tu::run<double, false, true>((const double*)d_keys, n, B, nullptr, kPredMixed,
                                                       (double*)d_out_keys, nullptr, ws, ws_bytes, s, info, d_bucket,
                                                       nullptr, blo, false, false, nullptr);
}

// ---------------------------------------------------------------- K8: primitive sweeps (A14)
extern "C" int mlsort_selftest_monotone(int32_t primitive, uint64_t* descents, uint64_t* evaluated,
                                        double* max_rel_err, void* stream) {
    if (primitive < kSweepEx2 || primitive > kSweepLogistic) return MLSORT_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    SweepOut* d = nullptr;
    CK(cudaMalloc(&d, sizeof(SweepOut)));
    SweepOut h;
    std::memset(&h, 0, sizeof(h));
    cudaError_t e = cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, s);
    auto pair = [](float v) {
        uint32_t b;
        std::memcpy(&b, &v, 4);
        return ((unsigned long long)b << 32) | b;
    };
    if (e == cudaSuccess) {
        k_sweep_monotone<<<num_sms() * 8, 256, 0, s>>>(primitive, pair(2.001281198f), pair(1.0f), d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d);
    CK(e);
    if (descents) *descents = h.descents;
    if (evaluated) *evaluated = h.evaluated;
    if (max_rel_err) {
        float f;
        std::memcpy(&f, &h.max_rel_err_bits, 4);
        *max_rel_err = f;
    }
    return MLSORT_OK;
}
#endif  // MLSORT_IN_TU(0)
