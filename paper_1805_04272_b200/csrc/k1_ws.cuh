// k1_ws.cuh -- K1 (v3): warp-specialized, persistent predict + bucket + tile partition.
//
// PAPER.md §2: every key's rank is estimated independently by the network (Eq. 3, l.73-76;
// r = round(y*B), l.65) and the keys are put into their rank buckets (l.86).  On B200 the
// estimate is SFU/FMA-bound and the partition is latency/LSU-bound, so one CTA per SM runs
// both concurrently on different warps instead of alternating phases:
//   * predictor warps (kPredWarps) evaluate the GVM for tile k into bucket buffer sb[k & 1];
//   * partition warps (kPartWarps) take the previous tile from the other buffer: coarse-id
//     histogram (shared atomics), scan, one global reservation atomic per non-empty coarse
//     bucket, stable-by-position staging, and the store of every piece into its coarse
//     bucket's region (keys, fine ids, input indices) -- the same output contract as
//     k1_predict_partition (regions contiguous per coarse bucket, cursors = exact sizes).
// The handoff is a double buffer guarded by named barriers (FULL[i]: predictors -> partition,
// EMPTY[i]: partition -> predictors), so the SFU never waits for the partition.
#pragma once

#include <climits>
#include <type_traits>

#include "common.cuh"
#include "predict.cuh"
#include "k1_partition.cuh"

namespace mlsort {

#ifndef MLSORT_K1_PARTW
#define MLSORT_K1_PARTW 8
#endif
#ifndef MLSORT_K1_PREDW
#define MLSORT_K1_PREDW 24
#endif
#ifndef MLSORT_K1_SETMAXNREG
#define MLSORT_K1_SETMAXNREG 0  // 1: plain path moves registers from the partition warps (40) to the
                                // predictor warps (72) with setmaxnreg (launched at 64 each)
#endif
#ifndef MLSORT_K1_GROUP24
#define MLSORT_K1_GROUP24 1    // grouped variant: 24 predictor warps, u re-read from the keys (0: 16 warps, u in smem)
#endif
constexpr int kPartWarps = MLSORT_K1_PARTW;   // (macros: warp-split experiments)
constexpr int kPartThreads = kPartWarps * 32;     // 256
constexpr int kClasses = 64;

// Warp split and tile of one k1_ws variant.  Plain: 24 predictor warps (1024 threads, 64
// registers).  GROUP: 24 predictor warps too (MLSORT_K1_GROUP24): the class order keeps only
// the tile offsets in shared memory and phase D re-reads each key from the tile in global
// memory (L2-resident); 16 warps and u in shared memory otherwise.
template <typename KeyT, bool GROUP>
struct WsCfg {
    static constexpr int kPredWarps = GROUP ? (MLSORT_K1_GROUP24 ? 24 : 16) : MLSORT_K1_PREDW;
    static constexpr int kThreads = (kPredWarps + kPartWarps) * 32;
    static constexpr int kPredThreads = kPredWarps * 32;
    // keys per predictor thread per tile (f64 too: the per-tile partition work -- zeroing and
    // scanning C counters, one reservation atomic per non-empty coarse bucket -- is amortised
    // over more keys; f64 plans then run without key staging)
    static constexpr int kKPT = 16;
    static constexpr int kT = kPredThreads * kKPT;
};

template <typename KeyT>
__host__ __device__ constexpr int ws_tile(bool group = false) {
    return group ? WsCfg<KeyT, true>::kT : WsCfg<KeyT, false>::kT;
}
inline int ws_threads(bool group) { return group ? WsCfg<float, true>::kThreads : WsCfg<float, false>::kThreads; }

// smem: sb[2][T] u32 | stage_key[T] KeyT (staged plans) | hist[C'] u32 | gbase[C'] u32 | stage_e[T] u16 |
//       (GROUP: cls_u[T] f32 | cls_e[T] u16 | chist[64] | ccur[64] | lut[2048] u8) | scratch
// (C' = C rounded up to a multiple of 4 so every array stays 16-B aligned).  Without key staging
// (K1Params::flags bit0 clear: plans whose C does not leave room for it) the piece stores
// re-read each key from the tile in global memory (L2-resident) instead of shared memory.
__host__ __device__ inline uint32_t k1ws_c2(uint32_t num_coarse) { return (num_coarse + 3u) & ~3u; }
inline size_t k1ws_smem_bytes(size_t ks, uint32_t tile, uint32_t num_coarse, bool group = false, bool stage = true) {
    return (size_t)tile * 8 + (stage ? (size_t)tile * ks : 0) + (size_t)k1ws_c2(num_coarse) * 8 + (size_t)tile * 2 +
           (group ? (size_t)tile * (MLSORT_K1_GROUP24 ? 2 : 6) + kClasses * 8 + 2048 : 0) +
           256;
}
constexpr uint32_t kK1StageKeys = 1u;      // K1Params::flags
// gbase[c] holds (region slot of the tile's staged position 0) + T, so it is never negative and a
// staged element at position pos goes to gbase[c] + pos - T; region slots + T stay below 2^32 - 1
// (checked by the plan), which leaves 0xFFFFFFFF free as the marker of an overflowed piece.
constexpr uint32_t kOverflowBase = 0xFFFFFFFFu;

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// KGW = keys evaluated together per predictor thread (ILP); PARTITION = false skips the
// partition work (scripts/k1_bench.cu uses it to measure the predictor warps alone).
// GROUP = true (packed predictor only): each tile is first grouped by a 64-class value proxy
// so a warp's 256 keys span a narrow range and saturated neuron pairs are skipped
// (gvm_forward_skip), with 16 predictor warps and the tile's u values kept in shared memory in
// class order.
template <typename KeyT, int MPAD, int PRED, bool PERM, int KGW = 8, bool PARTITION = true, bool GROUP = false>
__global__ void __launch_bounds__(WsCfg<KeyT, GROUP>::kThreads, 1)
k1_ws(const KeyT* __restrict__ keys, K1Params p, KeyT* __restrict__ reg_keys,
      uint16_t* __restrict__ reg_fine, uint32_t* __restrict__ reg_idx, uint32_t* __restrict__ cursor,
      DevStatus* __restrict__ st, const unsigned long long* __restrict__ rbase, FoldedWeights fw) {
    // (fw last: its hot members then sit in the first 4 KB of the parameter bank)
    using Cfg = WsCfg<KeyT, GROUP>;
    constexpr int T = Cfg::kT;
    constexpr int KPT = Cfg::kKPT;
    constexpr int kPredWarps = Cfg::kPredWarps;
    constexpr int kPredThreads = Cfg::kPredThreads;
    constexpr int kWsThreads = Cfg::kThreads;
    constexpr int kGroupWs = KGW;
    enum { kFull0 = 1, kEmpty0 = 3, kPart = 5, kPred = 6 };
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* sb = reinterpret_cast<uint32_t*>(smem);                         // [2][T]
    const bool staged = (p.flags & kK1StageKeys) != 0;
    KeyT* stage_key = reinterpret_cast<KeyT*>(smem + (size_t)T * 8);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + (size_t)T * 8 + (staged ? (size_t)T * sizeof(KeyT) : 0));
    const uint32_t C = p.num_coarse;
    uint32_t* gbase = hist + k1ws_c2(C);                   // region slot of staged position 0, + T
    uint16_t* stage_e = reinterpret_cast<uint16_t*>(gbase + k1ws_c2(C));
    constexpr bool kClsU = GROUP && !MLSORT_K1_GROUP24;
    float* cls_u = reinterpret_cast<float*>(stage_e + T);                   // GROUP (16 warps): u in class order
    uint16_t* cls_e = reinterpret_cast<uint16_t*>(cls_u + (kClsU ? T : 0));  // GROUP: tile offsets
    uint32_t* chist = reinterpret_cast<uint32_t*>(cls_e + (GROUP ? T : 0));
    uint32_t* ccur = chist + (GROUP ? kClasses : 0);
    unsigned char* lut = reinterpret_cast<unsigned char*>(ccur + (GROUP ? kClasses : 0));
    uint32_t* scratch = reinterpret_cast<uint32_t*>(lut + (GROUP ? 2048 : 0));

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = p.num_tiles;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (GROUP) {
        for (int i = tid; i < 2048 / 4; i += kWsThreads)
            reinterpret_cast<uint32_t*>(lut)[i] = reinterpret_cast<const uint32_t*>(fw.lut)[i];
        if (tid < kClasses) chist[tid] = 0u;
        __syncthreads();
    }

    if (GROUP && warp < kPredWarps) {
        // ===================================================== predictor warps (value-grouped)
        // A: load the tile (coalesced), validate, tail counts, u, class = lut[ordbits(u) >> 21],
        //    class histogram (shared atomics).   B: scan the 64 classes.   C: scatter (u, offset)
        //    into class order.   D: each warp evaluates 512 consecutive keys of the class order
        //    (two groups of 256: a narrow u range) with saturated-pair skipping; b -> sb[buf][e].
        uint32_t tail_lo = 0, tail_hi = 0;
        for (uint32_t k = 0; k < my_tiles; ++k) {
            const uint32_t tile = p.tile0 + blockIdx.x + k * gridDim.x;
            const uint64_t base = (uint64_t)tile * T;
            const uint32_t cnt = (uint32_t)min((uint64_t)T, p.n - base);
            const int buf = k & 1;
            float ua[KPT];
            uint32_t cls4[KPT / 4];                              // 8-bit classes, 4 per word
#pragma unroll
            for (int i = 0; i < KPT / 4; ++i) cls4[i] = 0u;
#pragma unroll
            for (int g = 0; g < KPT / 8; ++g) {
                KeyT xv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t e = tid + kPredThreads * (g * 8 + q);
                    xv[q] = e < cnt ? keys[base + e] : (KeyT)p.lo_d;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int i = g * 8 + q;
                    const uint32_t e = tid + kPredThreads * i;
                    KeyT x = xv[q];
                    if (!KeyTraits<KeyT>::finite(x)) {
                        atomicMin(&st->bad_index, (unsigned long long)(base + e));
                        x = (KeyT)p.lo_d;
                    }
                    if (e < cnt) {
                        if (sizeof(KeyT) == 4) {
                            tail_lo += (float)x < p.lo_tf;
                            tail_hi += (float)x > p.hi_tf;
                        } else {
                            tail_lo += (double)x < p.lo_d;
                            tail_hi += (double)x > p.hi_d;
                        }
                    }
                    float ulo;
                    key_to_u<KeyT>(x, p, ua[i], ulo);
                    const uint32_t c = e < cnt ? (uint32_t)lut[f32_ordbits(ua[i]) >> 21] : (uint32_t)kClasses;
                    cls4[i >> 2] |= c << ((i & 3) * 8);
                    if (c < kClasses) atomicAdd(&chist[c], 1u);
                }
            }
            nbar_sync(kPred, kPredThreads);
            if (warp == 0) {                                     // B: exclusive scan of 64 classes
                const uint32_t v0 = chist[2 * lane], v1 = chist[2 * lane + 1];
                uint32_t x = v0 + v1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t yy = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += yy;
                }
                const uint32_t ex = x - v0 - v1;
                ccur[2 * lane] = ex;
                ccur[2 * lane + 1] = ex + v0;
                chist[2 * lane] = 0u;
                chist[2 * lane + 1] = 0u;
            }
            nbar_sync(kPred, kPredThreads);
#pragma unroll
            for (int i = 0; i < KPT; ++i) {                      // C: scatter in class order
                const uint32_t c = (cls4[i >> 2] >> ((i & 3) * 8)) & 0xffu;
                if (c < kClasses) {
                    const uint32_t pos = atomicAdd(&ccur[c], 1u);
                    if (kClsU) cls_u[pos] = ua[i];
                    cls_e[pos] = (uint16_t)(tid + kPredThreads * i);
                }
            }
            nbar_sync(kPred, kPredThreads);
            if (k >= 2) nbar_sync(kEmpty0 + buf, kWsThreads);    // partition released sb[buf]
            uint32_t* sbb = sb + buf * T;
            // D: this warp evaluates positions [w*KPT*32, (w+1)*KPT*32) of the class order
            constexpr int GD = KPT / kGroupWs;
#pragma unroll 1
            for (int g = 0; g < GD; ++g) {
                float u[kGroupWs], ul[kGroupWs];
                uint32_t ec[kGroupWs];
                int32_t y[kGroupWs];
                float mn = INFINITY, mx = -INFINITY;
                bool safe = true;
                KeyT xg[kGroupWs];
                if (!kClsU) {                                    // gather the group's keys (L2)
#pragma unroll
                    for (int q = 0; q < kGroupWs; ++q) {
                        const uint32_t pos = (uint32_t)warp * (KPT * 32) + (g * kGroupWs + q) * 32 + lane;
                        ec[q] = pos < cnt ? (uint32_t)cls_e[pos] : 0xffffffffu;
                    }
#pragma unroll
                    for (int q = 0; q < kGroupWs; ++q) xg[q] = ec[q] != 0xffffffffu ? keys[base + ec[q]] : (KeyT)p.lo_d;
                }
#pragma unroll
                for (int q = 0; q < kGroupWs; ++q) {
                    const uint32_t pos = (uint32_t)warp * (KPT * 32) + (g * kGroupWs + q) * 32 + lane;
                    const bool valid = pos < cnt;
                    if (kClsU) {
                        u[q] = valid ? cls_u[pos] : 0.0f;
                        ec[q] = valid ? (uint32_t)cls_e[pos] : 0xffffffffu;
                    } else {                                     // the same u as phase A
                        KeyT x = xg[q];
                        if (!KeyTraits<KeyT>::finite(x)) x = (KeyT)p.lo_d;
                        float ulo;
                        key_to_u<KeyT>(x, p, u[q], ulo);
                        if (!valid) u[q] = 0.0f;
                    }
                    ul[q] = 0.0f;
                    if (valid) {
                        mn = fminf(mn, u[q]);
                        mx = fmaxf(mx, u[q]);
                    }
                    safe &= (u[q] >= fw.u_safe_lo) & (u[q] <= fw.u_safe_hi);
                }
                // warp-wide range of u (order-preserving bits; empty lanes contribute nothing)
                const uint32_t omn = __reduce_min_sync(0xffffffffu, f32_ordbits(mn));
                const uint32_t omx = __reduce_max_sync(0xffffffffu, f32_ordbits(mx));
                const float umin = __uint_as_float((omn & 0x80000000u) ? (omn & 0x7fffffffu) : ~omn);
                const float umax = __uint_as_float((omx & 0x80000000u) ? (omx & 0x7fffffffu) : ~omx);
                if (__all_sync(0xffffffffu, safe))
                    gvm_forward_skip<MPAD, kGroupWs, false>(fw, u, umin, umax, y);
                else
                    gvm_forward_skip<MPAD, kGroupWs, true>(fw, u, umin, umax, y);
#pragma unroll
                for (int q = 0; q < kGroupWs; ++q)
                    if (ec[q] != 0xffffffffu) sbb[ec[q]] = bucket_of_fxp(y[q], p.bm);
            }
            nbar_arrive(kFull0 + buf, kWsThreads);               // sb[buf] is ready
        }
        tail_lo = __reduce_add_sync(0xffffffffu, tail_lo);
        tail_hi = __reduce_add_sync(0xffffffffu, tail_hi);
        if (lane == 0) {
            if (tail_lo) atomicAdd(&st->tail_lo, (unsigned long long)tail_lo);
            if (tail_hi) atomicAdd(&st->tail_hi, (unsigned long long)tail_hi);
        }
        return;
    }

    if (warp < kPredWarps) {
        // ===================================================== predictor warps
        if (MLSORT_K1_SETMAXNREG && kPredWarps % 4 == 0 && kPartWarps % 4 == 0)
            asm volatile("setmaxnreg.inc.sync.aligned.u32 72;\n" ::: "memory");
        // The (tile, group) sequence is flattened so the keys of the next group -- possibly
        // the first group of the next tile -- are loaded while the current group is evaluated.
        constexpr int G = KPT / kGroupWs;                  // groups per tile
        // (128-bit key loads / bucket stores here need quad-aligned registers and made this
        // 64-register kernel spill: scalar, coalesced across the warp)
        uint32_t tail_lo = 0, tail_hi = 0;
        const uint32_t nsteps = my_tiles * G;
        KeyT xn[kGroupWs];
        auto load_group = [&](uint32_t step) {
            const uint32_t k = step / G, g = step - k * G;
            const uint64_t base = (uint64_t)(p.tile0 + blockIdx.x + k * gridDim.x) * T;
            const uint32_t cnt = (uint32_t)min((uint64_t)T, p.n - base);
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) {
                const uint32_t e = tid + kPredThreads * (g * kGroupWs + q);
                xn[q] = e < cnt ? keys[base + e] : (KeyT)p.lo_d;
            }
        };
        if (nsteps) load_group(0);
#pragma unroll 1
        for (uint32_t step = 0; step < nsteps; ++step) {
            const uint32_t k = step / G, g = step - k * G;
            const uint64_t base = (uint64_t)(p.tile0 + blockIdx.x + k * gridDim.x) * T;
            const uint32_t cnt = (uint32_t)min((uint64_t)T, p.n - base);
            const int buf = k & 1;
            if (g == 0 && k >= 2) nbar_sync(kEmpty0 + buf, kWsThreads);   // partition released sb[buf]
            KeyT xc[kGroupWs];
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) xc[q] = xn[q];
            if (step + 1 < nsteps) load_group(step + 1);
            // validation (A0) and tail counts: a warp whose keys are all inside [input_lo,
            // input_hi] (finite, no tail; padding keys are input_lo) skips both
            bool inr = true;
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) {
                if (sizeof(KeyT) == 4)
                    inr &= ((float)xc[q] >= p.lo_tf) & ((float)xc[q] <= p.hi_tf);
                else
                    inr &= ((double)xc[q] >= p.lo_d) & ((double)xc[q] <= p.hi_d);
            }
            if (!__all_sync(0xffffffffu, inr)) {
#pragma unroll
                for (int q = 0; q < kGroupWs; ++q) {
                    const uint32_t e = tid + kPredThreads * (g * kGroupWs + q);
                    KeyT x = xc[q];
                    if (!KeyTraits<KeyT>::finite(x)) {
                        atomicMin(&st->bad_index, (unsigned long long)(base + e));
                        x = (KeyT)p.lo_d;
                    }
                    if (e < cnt) {
                        if (sizeof(KeyT) == 4) {
                            tail_lo += (float)x < p.lo_tf;
                            tail_hi += (float)x > p.hi_tf;
                        } else {
                            tail_lo += (double)x < p.lo_d;
                            tail_hi += (double)x > p.hi_d;
                        }
                    }
                    xc[q] = x;
                }
            }
            float u[kGroupWs], ul[kGroupWs];
            int32_t y[kGroupWs];
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) key_to_u<KeyT>(xc[q], p, u[q], ul[q]);
            // overflow guard: the per-pair clamp when the weights admit it (packed predictor),
            // else a warp-uniform choice of the clamp-free chain when every key of the warp is
            // inside the safe range, and the per-activation clamp otherwise
            if (PRED == kPredPacked && fw.pair_clamp) {
                gvm_forward_fxp<MPAD, PRED, kGroupWs, kClampPair>(fw, u, ul, y);
            } else {
                bool safe = true;
#pragma unroll
                for (int q = 0; q < kGroupWs; ++q) safe &= (u[q] >= fw.u_safe_lo) & (u[q] <= fw.u_safe_hi);
                if (__all_sync(0xffffffffu, safe))
                    gvm_forward_fxp<MPAD, PRED, kGroupWs, kClampNone>(fw, u, ul, y);
                else
                    gvm_forward_fxp<MPAD, PRED, kGroupWs, kClampAct>(fw, u, ul, y);
            }
            uint32_t* sbb = sb + buf * T;
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) sbb[tid + kPredThreads * (g * kGroupWs + q)] = bucket_of_fxp(y[q], p.bm);
            if (g == G - 1) nbar_arrive(kFull0 + buf, kWsThreads);        // sb[buf] is ready
        }
        tail_lo = __reduce_add_sync(0xffffffffu, tail_lo);
        tail_hi = __reduce_add_sync(0xffffffffu, tail_hi);
        if (lane == 0) {
            if (tail_lo) atomicAdd(&st->tail_lo, (unsigned long long)tail_lo);
            if (tail_hi) atomicAdd(&st->tail_hi, (unsigned long long)tail_hi);
        }
        return;
    }

    // ===================================================== partition warps
    if (MLSORT_K1_SETMAXNREG && !GROUP && kPredWarps % 4 == 0 && kPartWarps % 4 == 0)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    const int pt = tid - kPredThreads;                 // 0 .. kPartThreads-1
    const int pw = warp - kPredWarps;
    const uint32_t fbits = p.fine_bits;
    const uint32_t fmask = (1u << fbits) - 1u;
    bool over = false;
    for (uint32_t k = 0; k < my_tiles; ++k) {
        const uint32_t tile = p.tile0 + blockIdx.x + k * gridDim.x;
        const uint64_t base = (uint64_t)tile * T;
        const uint32_t cnt = (uint32_t)min((uint64_t)T, p.n - base);
        const int buf = k & 1;
        const uint32_t* sbb = sb + buf * T;
        for (uint32_t c = pt; c < k1ws_c2(C); c += kPartThreads) hist[c] = 0u;
        nbar_sync(kFull0 + buf, kWsThreads);           // predictors finished tile k (also orders the zeroing)
        if (!PARTITION) {
            if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);
            continue;
        }
        // ---- coarse histogram
#pragma unroll 4
        for (uint32_t e = pt; e < cnt; e += kPartThreads) atomicAdd(&hist[sbb[e] >> fbits], 1u);
        nbar_sync(kPart, kPartThreads);
        // ---- scan + reservation of this tile's piece in every region.  gbase[c] = region slot of
        // the tile's staged position 0 for coarse bucket c, plus T, so a staged element at position
        // pos goes to gbase[c] + pos - T.  Regions start at c * capc, or at rbase[c] (sampled sizes,
        // K0, or exact ones: the retry after an overflow).  A piece that would overflow its region
        // is marked kOverflowBase and not stored; the call then retries with exact regions from the
        // final cursors.  Each lane takes 4 consecutive counters (128-bit shared loads and stores,
        // conflict-free), so a warp row covers 128 coarse buckets; counters are zeroed up to
        // k1ws_c2(C), a multiple of 4.
        {
            const uint32_t C4 = k1ws_c2(C);
            const uint32_t chunk = ((C4 / 4u + kPartWarps - 1u) / kPartWarps) * 4u;
            const uint32_t b0 = min(C4, (uint32_t)pw * chunk), b1 = min(C4, b0 + chunk);
            uint32_t carry = 0;
#pragma unroll 2
            for (uint32_t r = b0; r < b1; r += 128u) {
                const uint32_t c0 = r + 4u * (uint32_t)lane;
                const bool in = c0 < b1;
                const uint4 v4 = in ? *reinterpret_cast<const uint4*>(hist + c0) : make_uint4(0u, 0u, 0u, 0u);
                const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
                uint32_t g[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) g[h] = vv[h] ? atomicAdd(&cursor[c0 + h], vv[h]) : 0u;   // (pads are 0)
                const uint32_t s4 = vv[0] + vv[1] + vv[2] + vv[3];
                uint32_t x = s4;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t yy = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += yy;
                }
                if (in) {
                    uint32_t ex = carry + x - s4;              // exclusive within the warp's chunk
                    uint32_t exs[4], gbs[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const uint32_t c = c0 + h;
                        exs[h] = ex;
                        gbs[h] = kOverflowBase;
                        if (c < C) {
                            // region capacity: capc (fixed layout) or rbase[c+1] - rbase[c]
                            // (sampled / exact layouts, K0 / the retry)
                            const unsigned long long rcap = rbase ? rbase[c + 1] - rbase[c] : (unsigned long long)p.capc;
                            const bool fits = (unsigned long long)g[h] + vv[h] <= rcap;
                            over |= !fits;
                            const long long rb = rbase ? (long long)rbase[c] : (long long)c * p.capc;
                            if (fits) gbs[h] = (uint32_t)(rb + (long long)g[h] + (long long)T - (long long)ex);
                        }
                        ex += vv[h];
                    }
                    *reinterpret_cast<uint4*>(hist + c0) = make_uint4(exs[0], exs[1], exs[2], exs[3]);
                    *reinterpret_cast<uint4*>(gbase + c0) = make_uint4(gbs[0], gbs[1], gbs[2], gbs[3]);
                }
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) scratch[pw] = carry;
            nbar_sync(kPart, kPartThreads);
            uint32_t add = 0;
            for (int w = 0; w < pw; ++w) add += scratch[w];
            if (add)
                for (uint32_t c = b0 + lane; c < b1; c += 32) {
                    hist[c] += add;
                    if (gbase[c] != kOverflowBase) gbase[c] -= add;
                }
        }
        nbar_sync(kPart, kPartThreads);
        // ---- stage the tile partitioned by coarse id (position -> original offset e, key), then
        // store every piece into its coarse bucket's region (32-bit region slots; an overflowed
        // piece, gbase = kOverflowBase, is skipped by predication)
        auto stage_store = [&](auto staged_c) {
            constexpr bool kStaged = decltype(staged_c)::value;
#pragma unroll 4
            for (uint32_t e = pt; e < cnt; e += kPartThreads) {
                const uint32_t pos = atomicAdd(&hist[sbb[e] >> fbits], 1u);
                stage_e[pos] = (uint16_t)e;
                if (kStaged) stage_key[pos] = keys[base + e];   // L2-resident re-read
            }
            nbar_sync(kPart, kPartThreads);
            KeyT* rk = reg_keys - T;                            // gbase[c] carries + T
            uint16_t* rf = reg_fine - T;
            uint32_t* ri = PERM ? reg_idx - T : nullptr;
            const KeyT* kb = keys + base;
#pragma unroll 4
            for (uint32_t pos = pt; pos < cnt; pos += kPartThreads) {
                const uint32_t e = stage_e[pos];
                const uint32_t b = sbb[e];
                const uint32_t gb = gbase[b >> fbits];
                const KeyT kv = kStaged ? stage_key[pos] : kb[e];
                const bool ok = gb != kOverflowBase;
                const uint32_t dst = gb + pos;
                if (__all_sync(__activemask(), ok)) {          // (overflowed pieces are rare)
                    rk[dst] = kv;
                    rf[dst] = (uint16_t)(b & fmask);
                    if (PERM) ri[dst] = (uint32_t)(base + e);
                } else if (ok) {
                    rk[dst] = kv;
                    rf[dst] = (uint16_t)(b & fmask);
                    if (PERM) ri[dst] = (uint32_t)(base + e);
                }
            }
        };
        if (staged)
            stage_store(std::true_type{});
        else
            stage_store(std::false_type{});
        if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);   // sb[buf] may be refilled
        nbar_sync(kPart, kPartThreads);                // stage_* / hist free for the next tile
    }
    if (over) atomicAdd(&st->region_overflow, 1ull);
}

}  // namespace mlsort
