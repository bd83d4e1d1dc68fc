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
#ifndef MLSORT_K1_PHIST
#define MLSORT_K1_PHIST 0      // 1: predictor warps build the coarse histogram (measured slower:
                               // C2 K1 1.011 -> 1.043 ms, profiles/r02/ab_k1_phist.log -- K1 is
                               // bound by the predictor warps' issue, so work moved there costs)
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
//       (GROUP: cls_u[T] f32 | cls_e[T] u16 | chist[64] | ccur[64] | lut[2048] u8) |
//       (plain, MLSORT_K1_PHIST: hp[2][C'/2] u32 = u16 counter pairs per buffer) | scratch
// (C' = C rounded up to a multiple of 4 so every array stays 16-B aligned).  Without key staging
// (K1Params::flags bit0 clear: plans whose C does not leave room for it) the piece stores
// re-read each key from the tile in global memory (L2-resident) instead of shared memory.
__host__ __device__ inline uint32_t k1ws_c2(uint32_t num_coarse) { return (num_coarse + 3u) & ~3u; }
inline size_t k1ws_smem_bytes(size_t ks, uint32_t tile, uint32_t num_coarse, bool group = false, bool stage = true) {
    return (size_t)tile * 8 + (stage ? (size_t)tile * ks : 0) + (size_t)k1ws_c2(num_coarse) * 8 + (size_t)tile * 2 +
           (group ? (size_t)tile * (MLSORT_K1_GROUP24 ? 2 : 6) + kClasses * 8 + 2048
                  : (MLSORT_K1_PHIST ? (size_t)k1ws_c2(num_coarse) * 4 : 0)) +
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
    // plain path: the predictor warps count each tile's coarse buckets into hp[buf] (two u16
    // counters per word); the partition warps read and clear them in their scan
    constexpr bool kPH = !GROUP && MLSORT_K1_PHIST;
    uint32_t* hp = reinterpret_cast<uint32_t*>(lut + (GROUP ? 2048 : 0));
    const uint32_t hpw = k1ws_c2(p.num_coarse) / 2;           // words per buffer
    uint32_t* scratch = hp + (kPH ? 2 * hpw : 0);

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
    if (kPH) {
        for (uint32_t i = tid; i < 2 * hpw; i += kWsThreads) hp[i] = 0u;
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
        // The (tile, group) sequence is flattened so the keys of the next group -- possibly
        // the first group of the next tile -- are loaded while the current group is evaluated.
        constexpr int G = KPT / kGroupWs;                  // groups per tile
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
            float u[kGroupWs], ul[kGroupWs];
            int32_t y[kGroupWs];
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
                key_to_u<KeyT>(x, p, u[q], ul[q]);
            }
            // warp-uniform choice: the clamp-free predictor when every key of the warp is inside
            // the safe range (all keys but far tails)
            bool safe = true;
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) safe &= (u[q] >= fw.u_safe_lo) & (u[q] <= fw.u_safe_hi);
            if (__all_sync(0xffffffffu, safe))
                gvm_forward_fxp<MPAD, PRED, kGroupWs, false>(fw, u, ul, y);
            else
                gvm_forward_fxp<MPAD, PRED, kGroupWs, true>(fw, u, ul, y);
            uint32_t* sbb = sb + buf * T;
#pragma unroll
            for (int q = 0; q < kGroupWs; ++q) {
                const uint32_t e = tid + kPredThreads * (g * kGroupWs + q);
                const uint32_t b = bucket_of_fxp(y[q], p.bm);
                sbb[e] = b;
                if (kPH && e < cnt) {
                    const uint32_t c = b >> p.fine_bits;
                    atomicAdd(&hp[buf * hpw + (c >> 1)], 1u << ((c & 1u) << 4));
                }
            }
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
        if (!kPH)
            for (uint32_t c = pt; c < k1ws_c2(C); c += kPartThreads) hist[c] = 0u;
        nbar_sync(kFull0 + buf, kWsThreads);           // predictors finished tile k (also orders the zeroing)
        if (!PARTITION) {
            if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);
            continue;
        }
        // ---- coarse histogram (plain path: already built by the predictor warps in hp[buf])
        if (!kPH) {
#pragma unroll 4
            for (uint32_t e = pt; e < cnt; e += kPartThreads) atomicAdd(&hist[sbb[e] >> fbits], 1u);
            nbar_sync(kPart, kPartThreads);
        }
        // ---- scan (warp rows, conflict-free) + reservation of this tile's piece in every region.
        // gbase[c] = region slot of the tile's staged position 0 for coarse bucket c, so a staged
        // element at position pos goes to gbase[c] + pos.  Regions start at c * capc, or at
        // rbase[c] (sampled sizes, K0, or exact ones: the retry after an overflow).  A piece that would overflow
        // its region is marked kOverflowBase and not stored; the call then retries with exact
        // regions from the final cursors.
        {
            // (even chunks: a u16 counter pair of hp never straddles two warps)
            const uint32_t chunk = (((C + kPartWarps - 1) / kPartWarps) + 1u) & ~1u;
            const uint32_t b0 = min(C, (uint32_t)pw * chunk), b1 = min(C, b0 + chunk);
            uint32_t carry = 0;
#pragma unroll 4
            for (uint32_t r = b0; r < b1; r += 32) {
                const uint32_t c = r + lane;
                uint32_t v;
                if (kPH) {                                     // read and clear the predictor's counters
                    uint32_t* hw = &hp[buf * hpw + (c >> 1)];
                    const uint32_t wv = c < b1 ? *hw : 0u;
                    v = (wv >> ((c & 1u) << 4)) & 0xffffu;
                    __syncwarp();
                    if (c < b1 && !(c & 1u)) *hw = 0u;
                } else {
                    v = c < b1 ? hist[c] : 0u;
                }
                const uint32_t g = v ? atomicAdd(&cursor[c], v) : 0u;
                uint32_t x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t yy = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += yy;
                }
                const uint32_t ex = carry + x - v;             // exclusive within the warp's chunk
                if (c < b1) {
                    hist[c] = ex;
                    // region capacity: capc (fixed layout) or rbase[c+1] - rbase[c] (sampled /
                    // exact layouts, K0 / the retry)
                    const unsigned long long rcap = rbase ? rbase[c + 1] - rbase[c] : (unsigned long long)p.capc;
                    const bool fits = (unsigned long long)g + v <= rcap;
                    over |= !fits;
                    const long long rb = rbase ? (long long)rbase[c] : (long long)c * p.capc;
                    gbase[c] = fits ? (uint32_t)(rb + (long long)g + (long long)T - (long long)ex) : kOverflowBase;
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
        // ---- stage the tile partitioned by coarse id (position -> original offset e, key)
#pragma unroll 4
        for (uint32_t e = pt; e < cnt; e += kPartThreads) {
            const uint32_t pos = atomicAdd(&hist[sbb[e] >> fbits], 1u);
            stage_e[pos] = (uint16_t)e;
            if (staged) stage_key[pos] = keys[base + e];       // L2-resident re-read
        }
        nbar_sync(kPart, kPartThreads);
        // ---- store every piece into its coarse bucket's region
#pragma unroll 4
        for (uint32_t pos = pt; pos < cnt; pos += kPartThreads) {
            const uint32_t e = stage_e[pos];
            const uint32_t b = sbb[e];
            const uint32_t gb = gbase[b >> fbits];
            if (gb != kOverflowBase) {
                const size_t dst = (size_t)gb + pos - T;
                reg_keys[dst] = staged ? stage_key[pos] : keys[base + e];
                reg_fine[dst] = (uint16_t)(b & fmask);
                if (PERM) reg_idx[dst] = (uint32_t)(base + e);
            }
        }
        if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);   // sb[buf] may be refilled
        nbar_sync(kPart, kPartThreads);                // stage_* / hist free for the next tile
    }
    if (over) atomicAdd(&st->region_overflow, 1ull);
}

}  // namespace mlsort
