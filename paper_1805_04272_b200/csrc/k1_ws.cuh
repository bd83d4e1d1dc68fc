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

#include "common.cuh"
#include "predict.cuh"
#include "k1_partition.cuh"

namespace mlsort {

constexpr int kWsThreads = 1024;
constexpr int kPredWarps = 24;
constexpr int kPartWarps = 8;
constexpr int kPredThreads = kPredWarps * 32;     // 768
constexpr int kPartThreads = kPartWarps * 32;     // 256

template <typename KeyT> struct WsTile;
template <> struct WsTile<float> { static constexpr int kKeysPerThread = 16; };
template <> struct WsTile<double> { static constexpr int kKeysPerThread = 8; };

template <typename KeyT>
__host__ __device__ constexpr int ws_tile() { return kPredThreads * WsTile<KeyT>::kKeysPerThread; }

// smem: sb[2][T] u32 | stage_key[T] KeyT | hist[C'] u32 | gbase[C'] i64 | stage_e[T] u16 | scratch
// (C' = C rounded up to even so gbase is 8-B aligned)
__host__ __device__ inline uint32_t k1ws_c2(uint32_t num_coarse) { return (num_coarse + 1u) & ~1u; }
inline size_t k1ws_smem_bytes(size_t ks, uint32_t tile, uint32_t num_coarse) {
    return (size_t)tile * 8 + (size_t)tile * ks + (size_t)k1ws_c2(num_coarse) * 12 + (size_t)tile * 2 + 256;
}

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// KGW = keys evaluated together per predictor thread (ILP); PARTITION = false skips the
// partition work (scripts/k1_bench.cu uses it to measure the predictor warps alone).
template <typename KeyT, int MPAD, int PRED, bool PERM, int KGW = 8, bool PARTITION = true>
__global__ void __launch_bounds__(kWsThreads, 1)
k1_ws(const KeyT* __restrict__ keys, FoldedWeights fw, K1Params p, KeyT* __restrict__ reg_keys,
      uint16_t* __restrict__ reg_fine, uint32_t* __restrict__ reg_idx, uint32_t* __restrict__ cursor,
      DevStatus* __restrict__ st) {
    constexpr int T = ws_tile<KeyT>();
    constexpr int KPT = WsTile<KeyT>::kKeysPerThread;
    constexpr int kGroupWs = KGW;
    enum { kFull0 = 1, kEmpty0 = 3, kPart = 5 };
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* sb = reinterpret_cast<uint32_t*>(smem);                         // [2][T]
    KeyT* stage_key = reinterpret_cast<KeyT*>(smem + (size_t)T * 8);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + (size_t)T * 8 + (size_t)T * sizeof(KeyT));
    const uint32_t C = p.num_coarse;
    long long* gbase = reinterpret_cast<long long*>(hist + k1ws_c2(C));   // region slot of position 0
    uint16_t* stage_e = reinterpret_cast<uint16_t*>(gbase + k1ws_c2(C));
    uint32_t* scratch = reinterpret_cast<uint32_t*>(
        (reinterpret_cast<uintptr_t>(stage_e + T) + 15) & ~(uintptr_t)15);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = p.num_tiles;
    const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

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
            const uint64_t base = (uint64_t)(blockIdx.x + k * gridDim.x) * T;
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
            const uint64_t base = (uint64_t)(blockIdx.x + k * gridDim.x) * T;
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
            for (int q = 0; q < kGroupWs; ++q)
                sbb[tid + kPredThreads * (g * kGroupWs + q)] = bucket_of_fxp(y[q], p.bm);
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
        const uint32_t tile = blockIdx.x + k * gridDim.x;
        const uint64_t base = (uint64_t)tile * T;
        const uint32_t cnt = (uint32_t)min((uint64_t)T, p.n - base);
        const int buf = k & 1;
        const uint32_t* sbb = sb + buf * T;
        for (uint32_t c = pt; c < C; c += kPartThreads) hist[c] = 0u;
        nbar_sync(kFull0 + buf, kWsThreads);           // predictors finished tile k (also orders the zeroing)
        if (!PARTITION) {
            if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);
            continue;
        }
        // ---- coarse histogram
#pragma unroll 4
        for (uint32_t e = pt; e < cnt; e += kPartThreads) atomicAdd(&hist[sbb[e] >> fbits], 1u);
        nbar_sync(kPart, kPartThreads);
        // ---- scan (warp rows, conflict-free) + reservation of this tile's piece in every region.
        // gbase[c] = slot of the tile's staged position 0 in the flat region array, so a staged
        // element at position pos goes to gbase[c] + pos.  A piece that would overflow its
        // region is redirected to the trash rows after the regions (the call then falls back).
        {
            const uint32_t chunk = (C + kPartWarps - 1) / kPartWarps;
            const uint32_t b0 = min(C, (uint32_t)pw * chunk), b1 = min(C, b0 + chunk);
            const long long trash = (long long)C * p.capc;
            uint32_t carry = 0;
#pragma unroll 4
            for (uint32_t r = b0; r < b1; r += 32) {
                const uint32_t c = r + lane;
                const uint32_t v = c < b1 ? hist[c] : 0u;
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
                    const bool fits = (unsigned long long)g + v <= p.capc;
                    over |= !fits;
                    gbase[c] = (fits ? (long long)c * p.capc + g : trash) - (long long)ex;
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
                    gbase[c] -= (long long)add;
                }
        }
        nbar_sync(kPart, kPartThreads);
        // ---- stage the tile partitioned by coarse id (position -> original offset e, key)
#pragma unroll 4
        for (uint32_t e = pt; e < cnt; e += kPartThreads) {
            const uint32_t pos = atomicAdd(&hist[sbb[e] >> fbits], 1u);
            stage_e[pos] = (uint16_t)e;
            stage_key[pos] = keys[base + e];                   // L2-resident re-read
        }
        nbar_sync(kPart, kPartThreads);
        // ---- store every piece into its coarse bucket's region
#pragma unroll 4
        for (uint32_t pos = pt; pos < cnt; pos += kPartThreads) {
            const uint32_t e = stage_e[pos];
            const uint32_t b = sbb[e];
            const size_t dst = (size_t)(gbase[b >> fbits] + (long long)pos);
            reg_keys[dst] = stage_key[pos];
            reg_fine[dst] = (uint16_t)(b & fmask);
            if (PERM) reg_idx[dst] = (uint32_t)(base + e);
        }
        if (k + 2 < my_tiles) nbar_arrive(kEmpty0 + buf, kWsThreads);   // sb[buf] may be refilled
        nbar_sync(kPart, kPartThreads);                // stage_* / hist free for the next tile
    }
    if (over) atomicAdd(&st->region_overflow, 1ull);
}

}  // namespace mlsort
