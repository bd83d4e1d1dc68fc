// k1_partition.cuh -- K1: fused predict + bucket + tile-local coarse partition.
//
// One CTA per tile of kTile consecutive keys (§2: "the estimation of ranking of
// each number is independent of each other", l.94).  Per key: u = x - lo; the GVM forward
// pass (Eq. 3) on the SFU/FMA pipes; the rank bucket b = round(y*B) (l.65); the coarse id
// c = b >> fine_bits.  Per tile: a shared-memory histogram over the C coarse ids, a block
// scan, a shared-memory scatter that partitions the tile by c, one global atomicAdd per
// non-empty coarse bucket that reserves the tile's piece in that bucket's region (regions
// are sized at kRegionFactor x the average bucket), and a store of every piece straight
// into its region (keys, fine bits b & (2^fine_bits - 1), and the input index for perm
// sorts).  K3 then reads each coarse bucket contiguously.  The
// per-bucket cursors end as the exact bucket sizes; an overfull region sets the overflow
// flag and the call falls back to the conventional sort.
#pragma once

#include "common.cuh"
#include "predict.cuh"

namespace mlsort {

constexpr int kTileSmall = 8192;              // keys per K1 tile (stable/perm sorts)
constexpr int kTileLarge = 16384;             // keys per K1 tile (key-only sorts)
constexpr int kGroup = 8;                      // keys evaluated together (ILP)

struct K1Params {
    double lo_d, hi_d;       // input_lo / input_hi of the weights (tail diagnostic)
    double x0_d;             // origin of u = x - x0 (f64 keys)
    float x0_f;              // origin of u = x - x0 (f32 keys; 0 or input_lo rounded)
    float lo_tf, hi_tf;      // f32 keys: x < lo_d <=> x < lo_tf, x > hi_d <=> x > hi_tf
    BucketMap bm;
    uint32_t fine_bits;      // b = c * 2^fine_bits + fine
    uint32_t num_coarse;     // C
    uint32_t num_tiles;      // tiles processed by this launch
    uint32_t capc;           // region capacity (elements) of every coarse bucket
    uint64_t n;
    uint32_t tile0;          // first tile of this launch (chunked launches overlap the H2D copy)
    // u is clamped into [u_cl_lo, u_cl_hi] (+-inf: no clamp).  Beyond these bounds EVERY neuron is
    // saturated, where each term of the packed predictor is an exact constant (DESIGN.md "K1
    // sparse evaluation"), so the clamp changes no output bit; inside them no logistic argument
    // exceeds 120, so the predictor needs no per-activation clamp (FoldedWeights::u_safe_*).
    float u_cl_lo, u_cl_hi;
    uint32_t flags;          // k1_ws: kK1StageKeys = keys staged in shared memory for the piece stores
};

template <typename KeyT> __device__ __forceinline__ void key_to_u(KeyT x, const K1Params& p, float& uh, float& ul);
template <> __device__ __forceinline__ void key_to_u<float>(float x, const K1Params& p, float& uh, float& ul) {
    uh = fminf(fmaxf(x - p.x0_f, p.u_cl_lo), p.u_cl_hi);
    ul = 0.0f;
}
// f64 keys: u = x - x0 in f64, rounded once to f32.  y then depends on x only through the
// monotone map x -> fl32(x - x0), so the predictor is monotone in x whenever it is monotone
// over f32 u (which the exhaustive K8 sweep checks), and the relative error of u (2^-24) costs
// at most |u dy/du| 2^-24 <~ 1e-7 of y.  Keys closer than one f32 ulp of u
// share a rank bucket; the fix-up orders them by the full f64 key.
template <> __device__ __forceinline__ void key_to_u<double>(double x, const K1Params& p, float& uh, float& ul) {
    uh = fminf(fmaxf((float)(x - p.x0_d), p.u_cl_lo), p.u_cl_hi);
    ul = 0.0f;
}

// Dynamic shared memory: stage_key[kTile] KeyT | stage_idx[kTile] u32 (PERM) | hist[C] u32
//                        | stage_fine[kTile] u16 | scratch.
inline size_t k1_smem_bytes(size_t ks, bool perm, uint32_t tile, uint32_t num_coarse) {
    return (size_t)num_coarse * 8 + (size_t)tile * ks + (perm ? (size_t)tile * 4 : 0) + (size_t)tile * 4 + 512;
}

// GIVEN = true is the multi-GPU receive side (mlsort_sort_records): the bucket travels with
// the key, so no prediction is repeated; bucket_in holds global buckets, b_lo is this rank's
// first bucket and idx_in the global input indices.
template <typename KeyT, int MPAD, int PRED, bool PERM, bool GIVEN, int kTile>
__global__ void __launch_bounds__(kThreads, 2)
k1_predict_partition(const KeyT* __restrict__ keys, FoldedWeights fw, K1Params p,
                     KeyT* __restrict__ reg_keys, uint16_t* __restrict__ reg_fine,
                     uint32_t* __restrict__ reg_idx, uint32_t* __restrict__ cursor,
                     DevStatus* __restrict__ st, const uint32_t* __restrict__ bucket_in = nullptr,
                     const uint32_t* __restrict__ idx_in = nullptr, uint32_t b_lo = 0,
                     const unsigned long long* __restrict__ rbase = nullptr) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t C = p.num_coarse;
    // layout: stage_key[kTile] KeyT | stage_idx[kTile] u32 (PERM) | stage_b[kTile] u32 | hist[C] u32
    //         | gadj[C] i32 | scratch
    KeyT* stage_key = reinterpret_cast<KeyT*>(smem);
    uint32_t* stage_idx = reinterpret_cast<uint32_t*>(smem + (size_t)kTile * sizeof(KeyT));
    uint32_t* stage_b = stage_idx + (PERM ? kTile : 0);
    uint32_t* hist = stage_b + kTile;
    int32_t* gadj = reinterpret_cast<int32_t*>(hist + C);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(gadj + C);

    constexpr int kKeysPerThread = kTile / kThreads;
    const int tid = threadIdx.x;
    const uint32_t tile = p.tile0 + blockIdx.x;
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
    // keys of the next group are loaded while the current group is evaluated
    KeyT xn[kGroup];
#pragma unroll
    for (int q = 0; q < kGroup; ++q) {
        const uint32_t e = tid + kThreads * q;
        xn[q] = (!GIVEN && e < cnt) ? keys[base + e] : (KeyT)p.lo_d;
    }
#pragma unroll 1
    for (int g = 0; g < (GIVEN ? 0 : kKeysPerThread / kGroup); ++g) {
        float u[kGroup], ul[kGroup];
        int32_t y[kGroup];
        KeyT xc[kGroup];
#pragma unroll
        for (int q = 0; q < kGroup; ++q) xc[q] = xn[q];
        if (g + 1 < kKeysPerThread / kGroup) {
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                const uint32_t e = tid + kThreads * ((g + 1) * kGroup + q);
                xn[q] = e < cnt ? keys[base + e] : (KeyT)p.lo_d;
            }
        }
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
            const uint32_t e = tid + kThreads * (g * kGroup + q);
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
        gvm_forward_dense<MPAD, PRED, kGroup>(fw, u, ul, y);
#pragma unroll
        for (int q = 0; q < kGroup; ++q) sb[tid + kThreads * (g * kGroup + q)] = bucket_of_fxp(y[q], p.bm);
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

    // ---- exclusive scan of hist; reserve this tile's piece in every coarse bucket's region
    const uint32_t per = (C + kThreads - 1) / kThreads;
    const uint32_t c0 = min(C, tid * per), c1 = min(C, c0 + per);
    uint32_t local = 0;
    for (uint32_t c = c0; c < c1; ++c) local += hist[c];
    uint32_t total;
    uint32_t run = block_exclusive_scan<kThreads>(local, scratch, &total);
#pragma unroll 8
    for (uint32_t c = c0; c < c1; ++c) {        // unrolled: the reservations are issued back to back
        const uint32_t h = hist[c];
        const uint32_t g = h ? atomicAdd(&cursor[c], h) : 0u;
        gadj[c] = (int32_t)g - (int32_t)run;     // region slot of staged element e = gadj[c] + e
        hist[c] = run;
        run += h;
    }
    __syncthreads();

    // ---- scatter into the shared staging area, partitioned by coarse id
#pragma unroll
    for (int k = 0; k < kKeysPerThread; ++k) {
        const uint32_t e = tid + kThreads * k;
        if (e < cnt) {
            const uint32_t pos = atomicAdd(&hist[bk[k] >> p.fine_bits], 1u);
            stage_key[pos] = keys[base + e];            // L2-resident re-read
            stage_b[pos] = bk[k];
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

    // ---- store every piece into its coarse bucket's region (coalesced within a piece)
    const uint32_t fmask = (1u << p.fine_bits) - 1u;
    bool over = false;
    for (uint32_t e = tid; e < cnt; e += kThreads) {
        const uint32_t b = stage_b[e];
        const uint32_t c = b >> p.fine_bits;
        const int32_t slot = gadj[c] + (int32_t)e;
        if ((unsigned long long)(uint32_t)slot < (rbase ? rbase[c + 1] - rbase[c] : (unsigned long long)p.capc)) {
            const size_t dst = (rbase ? (size_t)rbase[c] : (size_t)c * p.capc) + (uint32_t)slot;
            reg_keys[dst] = stage_key[e];
            reg_fine[dst] = (uint16_t)(b & fmask);
            if (PERM) reg_idx[dst] = stage_idx[e];
        } else {
            over = true;
        }
    }
    if (over) atomicAdd(&st->region_overflow, 1ull);
}

// Global starts of the coarse buckets: exclusive scan of the exact bucket sizes (the final
// region cursors), one CTA.  starts[C] = n.
// K0: per-call reset of the status word and the per-coarse-bucket bookkeeping (one launch
// instead of a host copy and three memsets).
static __global__ void __launch_bounds__(256)
k0_init(DevStatus* __restrict__ st, unsigned long long* __restrict__ range_start, uint64_t nranges,
        uint32_t* __restrict__ big_mark, uint32_t* __restrict__ cursor, uint32_t C, uint32_t* __restrict__ est) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < sizeof(DevStatus) / 8) reinterpret_cast<unsigned long long*>(st)[i] = i == 0 ? ~0ull : 0ull;
    if (i < nranges) range_start[i] = ~0ull;
    if (i < C) {
        big_mark[i] = 0u;
        cursor[i] = 0u;
        if (est) est[i] = 0u;
    }
}

static __global__ void __launch_bounds__(1024)
k2_coarse_starts(const uint32_t* __restrict__ cursor, uint32_t C, unsigned long long* __restrict__ starts,
                 bool one_pass, uint32_t mid_cap = 0, uint32_t* __restrict__ mid_list = nullptr,
                 DevStatus* __restrict__ st = nullptr) {
    __shared__ uint32_t scratch[64];
    __shared__ unsigned long long carry;
    // coarse buckets larger than the K3 primary pass holds (mid_cap > 0): listed here, so the
    // secondary pass can run concurrently with the primary one instead of after it
    if (mid_cap) {
        for (uint32_t c = threadIdx.x; c < C; c += 1024u)
            if (cursor[c] > mid_cap) mid_list[atomicAdd(&st->mid_count, 1ull)] = c;
    }
    const uint32_t k = (C + 1023u) / 1024u;              // counts per thread
    if (one_pass && k <= 16u) {                          // (one_pass: the total fits 32 bits)
        // one pass: every thread loads its k consecutive counts at once (one memory latency),
        // one block scan of the per-thread sums, then the k starts
        const uint32_t c0 = threadIdx.x * k;
        uint32_t v[16], tot = 0;
#pragma unroll
        for (uint32_t q = 0; q < 16; ++q) {
            v[q] = (q < k && c0 + q < C) ? cursor[c0 + q] : 0u;
            tot += v[q];
        }
        uint32_t all;
        unsigned long long run = block_exclusive_scan<1024>(tot, scratch, &all);
#pragma unroll
        for (uint32_t q = 0; q < 16; ++q) {
            if (q < k && c0 + q < C) {
                starts[c0 + q] = run;
                run += v[q];
            }
        }
        if (threadIdx.x == 0) starts[C] = all;
        return;
    }
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < C; b0 += 1024) {
        const uint32_t c = b0 + threadIdx.x;
        const uint32_t v = c < C ? cursor[c] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<1024>(v, scratch, &tot);
        if (c < C) starts[c] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) starts[C] = carry;
}

}  // namespace mlsort
