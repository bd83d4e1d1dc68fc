// k1_bench.cu -- standalone timing of K1 variants (k1_ws template knobs) on a C2-shaped input
// (2^26 f32 keys ~ N(0,1), M = 32, B = 2^26, C = 4096 coarse buckets).  Development tool, not
// part of libmlsort:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o k1b scripts/k1_bench.cu
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include <algorithm>

#include "../paper_1805_04272_b200/csrc/common.cuh"
#include "../paper_1805_04272_b200/csrc/predict.cuh"
#include "../paper_1805_04272_b200/csrc/k1_partition.cuh"
#include "../paper_1805_04272_b200/csrc/k1_ws.cuh"

using namespace mlsort;

__global__ void gen_keys(float* k, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
        float s = 0.f;
        for (int r = 0; r < 4; ++r) {
            h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12; h *= 0x297a2d39u; h ^= h >> 15;
            s += (float)(h >> 8) * (1.0f / 16777216.0f);
        }
        k[i] = (s - 2.0f) * 1.7320508f;       // ~N(0,1)
    }
}

template <typename K>
float time_kernel(K launch, uint32_t* cursor, uint32_t C, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f, tot = 0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaMemset(cursor, 0, C * 4);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) { best = ms < best ? ms : best; tot += ms; }
    }
    return tot / reps;
}

int main() {
    const uint64_t n = 1ull << 26, B = 1ull << 26;
    const uint32_t fb = 14, C = (uint32_t)(B >> fb), M = 32;
    const uint32_t capc = 65600;
    float* keys;
    cudaMalloc(&keys, n * 4);
    gen_keys<<<148 * 8, 256>>>(keys, n);
    const uint64_t slots = (uint64_t)C * capc + 16384;
    float* rk;
    uint16_t* rf;
    uint32_t *cursor;
    DevStatus* st;
    cudaMalloc(&rk, slots * 4);
    cudaMalloc(&rf, slots * 2);
    cudaMalloc(&cursor, C * 4);
    cudaMalloc(&st, sizeof(DevStatus));
    cudaMemset(st, 0, sizeof(DevStatus));

    FoldedWeights fw;
    std::memset(&fw, 0, sizeof(fw));
    const int S = 26;
    for (uint32_t j = 0; j < M; ++j) {       // monotone increasing net: centres spread over [-3, 3]
        const double slope = 3.0 + 0.2 * j, centre = -3.0 + 6.0 * j / (M - 1);
        fw.A[j] = (float)(-slope * 1.4426950408889634);
        fw.C[j] = (float)(slope * centre * 1.4426950408889634);
        fw.W[j] = (float)std::ldexp(1.0 / M, S);
        fw.Wn[j] = -fw.W[j];
    }
    auto pair = [](float v) { uint32_t b; std::memcpy(&b, &v, 4); return ((unsigned long long)b << 32) | b; };
    double ulo = -INFINITY, uhi = INFINITY;
    for (uint32_t j = 0; j < M; ++j) {
        const double A = fw.A[j], Cc = fw.C[j];
        if (A < 0) ulo = std::max(ulo, (59.0 - Cc) / A);
        else if (A > 0) uhi = std::min(uhi, (59.0 - Cc) / A);
    }
    fw.u_safe_lo = (float)ulo + 1e-3f;
    fw.u_safe_hi = uhi == INFINITY ? INFINITY : (float)uhi;
    printf("safe u range [%g, %g]\n", fw.u_safe_lo, fw.u_safe_hi);
    fw.one2 = pair(1.0f);
    fw.k1_2 = pair(2.001281198f);
    fw.magic2 = pair(12582912.0f);
    K1Params kp;
    std::memset(&kp, 0, sizeof(kp));
    kp.lo_d = -5; kp.hi_d = 5; kp.x0_d = 0; kp.x0_f = 0; kp.lo_tf = -5; kp.hi_tf = 5;
    kp.bm.Bf = (float)B; kp.bm.Bm1 = (uint32_t)(B - 1); kp.bm.B = B; kp.bm.S = S;
    kp.fine_bits = fb; kp.num_coarse = C; kp.capc = capc; kp.n = n;

    const double acts = (double)n * M;
    auto run = [&](auto kern, int kgw_tile_keys, const char* name) {
        const uint32_t T = (uint32_t)ws_tile<float>();
        kp.num_tiles = (uint32_t)((n + T - 1) / T);
        const size_t sm = k1ws_smem_bytes(4, T, C);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const float ms = time_kernel([&] { kern<<<148, ws_threads(false), sm>>>(keys, kp, rk, rf, nullptr, cursor, st, nullptr, fw); },
                                     cursor, C, 5);
        cudaError_t e = cudaGetLastError();
        printf("%-40s %8.3f ms  %6.2f act/clk/SM @1965  (%s)\n", name, ms, acts / (ms * 1e-3) / 148 / 1.965e9,
               cudaGetErrorString(e));
        (void)kgw_tile_keys;
    };
    run(k1_ws<float, 32, kPredPacked, false, 8, true>, 0, "ws packed KG8 + partition");
    run(k1_ws<float, 32, kPredPacked, false, 8, false>, 0, "ws packed KG8, no partition");
    run(k1_ws<float, 32, kPredPacked, false, 4, true>, 0, "ws packed KG4 + partition");
    run(k1_ws<float, 32, kPredPacked, false, 4, false>, 0, "ws packed KG4, no partition");
    run(k1_ws<float, 32, kPredMixed, false, 8, true>, 0, "ws mixed KG8 + partition");
    run(k1_ws<float, 32, kPredMufu, false, 8, false>, 0, "ws mufu KG8, no partition");
    return 0;
}
