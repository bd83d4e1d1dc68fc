// k3_bench.cu -- standalone timing of K3 (k3_local_sort) on synthetic C2-shaped regions
// (4096 coarse buckets of ~16384 keys, 16384 rank buckets each), with per-phase cycle
// accounting.  Development tool, not part of libmlsort:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLSORT_K3L_TIMING -I include \
//        -o k3b scripts/k3_bench.cu
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include "../paper_1805_04272_b200/csrc/common.cuh"
#include "../paper_1805_04272_b200/csrc/k3_local.cuh"

using namespace mlsort;

__device__ __forceinline__ uint32_t hsh(uint32_t h) {
    h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12; h *= 0x297a2d39u; h ^= h >> 15;
    return h;
}

// region of coarse bucket c: n_c elements, fine id uniform in [0, kfine), key bits increasing in
// (c, fine) with 2 random low bits (so a rank bucket holds ties and distinct keys)
__global__ void gen_regions(float* rk, uint16_t* rf, const unsigned long long* starts, uint32_t C, uint32_t capc,
                            uint32_t kfine) {
    const uint32_t c = blockIdx.x;
    const uint32_t n = (uint32_t)(starts[c + 1] - starts[c]);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t h = hsh(c * 0x9E3779B1u + i * 0x85EBCA77u);
        const uint32_t f = h % kfine;
        const uint32_t bits = 0x3F800000u + ((((uint32_t)c * kfine + f) << 2) | (hsh(h) & 3u));
        rk[(size_t)c * capc + i] = __uint_as_float(bits);
        rf[(size_t)c * capc + i] = (uint16_t)f;
    }
}

int main() {
    const uint32_t C = getenv("K3_FB13") ? 8192 : 4096, kfine = getenv("K3_FB13") ? 8192 : 16384;
    const uint32_t capc = 4 * kfine + 64;
    std::vector<unsigned long long> starts(C + 1, 0);
    uint32_t s = 12345;
    for (uint32_t c = 0; c < C; ++c) {
        s = s * 1664525u + 1013904223u;
        const uint32_t nc = kfine - 256 + (s >> 23);     // kfine +- 256
        starts[c + 1] = starts[c] + nc;
    }
    const uint64_t n = starts[C];
    float *rk, *out;
    uint16_t* rf;
    unsigned long long *d_starts, *range_start;
    uint32_t *big_list, *big_mark, *mid_list;
    DevStatus* st;
    cudaMalloc(&rk, (size_t)C * capc * 4);
    cudaMalloc(&rf, (size_t)C * capc * 2);
    cudaMalloc(&out, n * 4);
    cudaMalloc(&d_starts, (C + 1) * 8);
    cudaMalloc(&range_start, C * 8);
    cudaMalloc(&big_list, C * 4);
    cudaMalloc(&big_mark, C * 4);
    cudaMalloc(&mid_list, C * 4);
    cudaMalloc(&st, sizeof(DevStatus));
    cudaMemcpy(d_starts, starts.data(), (C + 1) * 8, cudaMemcpyHostToDevice);
    gen_regions<<<C, 256>>>(rk, rf, d_starts, C, capc, kfine);
    K3LParams kp;
    kp.capc = capc;
    kp.num_coarse = C;
    kp.kfine = kfine;
    const int NTB = getenv("K3_NT512") ? 512 : 1024;
    kp.cap = k3l_cap_for(NTB == 512 ? 115712 : 232448, 4, false, kfine, NTB);
    kp.verify = getenv("K3_VERIFY") ? 1 : 0;
    kp.secondary = 0;
    kp.to_mid = 0;
    const size_t sm = k3l_smem_bytes(4, false, kfine, kp.cap, NTB);
    auto kern = NTB == 512 ? k3_local_sort<float, false, 512> : k3_local_sort<float, false, 1024>;
    const int grid = NTB == 512 ? 296 : 148;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaMemset(st, 0, sizeof(DevStatus));
        cudaMemset(big_mark, 0, C * 4);
        cudaEventRecord(a);
        kern<<<grid, NTB, sm>>>(kp, rk, rf, nullptr, d_starts, out, nullptr, range_start, st, big_list, big_mark,
                                      mid_list, &st->ticket3, nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = std::min(best, ms);
    }
    printf("k3_local_sort: n=%llu cap=%u smem=%zu  best %.3f ms  (%.1f GB/s of 10 B/key)  %s\n",
           (unsigned long long)n, kp.cap, sm, best, n * 10.0 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    // per-phase cycles (last run), averaged over CTAs, per coarse bucket
    static unsigned long long ph[1024][8];
    cudaMemcpyFromSymbol(ph, g_k3l_phase, sizeof(ph));
    const char* names[8] = {"loop top / ticket", "zero+hist", "scan", "placement", "fixup in smem", "big buckets",
                            "verify+store", "-"};
    double tot = 0;
    for (int i = 0; i < 7; ++i) {
        double sum = 0;
        for (int bI = 0; bI < grid; ++bI) sum += ph[bI][i];
        sum /= grid;
        tot += sum;
        printf("  phase %-20s %10.0f cycles per CTA  (%6.0f per bucket)\n", names[i], sum, sum / ((double)C / grid));
    }
    printf("  total %.0f cycles per CTA\n", tot);
    // check sortedness
    std::vector<float> h(n);
    cudaMemcpy(h.data(), out, n * 4, cudaMemcpyDeviceToHost);
    uint64_t bad = 0;
    for (uint64_t i = 1; i < n; ++i) bad += h[i] < h[i - 1];
    DevStatus hs;
    cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
    printf("  inversions %llu, local_repairs %llu, mid %llu, big %llu\n", (unsigned long long)bad, hs.local_repairs,
           hs.mid_count, hs.big_count);
    return 0;
}
