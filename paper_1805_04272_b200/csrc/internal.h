// internal.h -- shared declarations of libmlsort.so (not part of the public ABI).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/mlsort.h"

namespace mlsort {

constexpr uint32_t kMaxNeurons = 64;   // padded to 16/32/64 in the kernels

// Host-resident GVM parameters (Eq. 3 symbols; S:91-S:97).  Immutable after creation.
struct Weights {
    uint32_t m = 0;
    std::vector<double> w1, w2, b, beta;
    double lo = 0.0, hi = 1.0;          // input normalisation bounds (reading A3)
    double final_loss = __builtin_nan("");
    uint64_t seed = 0;
};

bool monotone(const Weights& w);

}  // namespace mlsort
