// internal.h -- shared declarations of libmlsort.so (not part of the public ABI).
#pragma once

#include <cstdint>
#include <atomic>
#include <vector>

#include "../../include/mlsort.h"

namespace mlsort {

constexpr uint32_t kMaxNeurons = 64;   // padded to 16/32/64 in the kernels

// Host-resident GVM parameters (Eq. 3 symbols; S:91-S:97).  Immutable after creation.
// process-unique identity of a weights handle (keys the folded-constant cache in mlsort.cu;
// handles are immutable, so (serial, key dtype) determines the folded constants)
inline uint64_t next_weights_serial() {
    static std::atomic<uint64_t> counter{1};
    return counter.fetch_add(1);
}

struct Weights {
    uint64_t serial = next_weights_serial();
    uint32_t m = 0;
    std::vector<double> w1, w2, b, beta;
    double lo = 0.0, hi = 1.0;          // input normalisation bounds (reading A3)
    double final_loss = __builtin_nan("");
    uint64_t seed = 0;
};

bool monotone(const Weights& w);

}  // namespace mlsort
