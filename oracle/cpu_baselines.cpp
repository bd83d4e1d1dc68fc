// cpu_baselines.cpp -- conventional CPU sorts timed beside the oracle (SURVEY.md §8(d)
// "std::sort and std::stable_sort, 1 thread, on the same keys": the analogue of the paper's
// NumPy quicksort / mergesort context numbers).  TEST / BENCH INFRASTRUCTURE ONLY,
// like the rest of oracle/: the product never loads it.
#include <algorithm>
#include <cstdint>

extern "C" {

// Sort keys[0, n) in place with std::sort (stable == 0) or std::stable_sort (stable != 0),
// operator< on the keys (finite keys: the same order as IEEE totalOrder up to -0 / +0).
void cpu_std_sort_f32(float* keys, uint64_t n, int stable) {
    if (stable) std::stable_sort(keys, keys + n);
    else std::sort(keys, keys + n);
}

void cpu_std_sort_f64(double* keys, uint64_t n, int stable) {
    if (stable) std::stable_sort(keys, keys + n);
    else std::sort(keys, keys + n);
}

}
