// host_train.cpp -- mlsort_fit: the training step that precedes the hot path (host, untimed).
//
// The paper builds the training sequence A by drawing N0 keys at random, sorts it into A'
// and fits the network to the pairs (a'_i, i/N0) (§2 l.43); the GVM is trained
// "based on Monte-Carlo algorithm instead of back propagation" (l.63) with no rule given.
// This trainer follows SPEC.md's reading (S:133, S:170-S:172): single-coordinate Gaussian
// proposals, accept iff the MSE strictly decreases and the Eq. 4 sign condition holds.
// Repo decisions: quantile initialisation of the neuron centres
// (instead of S:172's random start), proposal scales tied to each neuron's width, and
// training on at most `max_pairs` evenly spaced ranks of the sorted sample.
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

using mlsort::Weights;

namespace {

struct Rng {   // xoshiro256** seeded by splitmix64
    uint64_t s[4];
    explicit Rng(uint64_t seed) {
        for (int i = 0; i < 4; ++i) {
            seed += 0x9E3779B97F4A7C15ull;
            uint64_t z = seed;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            s[i] = z ^ (z >> 31);
        }
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform() { return (next() >> 11) * 0x1.0p-53; }
    double normal() {
        double u1 = ((next() >> 11) + 1) * 0x1.0p-53, u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

inline double logistic(double t) { return 1.0 / (1.0 + std::exp(-t)); }

}  // namespace

extern "C" int mlsort_train_cfg_default(mlsort_train_cfg* cfg, uint32_t m) {
    if (!cfg || m < 1 || m > mlsort::kMaxNeurons) return MLSORT_ERR_INVALID_ARG;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->m = m;
    cfg->max_pairs = 4096;
    cfg->iterations = 6000 + 250ull * m;
    cfg->perturb_scale = 0.05;
    cfg->target_loss = 0.0;
    cfg->seed = 1;
    cfg->enforce_monotone = 1;
    return MLSORT_OK;
}

extern "C" int mlsort_fit(const void* h_sample, uint64_t n0, mlsort_dtype dtype,
                          const mlsort_train_cfg* cfg_in, mlsort_weights** out) {
    if (!h_sample || !out || n0 < 1 || (dtype != MLSORT_F32 && dtype != MLSORT_F64))
        return MLSORT_ERR_INVALID_ARG;
    mlsort_train_cfg cfg;
    if (cfg_in) cfg = *cfg_in;
    else mlsort_train_cfg_default(&cfg, 16);
    if (cfg.m < 1 || cfg.m > mlsort::kMaxNeurons || cfg.perturb_scale <= 0.0) return MLSORT_ERR_INVALID_ARG;
    const uint32_t M = cfg.m;

    // A' = sorted training sequence, ascending convention (reading A1).
    std::vector<double> a(n0);
    for (uint64_t i = 0; i < n0; ++i) {
        a[i] = dtype == MLSORT_F32 ? (double)static_cast<const float*>(h_sample)[i]
                                   : static_cast<const double*>(h_sample)[i];
        if (!std::isfinite(a[i])) return MLSORT_ERR_NONFINITE_KEY;
    }
    std::sort(a.begin(), a.end());
    const double lo = a.front(), hi = a.back();
    if (!(lo < hi)) return MLSORT_ERR_TRAIN;                  // S:134 degenerate range

    // Pairs (a'_i, i/N0), i = 0..N0-1, evenly subsampled by rank; the first and the
    // last rank are always kept.
    uint64_t P = (cfg.max_pairs && cfg.max_pairs < n0) ? cfg.max_pairs : n0;
    if (P < 2) P = n0;
    std::vector<double> xh(P), tgt(P);
    for (uint64_t k = 0; k < P; ++k) {
        uint64_t i = (P == n0) ? k : (uint64_t)((double)k * (double)(n0 - 1) / (double)(P - 1));
        xh[k] = 2.0 * (a[i] - lo) / (hi - lo) - 1.0;
        tgt[k] = (double)i / (double)n0;
    }

    // Initialisation (repo decision): neuron j is a logistic step of height 1/M centred at
    // the sample quantile (j+0.5)/M, with a width matched to the local quantile spacing.
    std::vector<double> w1(M, 1.0), w2(M, 1.0 / M), b(M), beta(M);
    auto quant = [&](double q) {
        double r = q * (double)(n0 - 1);
        uint64_t i = (uint64_t)r;
        double f = r - (double)i;
        double v = i + 1 < n0 ? a[i] * (1 - f) + a[i + 1] * f : a[i];
        return 2.0 * (v - lo) / (hi - lo) - 1.0;
    };
    for (uint32_t j = 0; j < M; ++j) b[j] = quant((j + 0.5) / M);
    for (uint32_t j = 0; j < M; ++j) {
        double left = quant(std::max(0.0, (j + 0.0) / M)), right = quant(std::min(1.0, (j + 1.0) / M));
        double d = std::max(right - left, 1e-7);
        beta[j] = 3.0 / d;
    }

    // Term matrix T[j][k] = w2_j f0(beta_j (w1_j x^_k - b_j)) and the running sum Y.
    std::vector<double> T((size_t)M * P), Y(P, 0.0), col(P);
    auto term_col = [&](double w1j, double w2j, double bj, double betaj, double* dst) {
        for (uint64_t k = 0; k < P; ++k) dst[k] = w2j * logistic(betaj * (w1j * xh[k] - bj));
    };
    auto rebuild = [&]() {
        std::fill(Y.begin(), Y.end(), 0.0);
        for (uint32_t j = 0; j < M; ++j) {
            term_col(w1[j], w2[j], b[j], beta[j], &T[(size_t)j * P]);
            for (uint64_t k = 0; k < P; ++k) Y[k] += T[(size_t)j * P + k];
        }
    };
    auto mse = [&]() {
        double s = 0;
        for (uint64_t k = 0; k < P; ++k) { double e = Y[k] - tgt[k]; s += e * e; }
        return s / (double)P;
    };
    rebuild();
    double loss = mse();

    // Range constraint (repo decision): the fitted CDF may not exceed
    // 1 - 1/(2 N0) at the largest sample key.  Without it the MSE optimum overshoots 1 near
    // the top and every key above that point collapses into the clamped last bucket
    // ("r_j would fall out of the range [0, N]").
    const double y_top_max = 1.0 - 0.5 / (double)n0;
    Rng rng(cfg.seed);
    uint64_t accepts = 0;
    for (uint64_t it = 0; it < cfg.iterations && loss > cfg.target_loss; ++it) {
        uint32_t j = (uint32_t)(rng.next() % M);
        uint32_t which = (uint32_t)(rng.next() & 3);
        double nw1 = w1[j], nw2 = w2[j], nb = b[j], nbeta = beta[j];
        double g = rng.normal() * cfg.perturb_scale;
        switch (which) {
            case 0: nw1 += g * std::fabs(nw1) + g * 1e-3; break;
            case 1: nw2 += g * std::max(std::fabs(nw2), 1.0 / M); break;
            case 2: nb += g * 2.0 * std::fabs(nw1) / std::max(std::fabs(nbeta * nw1), 1e-300) ; break;
            default: nbeta += g * std::fabs(nbeta) + g * 1e-3; break;
        }
        if (cfg.enforce_monotone && nw1 * nw2 * nbeta < 0.0) continue;     // Eq. 4
        if (!std::isfinite(nw1 * nw2 * nb * nbeta)) continue;
        term_col(nw1, nw2, nb, nbeta, col.data());
        const double* old = &T[(size_t)j * P];
        double s = 0;
        for (uint64_t k = 0; k < P; ++k) { double e = Y[k] - old[k] + col[k] - tgt[k]; s += e * e; }
        double nl = s / (double)P;
        if (Y[P - 1] - old[P - 1] + col[P - 1] > y_top_max && nl < loss) continue;
        if (nl < loss) {                                                   // S:133 strict decrease
            for (uint64_t k = 0; k < P; ++k) Y[k] += col[k] - old[k];
            std::copy(col.begin(), col.end(), T.begin() + (size_t)j * P);
            w1[j] = nw1; w2[j] = nw2; b[j] = nb; beta[j] = nbeta;
            loss = nl;
            if (++accepts % 1024 == 0) { rebuild(); loss = mse(); }
        }
    }
    rebuild();
    loss = mse();
    int rc = mlsort_weights_create(M, w1.data(), w2.data(), b.data(), beta.data(), lo, hi, out);
    if (rc == MLSORT_OK) {
        Weights* w = reinterpret_cast<Weights*>(*out);
        w->final_loss = loss;
        w->seed = cfg.seed;
    }
    return rc;
}
