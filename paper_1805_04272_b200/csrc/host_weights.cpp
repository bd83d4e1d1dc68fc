// host_weights.cpp -- GVM parameter handles, versioned JSON persistence, the Eq. 4
// monotonicity check and the Monte-Carlo trainer (host side of libmlsort.so).
//
// Paper: Zhao & Luo, arXiv 1805.04272 (PAPER.md, cited "P:n"); SPEC.md cited "S:n".
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

using mlsort::Weights;

// ------------------------------------------------------------------ status strings

extern "C" const char* mlsort_status_string(int s) {
    switch (s) {
        case MLSORT_OK: return "ok";
        case MLSORT_ERR_INVALID_ARG: return "invalid argument";
        case MLSORT_ERR_IO: return "I/O error";
        case MLSORT_ERR_PARSE: return "weights JSON parse error";
        case MLSORT_ERR_INVALID_WEIGHTS: return "invalid weights";
        case MLSORT_ERR_NONFINITE_KEY: return "non-finite key (NaN or Inf)";
        case MLSORT_ERR_CUDA: return "CUDA error";
        case MLSORT_ERR_WORKSPACE: return "workspace too small or misaligned";
        case MLSORT_ERR_CAPACITY: return "output capacity exceeded";
        case MLSORT_ERR_TRAIN: return "degenerate training sample";
        case MLSORT_ERR_INTERNAL: return "internal error";
        case MLSORT_ERR_NCCL: return "NCCL unavailable or failed";
        default: return "unknown status";
    }
}

extern "C" const char* mlsort_version(void) { return "mlsort-b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------------ weights handle

static int validate(uint32_t m, const double* w1, const double* w2, const double* b,
                    const double* beta, double lo, double hi) {
    if (m < 1 || m > mlsort::kMaxNeurons) return MLSORT_ERR_INVALID_WEIGHTS;
    for (uint32_t j = 0; j < m; ++j)
        if (!std::isfinite(w1[j]) || !std::isfinite(w2[j]) || !std::isfinite(b[j]) ||
            !std::isfinite(beta[j]))
            return MLSORT_ERR_INVALID_WEIGHTS;
    if (!std::isfinite(lo) || !std::isfinite(hi) || !(lo < hi)) return MLSORT_ERR_INVALID_WEIGHTS;
    return MLSORT_OK;
}

extern "C" int mlsort_weights_create(uint32_t m, const double* w1, const double* w2,
                                     const double* b, const double* beta, double lo,
                                     double hi, mlsort_weights** out) {
    if (!w1 || !w2 || !b || !beta || !out) return MLSORT_ERR_INVALID_ARG;
    int rc = validate(m, w1, w2, b, beta, lo, hi);
    if (rc) return rc;
    Weights* w = new (std::nothrow) Weights();
    if (!w) return MLSORT_ERR_INTERNAL;
    w->m = m;
    w->w1.assign(w1, w1 + m);
    w->w2.assign(w2, w2 + m);
    w->b.assign(b, b + m);
    w->beta.assign(beta, beta + m);
    w->lo = lo;
    w->hi = hi;
    *out = reinterpret_cast<mlsort_weights*>(w);
    return MLSORT_OK;
}

extern "C" void mlsort_weights_free(mlsort_weights* w) { delete reinterpret_cast<Weights*>(w); }

extern "C" int mlsort_weights_get(const mlsort_weights* wh, uint32_t* m, double* w1, double* w2,
                                  double* b, double* beta, double* lo, double* hi,
                                  double* final_loss) {
    if (!wh) return MLSORT_ERR_INVALID_ARG;
    const Weights* w = reinterpret_cast<const Weights*>(wh);
    if (m) *m = w->m;
    if (w1) std::copy(w->w1.begin(), w->w1.end(), w1);
    if (w2) std::copy(w->w2.begin(), w->w2.end(), w2);
    if (b) std::copy(w->b.begin(), w->b.end(), b);
    if (beta) std::copy(w->beta.begin(), w->beta.end(), beta);
    if (lo) *lo = w->lo;
    if (hi) *hi = w->hi;
    if (final_loss) *final_loss = w->final_loss;
    return MLSORT_OK;
}

// Eq. 4 written for the ascending convention (reading A1/A22): the per-neuron
// condition w1*w2*beta >= 0 makes every term of dy/dx non-negative because the
// logistic's derivative is positive; it is sufficient on all of R.
bool mlsort::monotone(const Weights& w) {
    for (uint32_t j = 0; j < w.m; ++j)
        if (w.w1[j] * w.w2[j] * w.beta[j] < 0.0) return false;
    return true;
}

extern "C" int mlsort_weights_check_monotone(const mlsort_weights* wh) {
    if (!wh) return -MLSORT_ERR_INVALID_ARG;
    return mlsort::monotone(*reinterpret_cast<const Weights*>(wh)) ? 1 : 0;
}

// ------------------------------------------------------------------ JSON

namespace {

struct JsonParser {
    const char* p;
    const char* end;
    bool ok = true;

    void ws() { while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p; }
    bool lit(char c) { ws(); if (p < end && *p == c) { ++p; return true; } return false; }
    bool str(std::string& s) {
        ws();
        if (p >= end || *p != '"') return false;
        ++p;
        s.clear();
        while (p < end && *p != '"') {
            if (*p == '\\') { ++p; if (p >= end) return false; }
            s.push_back(*p++);
        }
        if (p >= end) return false;
        ++p;
        return true;
    }
    bool num(double& v) {
        ws();
        char* e = nullptr;
        v = std::strtod(p, &e);
        if (e == p) return false;
        p = e;
        return true;
    }
    bool arr(std::vector<double>& a) {
        if (!lit('[')) return false;
        a.clear();
        if (lit(']')) return true;
        do {
            double v;
            if (!num(v)) return false;
            a.push_back(v);
        } while (lit(','));
        return lit(']');
    }
    bool skip_value() {   // strings, numbers, literals, nested arrays/objects
        ws();
        if (p >= end) return false;
        if (*p == '"') { std::string s; return str(s); }
        if (*p == '[' || *p == '{') {
            char open = *p, close = open == '[' ? ']' : '}';
            int depth = 0;
            bool in_str = false;
            for (; p < end; ++p) {
                if (in_str) { if (*p == '\\') ++p; else if (*p == '"') in_str = false; continue; }
                if (*p == '"') in_str = true;
                else if (*p == open) ++depth;
                else if (*p == close && --depth == 0) { ++p; return true; }
            }
            return false;
        }
        if (!strncmp(p, "true", 4)) { p += 4; return true; }
        if (!strncmp(p, "false", 5)) { p += 5; return true; }
        if (!strncmp(p, "null", 4)) { p += 4; return true; }
        double v;
        return num(v);
    }
};

}  // namespace

extern "C" int mlsort_weights_load(const char* path, mlsort_weights** out) {
    if (!path || !out) return MLSORT_ERR_INVALID_ARG;
    std::ifstream f(path, std::ios::binary);
    if (!f) return MLSORT_ERR_IO;
    std::stringstream ss;
    ss << f.rdbuf();
    std::string text = ss.str();
    JsonParser J{text.data(), text.data() + text.size()};
    std::vector<double> w1, w2, b, beta;
    double m = -1, lo = NAN, hi = NAN, loss = NAN, seed = 0, version = -1;
    std::string format, activation = "logistic";
    bool have[6] = {false, false, false, false, false, false};
    if (!J.lit('{')) return MLSORT_ERR_PARSE;
    if (!J.lit('}')) {
        do {
            std::string key;
            if (!J.str(key) || !J.lit(':')) return MLSORT_ERR_PARSE;
            bool good = true;
            if (key == "w1") good = J.arr(w1), have[0] = true;
            else if (key == "w2") good = J.arr(w2), have[1] = true;
            else if (key == "b") good = J.arr(b), have[2] = true;
            else if (key == "beta") good = J.arr(beta), have[3] = true;
            else if (key == "m") good = J.num(m);
            else if (key == "input_lo") good = J.num(lo), have[4] = true;
            else if (key == "input_hi") good = J.num(hi), have[5] = true;
            else if (key == "final_loss") { J.ws(); if (!strncmp(J.p, "null", 4)) J.p += 4; else good = J.num(loss); }
            else if (key == "seed") good = J.num(seed);
            else if (key == "version") good = J.num(version);
            else if (key == "format") good = J.str(format);
            else if (key == "activation") good = J.str(activation);
            else good = J.skip_value();
            if (!good) return MLSORT_ERR_PARSE;
        } while (J.lit(','));
        if (!J.lit('}')) return MLSORT_ERR_PARSE;
    }
    for (bool h : have) if (!h) return MLSORT_ERR_PARSE;
    if (!format.empty() && format != "mlsort-gvm") return MLSORT_ERR_PARSE;
    if (version > 1) return MLSORT_ERR_PARSE;
    if (activation != "logistic") return MLSORT_ERR_INVALID_WEIGHTS;   // reading A2
    size_t mm = w1.size();
    if (w2.size() != mm || b.size() != mm || beta.size() != mm) return MLSORT_ERR_INVALID_WEIGHTS;
    if (m >= 0 && (size_t)m != mm) return MLSORT_ERR_INVALID_WEIGHTS;
    int rc = mlsort_weights_create((uint32_t)mm, w1.data(), w2.data(), b.data(), beta.data(), lo, hi, out);
    if (rc == MLSORT_OK) {
        Weights* w = reinterpret_cast<Weights*>(*out);
        w->final_loss = loss;
        w->seed = (uint64_t)seed;
    }
    return rc;
}

static void put_arr(FILE* f, const char* name, const std::vector<double>& a) {
    fprintf(f, "  \"%s\": [", name);
    for (size_t i = 0; i < a.size(); ++i) fprintf(f, "%s%.17g", i ? ", " : "", a[i]);
    fprintf(f, "],\n");
}

extern "C" int mlsort_weights_save(const mlsort_weights* wh, const char* path) {
    if (!wh || !path) return MLSORT_ERR_INVALID_ARG;
    const Weights* w = reinterpret_cast<const Weights*>(wh);
    FILE* f = fopen(path, "w");
    if (!f) return MLSORT_ERR_IO;
    fprintf(f, "{\n  \"format\": \"mlsort-gvm\",\n  \"version\": 1,\n  \"activation\": \"logistic\",\n");
    fprintf(f, "  \"m\": %u,\n", w->m);
    put_arr(f, "w1", w->w1);
    put_arr(f, "w2", w->w2);
    put_arr(f, "b", w->b);
    put_arr(f, "beta", w->beta);
    fprintf(f, "  \"input_lo\": %.17g,\n  \"input_hi\": %.17g,\n", w->lo, w->hi);
    if (std::isfinite(w->final_loss)) fprintf(f, "  \"final_loss\": %.17g,\n", w->final_loss);
    else fprintf(f, "  \"final_loss\": null,\n");
    fprintf(f, "  \"seed\": %llu\n}\n", (unsigned long long)w->seed);
    int bad = ferror(f);
    if (fclose(f) != 0 || bad) return MLSORT_ERR_IO;
    return MLSORT_OK;
}
