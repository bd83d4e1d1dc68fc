// comm.cpp -- the multi-GPU path of libmlsort.so (SURVEY.md §8(b) mlsort_comm_*,
// mlsort_sort_dist; §8(e)).  One process per GPU; the library owns an NCCL communicator.
//
// PAPER.md §2 l.94 ("the prediction of each number is independent ... requires very little
// networking workload") and l.134 ("both N and M can be separated"): rank g holds a
// contiguous slice of the keys, predicts the GLOBAL rank bucket b of each (Eq. 3, l.65) and
// sends it to the owner floor(b*G/B), so rank g owns the rank range [gB/G, (g+1)B/G) (BJ:5).
// One grouped NCCL all-to-all-v moves the records (key, b, global index); the receiver sorts
// them without predicting again (b travels with the key).  Concatenating the ranks' runs in
// rank order is the global sorted array, bit-identical to the 1-GPU result:
// the owner is monotone in b, and a receiver lays its input out in source-rank order, so
// equal keys keep increasing global index.
//
// NCCL is loaded at mlsort_comm_init time (dlopen of libnccl.so.2, normally already mapped by
// the process's PyTorch), so libmlsort.so itself loads on hosts without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

using namespace mlsort;

struct mlsort_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
};

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {std::getenv("MLSORT_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            fprintf(stderr, "mlsort: cannot load NCCL (libnccl.so.2; set MLSORT_NCCL_LIB): %s\n", dlerror());
            return;
        }
#define SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
        SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(AllGather); SYM(Send); SYM(Recv);
        SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Send && api.Recv &&
                 api.GroupStart && api.GroupEnd && api.GetErrorString;
    });
    return api.ok ? &api : nullptr;
}

#define NC(x)                                                                                    \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess) {                                                                 \
            fprintf(stderr, "mlsort: NCCL error %s at %s:%d\n", nccl()->GetErrorString(r_),      \
                    __FILE__, __LINE__);                                                         \
            return MLSORT_ERR_NCCL;                                                              \
        }                                                                                        \
    } while (0)
#define CU(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            fprintf(stderr, "mlsort: CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                    __LINE__);                                                                   \
            return MLSORT_ERR_CUDA;                                                              \
        }                                                                                        \
    } while (0)

constexpr uint64_t kAl = 256;
inline uint64_t al(uint64_t x) { return (x + kAl - 1) / kAl * kAl; }

// bucket range [lo, hi) owned by rank g: exactly the b with floor(b*G/B) == g
inline void owner_range(uint64_t g, uint64_t G, uint64_t B, uint64_t& lo, uint64_t& hi) {
    lo = (g * B + G - 1) / G;
    hi = ((g + 1) * B + G - 1) / G;
}

struct DistLayout {
    uint64_t part = 0, rec_keys = 0, rec_b = 0, rec_idx = 0, recv_keys = 0, recv_b = 0, recv_idx = 0, msg = 0,
             rsort = 0, total = 0;
    uint64_t part_bytes = 0, rsort_bytes = 0;
};

// per-rank message of the count exchange: [send counts (G)] [capacity] [status] [bad global index]
// [keyspace] -- G + 4 words; of the boundary exchange: [count, first ord, first idx, last ord,
// last idx] -- 5 words
constexpr int kBnd = 5;

int dist_layout(uint32_t G, uint64_t n_local, uint64_t n_global, mlsort_dtype dt, const mlsort_opts* o, bool perm,
                uint64_t cap, DistLayout& L) {
    const uint64_t ks = dt == MLSORT_F32 ? 4 : 8;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n_global;
    if (B < 1 || B > (1ull << 30)) return MLSORT_ERR_INVALID_ARG;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t r = off;
        off += al(bytes);
        return r;
    };
    int rc = mlsort_dist_partition_workspace_size(n_local, dt, G, &L.part_bytes);
    if (rc) return rc;
    L.part = take(L.part_bytes);
    L.rec_keys = take(n_local * ks);
    L.rec_b = take(n_local * 4);
    L.rec_idx = take(perm ? n_local * 4 : 0);
    L.recv_keys = take(cap * ks);
    L.recv_b = take(cap * 4);
    L.recv_idx = take(perm ? cap * 4 : 0);
    L.msg = take((uint64_t)G * (G + 4 + kBnd) * 8 + (G + 4 + kBnd) * 8);
    // the receive-side sort: this rank's bucket range (monotone model) or all of [0, B)
    uint64_t a = 0, b = 0;
    if (cap > 0) {
        uint64_t lo, hi;
        owner_range(0, G, B, lo, hi);
        uint64_t width = hi - lo;
        for (uint32_t g = 1; g < G; ++g) {
            owner_range(g, G, B, lo, hi);
            width = std::max(width, hi - lo);
        }
        if ((rc = mlsort_sort_records_workspace_size(cap, dt, 0, std::max<uint64_t>(width, 1), &a))) return rc;
        if ((rc = mlsort_sort_records_workspace_size(cap, dt, 0, B, &b))) return rc;
    }
    L.rsort_bytes = std::max(a, b);
    L.rsort = take(L.rsort_bytes);
    L.total = off + kAl;
    return MLSORT_OK;
}

ncclDataType_t key_type(mlsort_dtype dt) { return dt == MLSORT_F32 ? ncclFloat32 : ncclFloat64; }

uint64_t ord_bits(const void* p, mlsort_dtype dt) {
    if (dt == MLSORT_F32) {
        uint32_t u;
        std::memcpy(&u, p, 4);
        return (u & 0x80000000u) ? (uint64_t)(~u) : (uint64_t)(u | 0x80000000u);
    }
    uint64_t u;
    std::memcpy(&u, p, 8);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct Timer {
    bool on = false;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[6] = {};
    int n = 0;
    void start(bool enable, cudaStream_t st) {
        on = enable;
        s = st;
        if (!on) return;
        for (auto& e : ev) cudaEventCreate(&e);
        cudaEventRecord(ev[0], s);
        n = 1;
    }
    void mark() {
        if (on && n < 6) cudaEventRecord(ev[n++], s);
    }
    void finish(mlsort_info* info) {
        if (!on) return;
        cudaEventSynchronize(ev[n - 1]);
        if (info) {
            for (int i = 1; i < n; ++i) cudaEventElapsedTime(&info->phase_ms[i - 1], ev[i - 1], ev[i]);
            cudaEventElapsedTime(&info->phase_ms[5], ev[0], ev[n - 1]);
        }
        for (auto& e : ev) cudaEventDestroy(e);
        on = false;
    }
    ~Timer() {
        if (on)
            for (auto& e : ev) cudaEventDestroy(e);
    }
};

}  // namespace

// ==================================================================== C ABI

extern "C" int mlsort_comm_unique_id(void* out_id) {
    if (!out_id) return MLSORT_ERR_INVALID_ARG;
    NcclApi* api = nccl();
    if (!api) return MLSORT_ERR_NCCL;
    ncclUniqueId id;
    NC(api->GetUniqueId(&id));
    std::memcpy(out_id, &id, sizeof(id));
    return MLSORT_OK;
}

extern "C" int mlsort_comm_init(int nranks, int rank, const void* unique_id, int device, mlsort_comm** out) {
    if (!out || !unique_id || nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || device < 0)
        return MLSORT_ERR_INVALID_ARG;
    *out = nullptr;
    NcclApi* api = nccl();
    if (!api) return MLSORT_ERR_NCCL;
    CU(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    mlsort_comm* c = new mlsort_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = api->CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        fprintf(stderr, "mlsort: ncclCommInitRank: %s\n", api->GetErrorString(r));
        delete c;
        return MLSORT_ERR_NCCL;
    }
    *out = c;
    return MLSORT_OK;
}

extern "C" int mlsort_comm_destroy(mlsort_comm* c) {
    if (!c) return MLSORT_OK;
    int rc = MLSORT_OK;
    if (c->comm && nccl() && nccl()->CommDestroy(c->comm) != ncclSuccess) rc = MLSORT_ERR_NCCL;
    delete c;
    return rc;
}

extern "C" int mlsort_sort_dist_workspace_size(uint32_t nranks, uint64_t n_local, uint64_t n_global, mlsort_dtype dt,
                                               const mlsort_opts* o, int want_perm, uint64_t out_capacity,
                                               uint64_t* bytes) {
    if (!bytes || nranks < 1 || nranks > 64 || (dt != MLSORT_F32 && dt != MLSORT_F64) || n_global >= (1ull << 32))
        return MLSORT_ERR_INVALID_ARG;
    DistLayout L;
    int rc = dist_layout(nranks, n_local, n_global, dt, o, want_perm != 0, out_capacity, L);
    if (rc) return rc;
    *bytes = L.total;
    return MLSORT_OK;
}

extern "C" int mlsort_sort_dist(mlsort_comm* c, const void* d_shard, uint64_t n_local, uint64_t global_offset,
                                uint64_t n_global, mlsort_dtype dt, const mlsort_weights* w, const mlsort_opts* o,
                                void* d_out_keys, uint32_t* d_out_perm, uint64_t out_capacity, uint64_t* out_count,
                                uint64_t* out_global_offset, void* d_ws, uint64_t ws_bytes, void* stream,
                                mlsort_info* info) {
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->bad_index = -1;
    }
    // argument errors are local (not collective): every rank must pass consistent arguments
    if (!c || !c->comm || !w || !out_count || (dt != MLSORT_F32 && dt != MLSORT_F64)) return MLSORT_ERR_INVALID_ARG;
    if (n_global >= (1ull << 32) || global_offset + n_local > n_global) return MLSORT_ERR_INVALID_ARG;
    if ((n_local && !d_shard) || (out_capacity && !d_out_keys)) return MLSORT_ERR_INVALID_ARG;
    if (o && (o->reserved[0] || o->reserved[1] || o->reserved[2])) return MLSORT_ERR_INVALID_ARG;
    NcclApi* api = nccl();
    if (!api) return MLSORT_ERR_NCCL;
    const uint32_t G = (uint32_t)c->nranks, me = (uint32_t)c->rank;
    const bool perm = d_out_perm != nullptr;
    const uint64_t ks = dt == MLSORT_F32 ? 4 : 8;
    const uint64_t B = (o && o->num_buckets) ? o->num_buckets : n_global;
    DistLayout L;
    int rc = dist_layout(G, n_local, n_global, dt, o, perm, out_capacity, L);
    if (rc) return rc;
    uintptr_t base = (reinterpret_cast<uintptr_t>(d_ws) + kAl - 1) / kAl * kAl;
    if (!d_ws || ws_bytes < L.total) return MLSORT_ERR_WORKSPACE;
    char* ws = reinterpret_cast<char*>(base);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timer tm;
    tm.start(o && o->timing, s);

    // ---- 1. predict + owner partition of this rank's shard (K_dist kernels)
    std::vector<uint64_t> send(G, 0);
    mlsort_info pinfo;
    int prc = MLSORT_OK;
    if (n_local > 0)
        prc = mlsort_dist_partition(d_shard, n_local, global_offset, n_global, dt, w, o, G, ws + L.rec_keys,
                                    reinterpret_cast<uint32_t*>(ws + L.rec_b),
                                    perm ? reinterpret_cast<uint32_t*>(ws + L.rec_idx) : nullptr, send.data(),
                                    ws + L.part, L.part_bytes, stream, &pinfo);
    else {
        std::memset(&pinfo, 0, sizeof(pinfo));
        pinfo.bad_index = -1;
        pinfo.fallback_used = mlsort_weights_check_monotone(w) == 1 ? 0 : 1;
    }
    if (prc != MLSORT_OK && prc != MLSORT_ERR_NONFINITE_KEY) return prc;
    tm.mark();

    // ---- 2. count exchange (collective also for errors, so no rank is left waiting in NCCL)
    const uint32_t S = G + 4;
    std::vector<uint64_t> msg(S), all((size_t)G * S);
    for (uint32_t g = 0; g < G; ++g) msg[g] = send[g];
    msg[G] = out_capacity;
    msg[G + 1] = (uint64_t)prc;
    msg[G + 2] = prc == MLSORT_ERR_NONFINITE_KEY ? global_offset + (uint64_t)pinfo.bad_index : ~0ull;
    msg[G + 3] = (uint64_t)pinfo.fallback_used;
    uint64_t* d_msg = reinterpret_cast<uint64_t*>(ws + L.msg);
    uint64_t* d_all = d_msg + S;
    CU(cudaMemcpyAsync(d_msg, msg.data(), S * 8, cudaMemcpyHostToDevice, s));
    NC(api->AllGather(d_msg, d_all, S, ncclUint64, c->comm, s));
    CU(cudaMemcpyAsync(all.data(), d_all, all.size() * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    tm.mark();
    uint64_t bad = ~0ull;
    bool keyspace = false;
    for (uint32_t g = 0; g < G; ++g) {
        bad = std::min(bad, all[(size_t)g * S + G + 2]);
        keyspace |= all[(size_t)g * S + G + 3] != 0;
    }
    if (info) {
        info->tail_lo = pinfo.tail_lo;
        info->tail_hi = pinfo.tail_hi;
        info->fallback_used = keyspace ? 1 : 0;
    }
    if (bad != ~0ull) {                                     // A11: lowest global index, every rank
        if (info) info->bad_index = (int64_t)bad;
        return MLSORT_ERR_NONFINITE_KEY;
    }
    uint64_t need = 0;
    bool any_over = false;
    std::vector<uint64_t> recv(G), soff(G + 1, 0), roff(G + 1, 0);
    for (uint32_t r = 0; r < G; ++r) {
        uint64_t nr = 0;
        for (uint32_t p = 0; p < G; ++p) nr += all[(size_t)p * S + r];
        if (nr > all[(size_t)r * S + G]) any_over = true;
        if (r == me) need = nr;
    }
    *out_count = need;
    if (any_over) return MLSORT_ERR_CAPACITY;               // consistent on every rank
    for (uint32_t p = 0; p < G; ++p) {
        recv[p] = all[(size_t)p * S + me];
        soff[p + 1] = soff[p] + send[p];
        roff[p + 1] = roff[p] + recv[p];
    }

    // ---- 3. one grouped all-to-all-v of the records (receive buffers in source-rank order)
    NC(api->GroupStart());
    for (uint32_t p = 0; p < G; ++p) {
        if (send[p]) {
            NC(api->Send(ws + L.rec_keys + soff[p] * ks, send[p], key_type(dt), (int)p, c->comm, s));
            NC(api->Send(ws + L.rec_b + soff[p] * 4, send[p], ncclUint32, (int)p, c->comm, s));
            if (perm) NC(api->Send(ws + L.rec_idx + soff[p] * 4, send[p], ncclUint32, (int)p, c->comm, s));
        }
        if (recv[p]) {
            NC(api->Recv(ws + L.recv_keys + roff[p] * ks, recv[p], key_type(dt), (int)p, c->comm, s));
            NC(api->Recv(ws + L.recv_b + roff[p] * 4, recv[p], ncclUint32, (int)p, c->comm, s));
            if (perm) NC(api->Recv(ws + L.recv_idx + roff[p] * 4, recv[p], ncclUint32, (int)p, c->comm, s));
        }
    }
    NC(api->GroupEnd());
    tm.mark();

    // ---- 4. local sort of the received records (no re-prediction; K1' partition .. K5)
    mlsort_info sinfo;
    std::memset(&sinfo, 0, sizeof(sinfo));
    if (need > 0) {
        uint64_t lo = 0, hi = B;
        if (!keyspace) owner_range(me, G, B, lo, hi);
        rc = mlsort_sort_records(ws + L.recv_keys, reinterpret_cast<uint32_t*>(ws + L.recv_b),
                                 perm ? reinterpret_cast<uint32_t*>(ws + L.recv_idx) : nullptr, need, dt, lo, hi,
                                 d_out_keys, d_out_perm, ws + L.rsort, L.rsort_bytes, stream, &sinfo);
        if (rc) return rc;
    }
    tm.mark();

    // ---- 5. global offset + cross-rank boundary verification (reading A14 at GPU boundaries)
    uint64_t bnd[kBnd] = {need, 0, 0, 0, 0};
    if (need > 0) {
        unsigned char kf[8] = {}, kl[8] = {};
        uint32_t pf = 0, pl = 0;
        CU(cudaMemcpyAsync(kf, d_out_keys, ks, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(kl, static_cast<char*>(d_out_keys) + (need - 1) * ks, ks, cudaMemcpyDeviceToHost, s));
        if (perm) {
            CU(cudaMemcpyAsync(&pf, d_out_perm, 4, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(&pl, d_out_perm + (need - 1), 4, cudaMemcpyDeviceToHost, s));
        }
        CU(cudaStreamSynchronize(s));
        bnd[1] = ord_bits(kf, dt);
        bnd[2] = pf;
        bnd[3] = ord_bits(kl, dt);
        bnd[4] = pl;
    }
    uint64_t* d_b = d_all + (size_t)G * S;
    uint64_t* d_ball = d_b + kBnd;
    std::vector<uint64_t> ball((size_t)G * kBnd);
    CU(cudaMemcpyAsync(d_b, bnd, sizeof(bnd), cudaMemcpyHostToDevice, s));
    NC(api->AllGather(d_b, d_ball, kBnd, ncclUint64, c->comm, s));
    CU(cudaMemcpyAsync(ball.data(), d_ball, ball.size() * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    tm.mark();
    uint64_t goff = 0, violations = 0;
    bool have = false;
    uint64_t last_ord = 0, last_idx = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const uint64_t* r = &ball[(size_t)g * kBnd];
        if (g < me) goff += r[0];
        if (r[0] == 0) continue;
        if (have) {
            const bool ok = perm ? (last_ord < r[1] || (last_ord == r[1] && last_idx < r[2])) : last_ord <= r[1];
            violations += ok ? 0 : 1;
        }
        have = true;
        last_ord = r[3];
        last_idx = r[4];
    }
    if (out_global_offset) *out_global_offset = goff;
    tm.finish(info);
    if (info) {
        info->repairs = sinfo.repairs + violations;
        info->fallback_used = (keyspace || sinfo.fallback_used) ? 1 : 0;
        info->num_coarse = sinfo.num_coarse;
        info->max_coarse = sinfo.max_coarse;
        info->big_buckets = sinfo.big_buckets;
        info->kernel_launches = pinfo.kernel_launches + sinfo.kernel_launches;
    }
    // both ownership rules are monotone in the key, so ranks cannot overlap; a violation here
    // means a device fault, reported rather than silently returned as a sorted array
    if (violations) return MLSORT_ERR_INTERNAL;
    return MLSORT_OK;
}
