/*
 * mlsort.h -- C ABI of the B200-native Machine Learning Sort library (libmlsort.so).
 *
 * Machine Learning Sort (Zhao & Luo, arXiv 1805.04272; /root/reference/PAPER.md = "P:n"):
 * a trained monotone 1->M->1 network (the paper's GVM, Eq. 3) predicts the
 * normalised rank y of every key; keys go to rank buckets r = round(y*B);
 * each bucket is sorted ("only the numbers inside each bucket need to be sorted");
 * the concatenation is the fully sorted output.  This library implements that
 * inference-and-placement phase with hand-written sm_100a CUDA kernels.  Training the
 * network on a small sample is a host step whose weights are data.
 *
 * Conventions (all entry points):
 *  - Return value: int status, 0 = MLSORT_OK, else an mlsort_status_code.  No C++
 *    exception ever crosses the ABI.  mlsort_status_string() names a code.
 *  - "d_" pointers are CUDA device pointers on the calling thread's current device,
 *    "h_" pointers are host pointers.  Pointers are borrowed: the caller owns every
 *    buffer, the library never frees or retains a caller pointer after returning.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Device
 *    work is stream-ordered on it.
 *  - Key dtypes: MLSORT_F32 (IEEE binary32) or MLSORT_F64 (binary64), little endian.
 *  - Order: ascending IEEE-754 totalOrder (-0.0 before +0.0); ties between
 *    bit-identical keys are broken by input index, so the output and the permutation
 *    are unique (readings A1, A9, A10).  NaN and +-Inf keys are rejected
 *    (reading A11).
 *  - Weights handles are immutable after creation and may be shared between threads
 *    (S:177).  Calls with distinct workspaces are re-entrant.
 */
#ifndef MLSORT_H
#define MLSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mlsort_status_code {
    MLSORT_OK = 0,
    MLSORT_ERR_INVALID_ARG = 1,      /* null pointer, bad size, bad enum, aliasing        */
    MLSORT_ERR_IO = 2,               /* weights file cannot be opened / written          */
    MLSORT_ERR_PARSE = 3,            /* weights JSON malformed                           */
    MLSORT_ERR_INVALID_WEIGHTS = 4,  /* m < 1, length mismatch, non-finite, lo >= hi     */
    MLSORT_ERR_NONFINITE_KEY = 5,    /* NaN or +-Inf key; info->bad_index = lowest index */
    MLSORT_ERR_CUDA = 6,             /* a CUDA runtime call failed                       */
    MLSORT_ERR_WORKSPACE = 7,        /* workspace too small or misaligned                */
    MLSORT_ERR_CAPACITY = 8,         /* distributed output larger than out_capacity      */
    MLSORT_ERR_TRAIN = 9,            /* degenerate training sample (all keys equal)      */
    MLSORT_ERR_INTERNAL = 10,        /* internal invariant violated (a bug)              */
    MLSORT_ERR_NCCL = 11             /* NCCL missing (libnccl.so.2) or an NCCL call failed */
};

typedef enum { MLSORT_F32 = 0, MLSORT_F64 = 1 } mlsort_dtype;

/* Which f32 formulation of the logistic the predict kernel uses.
 * All meet |y - y_fp64| <= 1e-5; the output sort is bit-exact for every choice. */
typedef enum {
    MLSORT_PRED_DEFAULT = 0,   /* library choice: MLSORT_PRED_PACKED for M <= 32,
                                  MLSORT_PRED_SKIP for M > 32                                  */
    MLSORT_PRED_MUFU = 1,      /* ex2 + rcp both on the SFU: 2 MUFU per activation             */
    MLSORT_PRED_MIXED = 2,     /* ex2 on the SFU; reciprocal split between SFU and scalar
                                  FMA-pipe Newton iterations                                   */
    MLSORT_PRED_PACKED = 3,    /* ex2 on the SFU; reciprocal on the FMA pipe with packed f32x2
                                  instructions (bit-trick seed, modified Newton + cubic step)  */
    MLSORT_PRED_SKIP = 4       /* MLSORT_PRED_PACKED arithmetic, skipping neuron pairs that are
                                  saturated over a warp's key range (their terms are exact
                                  constants): bit-identical outputs; the sort groups each tile
                                  by value first so warps span narrow ranges                    */
} mlsort_predictor;

/* Opaque host-resident GVM parameters {m, w1, w2, b, beta, input_lo, input_hi}
 * (Eq. 3 symbols, S:91-S:97). */
typedef struct mlsort_weights mlsort_weights;

typedef struct {
    uint64_t num_buckets;   /* B, the number of rank buckets; 0 means B = n          */
    int32_t  predictor;     /* mlsort_predictor                                             */
    int32_t  verify;        /* accepted for compatibility, no effect: the adjacent order of
                               every output pair is always verified (K3 inside each coarse
                               bucket, K5 at coarse boundaries; reading A14)          */
    int32_t  timing;        /* 1 = record CUDA events around each kernel phase and report
                               the device times in mlsort_info.phase_ms (bench/profiling)     */
    int32_t  reserved[3];   /* must be zero                                                 */
} mlsort_opts;

typedef struct {
    int64_t  bad_index;     /* lowest index of a NaN/+-Inf key, or -1                       */
    uint64_t repairs;       /* adjacent order violations found and repaired (A14)           */
    int32_t  fallback_used; /* 1 if non-monotone weights forced the conventional-sort path  */
    uint32_t num_coarse;    /* coarse partition size C used internally                      */
    uint64_t tail_lo;       /* keys below the weights' input_lo (P:121 tails, diagnostic)   */
    uint64_t tail_hi;       /* keys above input_hi                                          */
    uint64_t max_coarse;    /* largest coarse bucket                                        */
    uint64_t big_buckets;   /* coarse buckets that took the overflow path                   */
    uint64_t kernel_launches; /* device kernels launched by this call                      */
    float    phase_ms[6];   /* with opts->timing: K1 predict+partition, K2 coarse starts,
                               K3 cluster sort, K4 overflow gather, K5 verify, whole call     */
} mlsort_info;

/* Monte-Carlo trainer configuration (S:104-S:107, S:170-S:172; every value is a repo
 * decision because the paper gives no rule, P:63 / S:186). */
typedef struct {
    uint32_t m;                 /* hidden neurons M                                       */
    uint32_t max_pairs;         /* training pairs used (evenly spaced ranks), 0 = all     */
    uint64_t iterations;        /* Monte-Carlo proposals                                  */
    double   perturb_scale;     /* proposal step: N(0,1) * scale * (1 + |value|)          */
    double   target_loss;       /* early stop when MSE <= target_loss                     */
    uint64_t seed;              /* proposal RNG seed                                      */
    int32_t  enforce_monotone;  /* reject proposals breaking w1*w2*beta >= 0 (Eq. 4)      */
    int32_t  reserved;
} mlsort_train_cfg;

/* ------------------------------------------------------------------ misc */
const char* mlsort_status_string(int status);
const char* mlsort_version(void);

/* ------------------------------------------------------------------ weights (host) */

/* Copy m-long arrays into a new handle.  Errors: MLSORT_ERR_INVALID_ARG (null pointer),
 * MLSORT_ERR_INVALID_WEIGHTS (m < 1, non-finite value, lo >= hi; S:94-S:96). */
int mlsort_weights_create(uint32_t m, const double* h_w1, const double* h_w2,
                          const double* h_b, const double* h_beta, double input_lo,
                          double input_hi, mlsort_weights** out);

/* Parse the versioned JSON document {"format":"mlsort-gvm","version":1,"m",
 * "w1","w2","b","beta","input_lo","input_hi","activation":"logistic",...}.
 * Errors: MLSORT_ERR_IO, MLSORT_ERR_PARSE, MLSORT_ERR_INVALID_WEIGHTS. */
int mlsort_weights_load(const char* json_path, mlsort_weights** out);

/* Write the JSON document; doubles are printed with 17 significant digits so a
 * save/load round trip is bit-exact.  Errors: MLSORT_ERR_IO. */
int mlsort_weights_save(const mlsort_weights* w, const char* json_path);

void mlsort_weights_free(mlsort_weights* w);

/* Read back the parameters.  Any output pointer may be NULL; arrays must hold m doubles. */
int mlsort_weights_get(const mlsort_weights* w, uint32_t* m, double* h_w1, double* h_w2,
                       double* h_b, double* h_beta, double* input_lo, double* input_hi,
                       double* final_loss);

/* 1 if every neuron satisfies w1*w2*beta >= 0 -- the per-neuron sufficient form of
 * Eq. 4 for an ascending model (reading A22; S:120-S:128) -- else 0;
 * negative status on a null handle. */
int mlsort_weights_check_monotone(const mlsort_weights* w);

/* ------------------------------------------------------------------ training (host, untimed) */

/* Fill *cfg with the library defaults for m neurons. */
int mlsort_train_cfg_default(mlsort_train_cfg* cfg, uint32_t m);

/* Fit the GVM to the empirical CDF of a host sample (sort the training sequence,
 * pairs (a'_i, i/N0); Monte-Carlo search instead of back-propagation).  The
 * sample is copied and sorted; input_lo/hi = sample min/max.  Errors:
 * MLSORT_ERR_INVALID_ARG (n0 < 1, bad dtype), MLSORT_ERR_NONFINITE_KEY,
 * MLSORT_ERR_TRAIN (all sample keys equal). */
int mlsort_fit(const void* h_sample, uint64_t n0, mlsort_dtype dtype,
               const mlsort_train_cfg* cfg, mlsort_weights** out);

/* ------------------------------------------------------------------ the sort (device) */

/* Bytes of device workspace mlsort_sort needs for n keys (two-phase, CUB style). */
int mlsort_sort_workspace_size(uint64_t n, mlsort_dtype dtype, const mlsort_opts* opts,
                               int want_perm, uint64_t* bytes);

/* Sort n keys (§2: predict -> bucket -> place -> per-bucket fix-up).
 *  d_keys        [n] input keys (dtype), device.  Not modified.
 *  d_payload     [n] optional uint32 payload or NULL.
 *  d_out_keys    [n] sorted keys, device; must not alias d_keys.
 *  d_out_perm    [n] optional: d_out_perm[i] = input index of the i-th output (gather
 *                form, reading A18), or NULL for a key-only sort.  Needs n < 2^32.
 *  d_out_payload [n] optional: d_out_payload[i] = d_payload[d_out_perm[i]]; requires
 *                d_payload and d_out_perm.
 *  d_ws, ws_bytes device workspace of at least mlsort_sort_workspace_size() bytes,
 *                256-byte aligned.
 *  info          optional diagnostics (host).
 * n == 0 is a no-op returning MLSORT_OK.  A NaN/Inf key returns MLSORT_ERR_NONFINITE_KEY
 * with info->bad_index set (outputs undefined).  Non-monotone weights still give the
 * exact output through the verify/repair and fallback paths.
 * Synchronises `stream` once at the end to read the status word. */
int mlsort_sort(const void* d_keys, const uint32_t* d_payload, uint64_t n, mlsort_dtype dtype,
                const mlsort_weights* w, const mlsort_opts* opts, void* d_out_keys,
                uint32_t* d_out_perm, uint32_t* d_out_payload, void* d_ws, uint64_t ws_bytes,
                void* stream, mlsort_info* info);

/* Workspace for mlsort_sort_host: mlsort_sort's workspace plus device staging for the
 * input and output arrays. */
int mlsort_sort_host_workspace_size(uint64_t n, mlsort_dtype dtype, const mlsort_opts* opts,
                                    int want_perm, uint64_t* bytes);

/* End-to-end variant on HOST buffers: copies h_keys to the device (inside d_ws), runs
 * mlsort_sort, copies the sorted keys (and h_out_perm if non-NULL) back.  Host buffers
 * should be pinned for full PCIe/C2C bandwidth.  Same errors as mlsort_sort. */
int mlsort_sort_host(const void* h_keys, uint64_t n, mlsort_dtype dtype,
                     const mlsort_weights* w, const mlsort_opts* opts, void* h_out_keys,
                     uint32_t* h_out_perm, void* d_ws, uint64_t ws_bytes, void* stream,
                     mlsort_info* info);

/* The approximate-ranking phase alone ("the complexity of the prediction for each
 * number is only O(M)"): d_y[i] = f32 network output (Eq. 3) and/or
 * d_bucket[i] = clamp(round(y*B), 0, B-1) with B = num_buckets (0 => n).  Either output
 * may be NULL.  Does not synchronise; non-finite keys produce unspecified outputs. */
int mlsort_predict(const void* d_keys, uint64_t n, mlsort_dtype dtype, const mlsort_weights* w,
                   uint64_t num_buckets, int32_t predictor, float* d_y, uint32_t* d_bucket,
                   void* stream);

/* Diagnostic (reading A14; SURVEY.md §8(c) "exhaustive monotonicity", K8).  PAPER.md Eq. 4
 * (l.76-84) makes the network monotone in exact arithmetic; the f32 device predictor is
 * monotone if the approximate primitives it is built from are.  This evaluates one of them
 * on EVERY input of its domain, in ascending order, on the current device:
 *   0 ex2.approx.ftz.f32 over all non-NaN f32 (must be non-decreasing),
 *   1 the packed FMA-pipe reciprocal chain over every f32 d in [1, 2^61] (non-increasing;
 *     *max_rel_err = max |r d - 1|),
 *   2 rcp.approx.ftz.f32 over every positive f32 (non-increasing),
 *   3 the packed predictor's logistic term 1/(1 + ex2(min(a, 60))) over all non-NaN a
 *     (non-increasing).
 * *descents = adjacent input pairs whose outputs go the wrong way (0 = monotone);
 * *evaluated = inputs evaluated.  Any output pointer may be NULL.  Synchronises `stream`.
 * Sort correctness never depends on the result (every adjacent output pair is verified);
 * a descent would only cost repairs.  Errors: MLSORT_ERR_INVALID_ARG, MLSORT_ERR_CUDA. */
int mlsort_selftest_monotone(int32_t primitive, uint64_t* descents, uint64_t* evaluated,
                             double* max_rel_err, void* stream);

/* ------------------------------------------------------------------ multi-GPU building blocks
 * One process per GPU.  Rank g holds the contiguous input slice
 * starting at global index `global_offset`; every rank predicts the global bucket
 * b = round(y*B) of its keys and the owner rank floor(b*G/B), so rank g owns the rank
 * range [gB/G, (g+1)B/G) (BJ:5).  mlsort_sort_dist (below) runs the whole exchange with a
 * library-owned NCCL communicator; the two building blocks are exported for callers that
 * move the records themselves.  Concatenating the ranks' outputs in rank order gives the
 * global sorted array, identical to the 1-GPU result.
 * A model that fails Eq. 4 (mlsort_weights_check_monotone == 0) does not order the
 * buckets; mlsort_dist_partition then routes keys by key value instead (owner =
 * clamp(floor((x - input_lo) G / (input_hi - input_lo)), 0, G-1), monotone in x),
 * reports info->fallback_used = 1, and the receivers must sort with the bucket range
 * [0, B) (reading A14). */

int mlsort_dist_partition_workspace_size(uint64_t n_local, mlsort_dtype dtype, uint32_t nranks,
                                         uint64_t* bytes);

/* Predict + partition by owner.  Outputs, grouped by destination rank 0..G-1 (records of
 * one destination are contiguous, in input order):
 *   d_rec_keys [n_local] keys (dtype), d_rec_bucket [n_local] global bucket b (uint32),
 *   d_rec_index [n_local] global input index (uint32; global_offset + local index).
 *   h_send_counts [nranks] (host) number of records for each destination.
 * info->fallback_used = 1: routed by key value (non-monotone model, see above).
 * Synchronises `stream`.  Errors as mlsort_sort (non-finite keys, bad args). */
int mlsort_dist_partition(const void* d_shard, uint64_t n_local, uint64_t global_offset,
                          uint64_t n_global, mlsort_dtype dtype, const mlsort_weights* w,
                          const mlsort_opts* opts, uint32_t nranks, void* d_rec_keys,
                          uint32_t* d_rec_bucket, uint32_t* d_rec_index, uint64_t* h_send_counts,
                          void* d_ws, uint64_t ws_bytes, void* stream, mlsort_info* info);

int mlsort_sort_records_workspace_size(uint64_t n, mlsort_dtype dtype, uint64_t bucket_lo,
                                       uint64_t bucket_hi, uint64_t* bytes);

/* Sort n received records whose buckets lie in [bucket_lo, bucket_hi) (this rank's range)
 * by (key, index): outputs d_out_keys[n] and d_out_index[n] (global input indices).  No
 * prediction is repeated: the bucket travels with the key.  Synchronises `stream`. */
int mlsort_sort_records(const void* d_keys, const uint32_t* d_bucket, const uint32_t* d_index,
                        uint64_t n, mlsort_dtype dtype, uint64_t bucket_lo, uint64_t bucket_hi,
                        void* d_out_keys, uint32_t* d_out_index, void* d_ws, uint64_t ws_bytes,
                        void* stream, mlsort_info* info);

/* ------------------------------------------------------------------ multi-GPU sort (NCCL)
 * SURVEY.md §8(b)/(e); PAPER.md l.94 ("the prediction of each number is independent ...
 * requires very little networking workload"), l.134 ("both N and M can be separated").
 * One process per GPU; the library owns an NCCL communicator (libnccl.so.2 is loaded at
 * mlsort_comm_init; MLSORT_NCCL_LIB overrides its path).  Every call below is collective
 * over the communicator's ranks, in the same order, with consistent arguments; argument
 * errors are detected locally (not collectively) and are caller bugs. */
typedef struct mlsort_comm mlsort_comm;

/* Fill out_id (128 bytes, NCCL_UNIQUE_ID_BYTES) with a fresh NCCL unique id: called on one
 * rank, which then broadcasts the bytes to the others (e.g. torch.distributed).
 * Errors: MLSORT_ERR_INVALID_ARG, MLSORT_ERR_NCCL. */
int mlsort_comm_unique_id(void* out_id);

/* Create this rank's communicator on CUDA device `device` (ncclCommInitRank; collective).
 * nranks in [1, 64].  The caller owns *out and frees it with mlsort_comm_destroy.
 * Errors: MLSORT_ERR_INVALID_ARG, MLSORT_ERR_CUDA, MLSORT_ERR_NCCL. */
int mlsort_comm_init(int nranks, int rank, const void* unique_id, int device, mlsort_comm** out);

/* Destroy a communicator (NULL is a no-op).  Errors: MLSORT_ERR_NCCL. */
int mlsort_comm_destroy(mlsort_comm* comm);

/* Device workspace of mlsort_sort_dist for a rank holding n_local keys that may receive up
 * to out_capacity records (its output capacity). */
int mlsort_sort_dist_workspace_size(uint32_t nranks, uint64_t n_local, uint64_t n_global, mlsort_dtype dtype,
                                    const mlsort_opts* opts, int want_perm, uint64_t out_capacity,
                                    uint64_t* bytes);

/* Distributed sort of the global array whose keys [global_offset, global_offset + n_local)
 * are on this rank (device pointer d_shard; n_global < 2^32, B = opts->num_buckets or
 * n_global).  Steps: predict + owner partition (global buckets, owner floor(b G / B)); an
 * NCCL all-gather of the send counts; one grouped NCCL send/recv all-to-all-v of the
 * records (key, bucket, global index), received in source-rank order; the local sort of the
 * received records (no re-prediction); an NCCL all-gather of every rank's first/last
 * (key, index) that verifies the order across ranks and gives the global offset.
 * Outputs: d_out_keys[*out_count] = this rank's sorted run, d_out_perm (nullable; GLOBAL
 * input indices, stable), *out_global_offset = position of the run in the global sorted
 * array (sum of the lower ranks' counts).  The concatenation over ranks equals mlsort_sort
 * of the whole array on one GPU, bit for bit.  Caller owns every buffer; d_ws from
 * mlsort_sort_dist_workspace_size.  With opts->timing, info->phase_ms = {partition, count
 * exchange, all-to-all, local sort, boundary exchange, total}.
 * Errors (collective: every rank returns the same code):
 *   MLSORT_ERR_NONFINITE_KEY  info->bad_index = lowest GLOBAL index of a NaN/+-Inf key;
 *   MLSORT_ERR_CAPACITY       some rank would receive more than its out_capacity;
 *                             *out_count = this rank's required capacity;
 *   MLSORT_ERR_INTERNAL       the cross-rank order check failed (not reachable with either
 *                             ownership rule, which are monotone in the key);
 *   MLSORT_ERR_NCCL / MLSORT_ERR_CUDA / MLSORT_ERR_WORKSPACE. */
int mlsort_sort_dist(mlsort_comm* comm, const void* d_shard, uint64_t n_local, uint64_t global_offset,
                     uint64_t n_global, mlsort_dtype dtype, const mlsort_weights* w, const mlsort_opts* opts,
                     void* d_out_keys, uint32_t* d_out_perm, uint64_t out_capacity, uint64_t* out_count,
                     uint64_t* out_global_offset, void* d_ws, uint64_t ws_bytes, void* stream,
                     mlsort_info* info);

#ifdef __cplusplus
}
#endif
#endif /* MLSORT_H */
