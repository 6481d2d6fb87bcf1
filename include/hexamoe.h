/*
 * hexamoe.h -- C ABI of the B200-native HEXA-MoE expert-specific operators.
 *
 * This is the drop-in boundary for the reference `moekit` hot path
 * (/root/reference/proj/core/include/moekit/{routing,es_ops,moe_layer}.hpp).
 * Every entry point below names the reference function it replaces.  The
 * signatures are plain C: device pointers, sizes and a cudaStream_t; no C++
 * or torch types.  A host-side C++ shim that re-exposes the reference's
 * signatures, and the ctypes binding used by the Python package, are shown in
 * INTEGRATION.md.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers, dense row-major, with the
 *    reference's shapes: x N x D1, weights E x D1 x D2 (dim0 = expert), bias
 *    E x D2, ReIndex v int64[N'], idx int64[E+1] (routing.hpp:29-38).
 *  - `dtype` selects the arithmetic: HXM_BF16 = bf16 inputs on the tcgen05
 *    tensor cores with fp32 accumulation; HXM_F32 = fp32 inputs, fp32 FMA.
 *    Biases, outputs and gradients are always fp32.
 *  - Calls are asynchronous on `stream`.  Shape / argument checks run on the
 *    host before any launch, in the reference's order, and return
 *    HXM_ERR_SHAPE (reference ShapeError) or HXM_ERR_INVALID_ARG (reference
 *    std::invalid_argument).  Data-dependent checks that the reference
 *    performs while reading values (expert id out of range) are reported
 *    through a device status word (`status_dev`, may be NULL).
 *  - hxm_last_error() returns a thread-local message for the last failure.
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns HXM_ERR_CUDA.
 */
#ifndef HEXAMOE_H
#define HEXAMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hxm_stream_t; /* == cudaStream_t */

typedef enum hxm_status {
  HXM_OK = 0,
  HXM_ERR_SHAPE = 1,       /* moekit::ShapeError      (tensor.hpp:12-15)  */
  HXM_ERR_INVALID_ARG = 2, /* std::invalid_argument                       */
  HXM_ERR_CUDA = 3,
  HXM_ERR_NCCL = 4,
  HXM_ERR_CACHE = 5,       /* moekit::CacheError      (dist_sim.hpp:55-58) */
  HXM_ERR_UNSUPPORTED = 6
} hxm_status;

typedef enum hxm_dtype { HXM_F32 = 0, HXM_BF16 = 1 } hxm_dtype;

/* same order as moekit::ActivationKind (tensor.hpp:96) */
typedef enum hxm_activation {
  HXM_ACT_RELU = 0,
  HXM_ACT_GELU = 1,
  HXM_ACT_IDENTITY = 2
} hxm_activation;

/* moekit::EsOutputMode (es_ops.hpp:13) */
typedef enum hxm_out_mode { HXM_WRITE = 0, HXM_ACCUMULATE = 1 } hxm_out_mode;

const char* hxm_last_error(void);
int hxm_version(void);
/* Number of SMs of the current device, or -1 without a device. */
int hxm_device_sm_count(void);

/* ------------------------------------------------------------------------
 * Routing index build -- replaces moekit::build_reindex (routing.hpp:42-43,
 * routing.cpp:42-70).  Bit-exact: v is tokens grouped by expert, ascending
 * inside each segment, segments padded with -1 to a multiple of blk;
 * idx[0] = 0, idx[E] = N'.
 * ---------------------------------------------------------------------- */
/* Upper bound of N' = n + E*(blk-1): size of v. */
size_t hxm_reindex_bound(int64_t n_tokens, int64_t n_experts, int64_t blk);
size_t hxm_reindex_workspace_bytes(int64_t n_tokens, int64_t n_experts);
/* assignment: device int32[n_tokens].  v: device int64[bound];
 * idx: device int64[E+1].  status_dev (nullable, device int32): set to
 * HXM_ERR_INVALID_ARG when an expert id is out of range (routing.cpp:47-48);
 * the caller zeroes it.  blk == 0 -> HXM_ERR_INVALID_ARG before launch. */
hxm_status hxm_build_reindex(const int32_t* assignment, int64_t n_tokens,
                             int64_t n_experts, int64_t blk, int64_t* v,
                             int64_t* idx, void* workspace,
                             size_t workspace_bytes, int32_t* status_dev,
                             hxm_stream_t stream);

/* build_reindex_all (routing.hpp:46, routing.cpp:72-80): one ReIndex per
 * routing choice, all k built in the same three launches.  assignments:
 * device int32 k x n (RoutingChoice::assignments); choice i's v at
 * v + i * v_stride (v_stride >= hxm_reindex_bound), its idx at
 * idx + i * (E + 1).  Same checks and status word as hxm_build_reindex. */
size_t hxm_reindex_all_workspace_bytes(int64_t n_tokens, int64_t n_experts, int64_t k);
hxm_status hxm_build_reindex_all(const int32_t* assignments, int64_t k,
                                 int64_t n_tokens, int64_t n_experts,
                                 int64_t blk, int64_t* v, int64_t v_stride,
                                 int64_t* idx, void* workspace,
                                 size_t workspace_bytes, int32_t* status_dev,
                                 hxm_stream_t stream);

/* ------------------------------------------------------------------------
 * Operators -- replace moekit::esmm / ess / estmm / esfk (es_ops.hpp:37-65).
 * v/idx are a ReIndex built by hxm_build_reindex (or copied from the
 * reference); n_padded_bound >= N' = idx[E] (hxm_reindex_bound suffices).
 * Operator workspace: hxm_op_workspace_bytes().
 * ---------------------------------------------------------------------- */
size_t hxm_op_workspace_bytes(int64_t n_tokens, int64_t n_experts,
                              int64_t n_padded_bound, int64_t d1, int64_t d2);

/* esmm (es_ops.hpp:39-46): dest[t] (= | +=) bias[e(t)] + x[t] . W[e(t)].
 * w_transposed = 0: weights is E x D1 x D2 (reference layout).
 * w_transposed = 1: weights is E x D2 x D1 and W[e]^T is used -- this replaces
 * materialising transpose_experts (tensor.cpp:143-153).  bias: fp32 E x D2
 * or NULL.  dest: fp32 N x D2. */
hxm_status hxm_esmm(hxm_dtype dtype, const void* x, int64_t n_tokens,
                    int64_t d1, const void* weights, int64_t n_experts,
                    int64_t d2, int w_transposed, const float* bias,
                    const int64_t* v, const int64_t* idx,
                    int64_t n_padded_bound, hxm_out_mode mode, float* dest,
                    void* workspace, size_t workspace_bytes,
                    hxm_stream_t stream);

/* ess (es_ops.hpp:49): out[e] = sum of rows routed to e (fp32 E x D). */
hxm_status hxm_ess(hxm_dtype dtype, const void* x, int64_t n_tokens, int64_t d,
                   const int64_t* v, const int64_t* idx, int64_t n_experts,
                   int64_t n_padded_bound, float* out, void* workspace,
                   size_t workspace_bytes, hxm_stream_t stream);

/* estmm (es_ops.hpp:52-53): out[e] = sum_{t in e} x1[t]^T x2[t]
 * (fp32 E x D1 x D2; experts without tokens get zeros). */
hxm_status hxm_estmm(hxm_dtype dtype, const void* x1, const void* x2,
                     int64_t n_tokens, int64_t d1, int64_t d2,
                     const int64_t* v, const int64_t* idx, int64_t n_experts,
                     int64_t n_padded_bound, float* out, void* workspace,
                     size_t workspace_bytes, hxm_stream_t stream);

/* esfk (es_ops.hpp:55-65): grad_x = esmm(g, w_t, NULL) (write),
 * grad_b = ess(g), grad_w = estmm(x, g).  w_t is E x D2 x D1 as in the
 * reference; with w_transposed = 1 pass the un-transposed E x D1 x D2
 * weights instead. */
hxm_status hxm_esfk(hxm_dtype dtype, const void* x, const void* g,
                    int64_t n_tokens, int64_t d1, int64_t d2,
                    const void* w_t, int w_transposed, const int64_t* v,
                    const int64_t* idx, int64_t n_experts,
                    int64_t n_padded_bound, float* grad_x, float* grad_b,
                    float* grad_w, void* workspace, size_t workspace_bytes,
                    hxm_stream_t stream);

/* OpStats / per-operator work counters (es_ops.hpp:17-24), incremented the
 * way the reference's tiles do (es_ops.cpp:53-56, 80, 97-101, 124-127):
 * real slots count MACs (esmm, estmm: real * d1 * d2) or adds (ess:
 * real * d1), -1 pad slots count padding_slots once per operator pass; esfk
 * (x N x d1, g N x d2) is esmm + ess + estmm.  For a valid ReIndex real_slots
 * = n_tokens and padding_slots = idx[E] - n_tokens.  Host-side: the counters
 * depend only on the index, so no device work or sync is needed. */
typedef struct hxm_op_stats {
  uint64_t macs;
  uint64_t adds;
  uint64_t padding_slots;
} hxm_op_stats;
typedef enum hxm_op_kind {
  HXM_OP_ESMM = 0,
  HXM_OP_ESS = 1,
  HXM_OP_ESTMM = 2,
  HXM_OP_ESFK = 3
} hxm_op_kind;
void hxm_op_stats_add(hxm_op_kind op, int64_t real_slots, int64_t padding_slots,
                      int64_t d1, int64_t d2, hxm_op_stats* stats);

/* ------------------------------------------------------------------------
 * MoE layer -- replaces moekit::moe_forward / moe_backward
 * (moe_layer.hpp:61-73, moe_layer.cpp:30-122).  The k routing choices are
 * processed together: one combined expert-grouped index over the k*N
 * (token, choice) slots, so every per-expert GEMM runs once per layer
 * instead of once per choice.  The forward stash (ForwardStash,
 * moe_layer.hpp:39-46) lives in `workspace` in expert-sorted row order and
 * is consumed by hxm_moe_backward.
 * ---------------------------------------------------------------------- */
typedef struct hxm_layer_desc {
  int64_t n_tokens;   /* N                                   */
  int64_t n_experts;  /* E                                   */
  int64_t k;          /* routing choices per token           */
  int64_t d_in;       /* D_i                                 */
  int64_t hidden;     /* H (this rank's slice under TP)      */
  int64_t d_out;      /* D_o                                 */
  int32_t activation; /* hxm_activation                      */
  int32_t dtype;      /* hxm_dtype                           */
  int32_t add_b2;     /* 1: add b2 (rank 0 under model-centric TP,
                         dist_sim.cpp:486); 0: skip b2 / gb2 */
  int32_t capacity;   /* 0: expert-specific (every routed slot computed,
                         nothing padded or dropped).  > 0: the conventional
                         dispatch/combine baseline (gemm_oracle.cpp:75-139,
                         count_redundancy gemm_oracle.cpp:251-285): every
                         expert computes exactly `capacity` rows -- all k*N
                         (token, choice) slots compete, lowest slot ids are
                         kept, overflow is dropped (zero contribution),
                         shortfall rows are zero padding that the GEMMs
                         process.  Must be a multiple of 64. */
  int32_t weight_shards; /* 0 or 1: w1 / b1 / w2 in the reference layout
                         (E x D_i x H, E x H, E x H x D_o).  P > 1:
                         shard-major -- the data-centric TP cache filled by
                         an all-gather of P hidden shards straight into one
                         buffer, no repacking (dist_sim.cpp:367-368):
                         w1 P x E x D_i x h, b1 P x E x h, w2 P x E x h x D_o
                         with h = H / P (bf16 tcgen05 path; h a multiple of
                         64 and of the GEMMs' tile widths,
                         hxm_layer_weight_shards_ok). */
  int32_t reserved0;
  void* weights_ready;  /* cudaEvent_t or NULL: the forward waits on it
                         after its routing prologue and before the first
                         kernel that reads w1 / b1 / w2 -- the cache fill
                         (on a side stream) overlaps the index build. */
} hxm_layer_desc;

/* 1 if the layer can read shard-major weights split P ways (see
 * hxm_layer_desc.weight_shards), else 0. */
int hxm_layer_weight_shards_ok(const hxm_layer_desc* desc, int32_t n_shards);

size_t hxm_layer_workspace_bytes(const hxm_layer_desc* desc);

/* forward: x N x D_i (dtype), w1 E x D_i x H (dtype), b1 fp32 E x H,
 * w2 E x H x D_o (dtype), b2 fp32 E x D_o, assignments device int32 k x N
 * (RoutingChoice::assignments, routing.hpp:14-21).  y: fp32 N x D_o
 * (written, not accumulated).  status_dev as in hxm_build_reindex. */
hxm_status hxm_moe_forward(const hxm_layer_desc* desc, const void* x,
                           const void* w1, const float* b1, const void* w2,
                           const float* b2, const int32_t* assignments,
                           float* y, void* workspace, size_t workspace_bytes,
                           int32_t* status_dev, hxm_stream_t stream);

/* backward for the stash in `workspace`: g_y N x D_o (dtype).
 * Gradients (fp32, written): gw1 E x D_i x H, gb1 E x H, gw2 E x H x D_o,
 * gb2 E x D_o (skipped if add_b2 == 0; may be NULL then), gx N x D_i. */
hxm_status hxm_moe_backward(const hxm_layer_desc* desc, const void* x,
                            const void* w1, const void* w2, const void* g_y,
                            void* workspace, size_t workspace_bytes,
                            float* gw1, float* gb1, float* gw2, float* gb2,
                            float* gx, hxm_stream_t stream);

/* Debug/parity: copy the stash of choice `choice` back to token order as
 * fp32 N x H.  The device stash keeps what the backward needs of the
 * reference's (y1, y2) pair (moe_layer.hpp:39-46): dact = F'(y1) and
 * y2 = F(y1). */
hxm_status hxm_moe_stash_export(const hxm_layer_desc* desc,
                                const void* workspace, int64_t choice,
                                float* dact, float* y2, hxm_stream_t stream);

/* Algorithmic work counters (OpStats, es_ops.hpp:17-24), MACs per direction:
 * expert-specific (capacity 0) = k*N*(D_i*H + H*D_o) on real tokens only;
 * conventional baseline = E*capacity*(D_i*H + H*D_o), padding included
 * (count_redundancy's token_macs_oracle, gemm_oracle.cpp:281-282). */
uint64_t hxm_layer_forward_macs(const hxm_layer_desc* desc);

/* Which kernels the layer runs for this descriptor: 2 = bf16 tcgen05 GEMMs
 * on CTA pairs (cta_group::2, 256-row tiles), 1 = bf16 tcgen05 on single
 * CTAs, 0 = the fp32 SIMT path, -1 = invalid descriptor. */
int hxm_layer_path(const hxm_layer_desc* desc);

/* ------------------------------------------------------------------------
 * Input generators (the reference's own seeded streams, random.hpp:13-54,
 * routing.cpp:121-200), host memory.  Measurement inputs only.
 * ---------------------------------------------------------------------- */
/* dist: "uniform" | "zipf:<s>" | "fixed:<e>" | "balanced" */
hxm_status hxm_synthesize_routing(int64_t n_tokens, int64_t n_experts,
                                  int64_t k, const char* dist, uint64_t seed,
                                  int32_t* assignments_host);
/* make_random_params(E, D_i, H, D_o, ., Rng(seed), scale) followed by
 * random_matrix(N, D_i) from the same stream (moe_layer.cpp:136-147,
 * random.hpp:42-54; tools/commands.cpp:174-176), rounded to fp32. */
void hxm_make_layer_inputs(uint64_t seed, int64_t n_experts, int64_t d_in,
                           int64_t hidden, int64_t d_out, int64_t n_tokens,
                           double scale, float* w1, float* b1, float* w2,
                           float* b2, float* x);

/* ------------------------------------------------------------------------
 * Fused GEMM -> reduce-scatter over peer memory (tensor parallelism along H).
 *
 * Under model-centric TP every rank computes the partial y (forward) and the
 * partial g_x (backward) of ALL tokens on its H-slice; the reference sums
 * them with an all-reduce (dist_sim.cpp:483-487, 542).  Here the ESMM
 * epilogues reduce each output row straight into the buffer of the rank that
 * owns the token -- row t goes to rank t / rows_per_rank, local row
 * t % rows_per_rank -- through peer-mapped pointers (NVLink P2P / CUDA IPC),
 * so the reduce-scatter overlaps the GEMM tile by tile and no collective runs
 * afterwards.  Every rank's buffer must be zero before any rank launches, and
 * complete (all ranks' kernels done) before its owner reads it:
 * hxm_peer_barrier orders both over peer flags.
 * ---------------------------------------------------------------------- */
#define HXM_MAX_PEERS 8
typedef struct hxm_peer_rows {
  int32_t n_ranks;          /* P <= HXM_MAX_PEERS                          */
  int32_t reserved;
  int64_t rows_per_rank;    /* token rows owned per rank                   */
  float* ptrs[HXM_MAX_PEERS]; /* rank r's rows_per_rank x D fp32 buffer, as
                               mapped in this process                      */
} hxm_peer_rows;

/* hxm_moe_forward / hxm_moe_backward with y (resp. g_x) reduce-scattered to
 * the owners instead of written to a local N x D buffer. */
hxm_status hxm_moe_forward_tp(const hxm_layer_desc* desc, const void* x,
                              const void* w1, const float* b1, const void* w2,
                              const float* b2, const int32_t* assignments,
                              const hxm_peer_rows* y_rows, void* workspace,
                              size_t workspace_bytes, int32_t* status_dev,
                              hxm_stream_t stream);
hxm_status hxm_moe_backward_tp(const hxm_layer_desc* desc, const void* x,
                               const void* w1, const void* w2, const void* g_y,
                               void* workspace, size_t workspace_bytes,
                               float* gw1, float* gb1, float* gw2, float* gb2,
                               const hxm_peer_rows* gx_rows, hxm_stream_t stream);

/* Data-centric TP: the weight gradients reduce-scattered along H inside the
 * ESTMM epilogues -- gW1 (E x D_i x H) columns h go to rank h / span as its
 * E x D_i x span shard, gW2 (E x H x D_o) rows h to rank h / span as its
 * E x span x D_o shard (span = rows_per_rank of the tables; the reference
 * all-reduces them, dist_sim.cpp:397-398).  gb1, gb2, g_x stay local. */
hxm_status hxm_moe_backward_dc(const hxm_layer_desc* desc, const void* x,
                               const void* w1, const void* w2, const void* g_y,
                               void* workspace, size_t workspace_bytes,
                               const hxm_peer_rows* gw1_shards, float* gb1,
                               const hxm_peer_rows* gw2_shards, float* gb2,
                               float* gx, hxm_stream_t stream);

/* ------------------------------------------------------------------------
 * Tensor-parallel collectives over NCCL (the reference simulates them
 * in-process, dist_sim.cpp:127-176).  `comm` is an ncclComm_t (void*): one
 * the host created itself, or hxm_nccl_comm_init's.  NCCL is loaded at run
 * time; without it these return HXM_ERR_NCCL.  All run on `stream`.
 * ---------------------------------------------------------------------- */
hxm_status hxm_nccl_get_unique_id(unsigned char id[128]);
hxm_status hxm_nccl_comm_init(void** comm, int32_t n_ranks, const unsigned char id[128],
                              int32_t rank);
hxm_status hxm_nccl_comm_destroy(void* comm);

/* Data-centric (run_data_centric, dist_sim.cpp:352-452).  The cache is one
 * buffer of hxm_dc_cache_bytes(desc) holding the whole layer shard-major
 * (desc: the FULL layer, H = P * h); hxm_dc_cache_views gives the w1 / b1 /
 * w2 pointers to pass to hxm_moe_forward / hxm_moe_backward(_dc) with
 * desc.weight_shards = P.  hxm_dc_fill_cache all-gathers this rank's shards
 * (w1 E x D_i x h, b1 fp32 E x h, w2 E x h x D_o) into it
 * (PipelineSharedCache::fill, dist_sim.cpp:367-368); HXM_ERR_CACHE when
 * cache_bytes is too small (CacheError, dist_sim.cpp:104-125).
 * hxm_dc_allreduce_grads sums the parameter gradients over the ranks in
 * place (dist_sim.cpp:397-399; gb2 may be NULL). */
size_t hxm_dc_cache_bytes(const hxm_layer_desc* desc);
hxm_status hxm_dc_cache_views(const hxm_layer_desc* desc, void* cache, void** w1,
                              float** b1, void** w2);
hxm_status hxm_dc_fill_cache(void* comm, const hxm_layer_desc* desc, const void* w1_shard,
                             const float* b1_shard, const void* w2_shard, void* cache,
                             size_t cache_bytes, hxm_stream_t stream);
hxm_status hxm_dc_allreduce_grads(void* comm, const hxm_layer_desc* desc, float* gw1,
                                  float* gb1, float* gw2, float* gb2, hxm_stream_t stream);

/* Model-centric (run_model_centric, dist_sim.cpp:454-601): all_gather_rows
 * of equal per-rank row counts (x, g_y: any dtype, row_bytes each) and of
 * the k x n_local routing (out k x P*n_local, choice-major as
 * RoutingChoice); all_reduce_sum (fp32, in place) of the partial y / g_x. */
hxm_status hxm_tp_allgather_rows(void* comm, const void* local, int64_t rows_per_rank,
                                 int64_t row_bytes, void* out, hxm_stream_t stream);
hxm_status hxm_tp_allgather_assignments(void* comm, const int32_t* local, int64_t k,
                                        int64_t n_local, int32_t* out, hxm_stream_t stream);
hxm_status hxm_tp_allreduce_sum(void* comm, float* buf, int64_t n_elems, hxm_stream_t stream);

/* Peer-shareable device memory and its IPC handles (64 bytes). */
hxm_status hxm_peer_malloc(size_t bytes, void** ptr);
hxm_status hxm_peer_free(void* ptr);
hxm_status hxm_ipc_get_handle(void* ptr, unsigned char handle[64]);
hxm_status hxm_ipc_open_handle(const unsigned char handle[64], void** ptr);
hxm_status hxm_ipc_close_handle(void* ptr);

/* Device-side barrier over peer flags: flags.ptrs[r] is rank r's int32 flag
 * array (HXM_MAX_PEERS entries, zero-initialised, mapped here).  Rank `rank`
 * publishes `epoch` into every rank's slot [rank] (release, system scope) and
 * waits until its own slots all reach `epoch` (acquire).  Epochs increase. */
typedef struct hxm_peer_flags {
  int32_t n_ranks;
  int32_t rank;
  int32_t* ptrs[HXM_MAX_PEERS];
} hxm_peer_flags;
hxm_status hxm_peer_barrier(const hxm_peer_flags* flags, int32_t epoch,
                            hxm_stream_t stream);

/* ------------------------------------------------------------------------
 * Live kernel timing (bench.py roofline) and launch counting.  When enabled,
 * every kernel region is bracketed by CUDA events on its launch stream.
 * ---------------------------------------------------------------------- */
void hxm_profile_enable(int on);
void hxm_profile_reset(void);
/* Aggregates recorded regions by name (synchronises on their events).
 * names: max * name_len chars.  kind: 0 = work is FLOP, 1 = bytes.
 * Returns the number of names written, -1 on a CUDA error. */
int hxm_profile_read(int max, char* names, int name_len, double* total_ms,
                     int64_t* launches, double* work, int32_t* kind);
/* Same aggregation plus the algorithmic HBM bytes of each region (0 when the
 * region only states FLOP): GEMM regions carry both, so a caller can place
 * each kernel under the tensor or the HBM roofline. */
int hxm_profile_read2(int max, char* names, int name_len, double* total_ms,
                      int64_t* launches, double* work, int32_t* kind, double* bytes);
/* Kernels launched by this library since load. */
uint64_t hxm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HEXAMOE_H */
