/*
 * eps_capi.h -- the drop-in C ABI of the B200 PipeTransformer hot path.
 *
 * The reference (arxiv 2102.03161 artifact, /root/reference/proj) exposes a
 * header-only C++ API in namespace `eps` (proj/include/eps/<module>.hpp).  This file
 * is the flat, FFI-friendly boundary over the same operators plus the sm_100a
 * data plane: plain pointers and sizes, caller-owned buffers, `int` status
 * codes and a thread-local error string.  Each entry cites the reference
 * interface it replaces.  INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * The same header is compiled twice:
 *   - into paper_2102_03161_b200/libeps_b200.so (prefix `eps_`), the product;
 *   - into oracle/_ref/libeps_ref.so (prefix `epsref_`, control plane only)
 *     against the *reference's own* sources, which is how the parity tests
 *     compare the two implementations call for call.
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument), 2 domain
 * (std::domain_error), 3 logic (std::logic_error), 4 config (ConfigError),
 * 5 io (IoError), 6 cuda, 7 nccl, 8 capacity (output buffer too small),
 * 9 other.
 */
#ifndef EPS_CAPI_H_
#define EPS_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef EPS_CAPI_PREFIX
#define EPS_FN(name) eps_##name
#else
#define EPS_CAPI_CAT2(a, b) a##b
#define EPS_CAPI_CAT(a, b) EPS_CAPI_CAT2(a, b)
#define EPS_FN(name) EPS_CAPI_CAT(EPS_CAPI_PREFIX, name)
#endif

enum {
  EPS_OK = 0,
  EPS_EINVAL = 1,
  EPS_EDOMAIN = 2,
  EPS_ELOGIC = 3,
  EPS_ECONFIG = 4,
  EPS_EIO = 5,
  EPS_ECUDA = 6,
  EPS_ENCCL = 7,
  EPS_ECAPACITY = 8,
  EPS_EOTHER = 9
};

#define EPS_MAX_STAGES 64

/* ---- value types (mirror the eps:: structs) --------------------------- */

/* ModelSpec (model.hpp:15-30); arrays are caller-owned. */
typedef struct {
  int layers;
  const int64_t* attention_params; /* [layers] */
  const int64_t* mlp_params;       /* [layers] */
  const int64_t* activation_bytes; /* [2*layers+1] */
  int bytes_per_param;
} eps_model_t;

/* ClusterSpec (model.hpp:32-41). */
typedef struct {
  int node_count;
  int gpus_per_node;
  double gpu_memory_bytes;
  double intra_node_bandwidth;
  double inter_node_bandwidth;
} eps_cluster_t;

/* CostModel (cost_model.hpp:11-25), without the transition table. */
typedef struct {
  double c_fwd;
  double backward_ratio;
  double c_update;
  double per_microbatch_overhead;
  double allreduce_bucket_bytes;
  double comm_latency;
} eps_cost_model_t;

/* CacheTierParams (autocache.hpp:11-22). */
typedef struct {
  double host_bandwidth;
  double disk_bandwidth;
  double host_capacity_bytes;
  int window_batches;
  int block_batches;
  double read_latency;
} eps_cache_tiers_t;

/* Active sublayer sequence (SublayerSeq, model.hpp:66-74).  global_index
 * may be NULL: then sublayer i has global index 2*frozen_layers + i. */
typedef struct {
  int n;
  const int64_t* params;
  const int* global_index;
  int64_t frozen_params;
  int frozen_layers;
} eps_seq_t;

/* PartitionPlan (autopipe.hpp:22-34). */
typedef struct {
  int pipeline_length;
  int begin[EPS_MAX_STAGES];
  int end[EPS_MAX_STAGES];
  int64_t param_sums[EPS_MAX_STAGES];
  double effective_sizes[EPS_MAX_STAGES];
  int64_t frozen_params;
  int frozen_layers;
  double lambda_frozen;
} eps_plan_t;

/* StageLoad (schedule.hpp:27-32). */
typedef struct {
  double fwd_params;
  double bwd_params;
  double prefix_seconds_per_sample;
  double in_bytes_per_sample;
} eps_stage_load_t;

/* TimedBlock (schedule.hpp:14-21); kind: 0 F, 1 B, 2 U, 3 XFER, 4 AR. */
typedef struct {
  int device;
  int kind;
  double start;
  double end;
  int micro_batch;
  int bucket;
} eps_block_t;

/* IterationSchedule scalars (schedule.hpp:47-58). */
typedef struct {
  double makespan;
  double compute_makespan;
  double makespan_without_ar;
  double total_bubble;
  double allreduce_seconds;
  double transfer_seconds;
  double compute_seconds;
  double exposed_comm;
  int n_blocks;
} eps_schedule_summary_t;

/* TransitionMessage (autodp.hpp:47-56). */
typedef struct {
  int sender;
  int receiver;
  int epoch;
  double lr_schedule_position;
  int frozen_layers;
  int new_pipeline_length;
  int span_first;
  int span_length;
  char weights_version[32];
} eps_msg_t;

/* EpochRow (runner.hpp:15-31). */
typedef struct {
  int epoch;
  int l_frozen;
  int pipeline_length;
  int replica_width;
  int micro_batches;
  double iteration_time;
  double epoch_time;
  double throughput;
  double bubble_time;
  double comm_time;
  double exposed_comm_time;
  int cache_enabled;
  double transition_overhead;
  double cache_transition_time;
  double stall_time;
} eps_epoch_row_t;

typedef struct {
  double total_seconds;
  double baseline_total_seconds;
  double speedup;
  double comm_ratio;
  double frozen_forward_per_sample;
  double final_prefix_forward_per_sample;
  int n_epochs;
  int n_transitions;
  int n_cache_events;
} eps_run_summary_t;

typedef struct eps_freeze eps_freeze_t;     /* FreezeState */
typedef struct eps_scenario eps_scenario_t; /* ScenarioConfig */

/* ---- errors ----------------------------------------------------------- */
const char* EPS_FN(last_error)(void);

/* ---- model.hpp -------------------------------------------------------- */
/* vit_b16() / bert_large() presets (model.cpp:125-179). */
int EPS_FN(model_preset)(const char* name, int64_t* attention_params, int64_t* mlp_params,
                         int64_t* activation_bytes, int cap_layers, int* layers);
int EPS_FN(model_validate)(const eps_model_t* model);
int EPS_FN(model_prefix_params)(const eps_model_t* model, int layer, int64_t* out);
/* m_partition (model.cpp:79-92). */
int EPS_FN(m_partition)(const eps_model_t* model, int l_frozen, int64_t* params,
                        int* global_index, int cap, int* n, int64_t* frozen_params);

/* ---- freeze.hpp ------------------------------------------------------- */
int EPS_FN(freeze_create)(double alpha, eps_freeze_t** out);
void EPS_FN(freeze_destroy)(eps_freeze_t* state);
int EPS_FN(freeze_frozen_count)(const eps_freeze_t* state, int* out);
/* next_frozen_count (freeze.cpp:22-50). */
int EPS_FN(next_frozen_count)(eps_freeze_t* state, const double* norms, int n_norms,
                              int layer_count, int* out, double* raw_bound);
/* frozen_bound_closed_form (freeze.cpp:52-60). */
int EPS_FN(frozen_bound_closed_form)(int timestep, int layer_count, double alpha, double* out);
/* SyntheticNormSource::at_epoch (freeze.cpp:121-152); profile 0 monotone, 1 early-random. */
int EPS_FN(synthetic_norms)(int profile, uint64_t seed, int layers, int switchover_epoch,
                            int epoch, double* out);
/* TraceNormSource (freeze.cpp:62-113). */
int EPS_FN(trace_norms)(const char* csv_path, int epoch, double* out, int cap, int* layers);

/* ---- autopipe.hpp ----------------------------------------------------- */
/* load_balance (autopipe.cpp:55-122); criterion 0 normalized-stddev, 1 paper-variance. */
int EPS_FN(load_balance)(const eps_seq_t* seq, int partitions, double lambda_frozen,
                         int criterion, eps_plan_t* out);
/* try_compress (autopipe.cpp:124-158). */
int EPS_FN(try_compress)(const eps_seq_t* seq, int current_k, double lambda_frozen,
                         double m_gpu_initial, int criterion, eps_plan_t* out,
                         int* attempt_k, double* attempt_max_eff, int attempt_cap,
                         int* n_attempts);

/* ---- schedule.hpp / chunks.hpp ---------------------------------------- */
/* build_schedule (schedule.cpp:19-199). */
int EPS_FN(build_schedule)(const eps_stage_load_t* stages, int n_stages, int micro_batches,
                           double per_pipeline_batch, int integer_microbatches,
                           int replica_width, int group_spans_nodes, double intra_bandwidth,
                           double inter_bandwidth, int bytes_per_param,
                           const eps_cost_model_t* cm, eps_schedule_summary_t* summary,
                           double* bubble_per_device, eps_block_t* blocks, int block_cap);
/* schedule_iteration (schedule.cpp:233-253). */
int EPS_FN(schedule_iteration)(const eps_plan_t* plan, const eps_model_t* model,
                               const eps_seq_t* seq, int micro_batches,
                               double per_pipeline_batch, int replica_width,
                               const eps_cluster_t* cluster, const eps_cost_model_t* cm,
                               int cache_enabled, double cache_read_seconds_per_sample,
                               eps_schedule_summary_t* summary);
/* optimal_chunks (chunks.cpp:5-24); times_out gets 5K+1 makespans. */
int EPS_FN(optimal_chunks)(const eps_plan_t* plan, const eps_model_t* model,
                           const eps_seq_t* seq, double per_pipeline_batch, int replica_width,
                           const eps_cluster_t* cluster, const eps_cost_model_t* cm,
                           int cache_enabled, double cache_read_seconds_per_sample,
                           int* chosen, double* times_out, int times_cap);

/* ---- autodp.hpp ------------------------------------------------------- */
/* Topology (autodp.cpp:11-79). */
int EPS_FN(topology)(const eps_cluster_t* cluster, int pipeline_length, int* active_ranks,
                     int cap, int* n_active, int* replica_width);
/* transition (autodp.cpp:81-111). */
int EPS_FN(transition)(const eps_cluster_t* cluster, int old_k, int new_k, int epoch,
                       double lr_schedule_position, int frozen_layers,
                       const char* weights_version, eps_msg_t* msgs, int cap, int* n);
/* redistribute (autodp.cpp:113-151): ids holds all shards back to back,
 * offsets[R+1] delimits them, ranks[R] are the owning active ranks. */
int EPS_FN(redistribute)(int64_t dataset_size, const eps_cluster_t* cluster,
                         int pipeline_length, int epoch, uint64_t seed, int* ranks,
                         int64_t* offsets, int64_t* ids);
/* ddp_skip_set (autodp.cpp:153-161). */
int EPS_FN(ddp_skip_set)(const eps_plan_t* plan, const eps_seq_t* seq, int* global_index,
                         int cap, int* n, int64_t* param_count);

/* ---- autocache.hpp ---------------------------------------------------- */
int EPS_FN(cache_read_seconds_per_sample)(const eps_model_t* model, int boundary_layer,
                                          const eps_cache_tiers_t* tiers, double* out);
/* should_cache (autocache.cpp:31-43). */
int EPS_FN(should_cache)(int l_frozen, const eps_model_t* model, const eps_cost_model_t* cm,
                         const eps_cache_tiers_t* tiers, double microbatch_samples,
                         int* enable, double* read_seconds, double* forward_seconds);
/* cache_transition (autocache.cpp:45-67). */
int EPS_FN(cache_transition)(int enabled, int boundary_layer, const eps_cache_tiers_t* tiers,
                             int old_boundary, int new_boundary, const eps_model_t* model,
                             const eps_cost_model_t* cm, double* read_s, double* compute_s,
                             double* write_s);

/* One epoch of the modeled disk -> host window (CacheTierSim,
 * autocache.cpp:69-150) as runner.cpp:258-265 charges it: batches consumed in
 * order, each taking iteration_seconds plus its stall.  out: [total stall s,
 * max resident bytes, prefetches, evictions, sliding (0/1)]. */
int EPS_FN(cache_tier_epoch)(const eps_cache_tiers_t* tiers, double bytes_per_batch,
                             int total_batches, double iteration_seconds, double* out);

/* ---- scenario.hpp / runner.hpp ---------------------------------------- */
int EPS_FN(scenario_load)(const char* path, eps_scenario_t** out);
int EPS_FN(scenario_parse)(const char* json_text, eps_scenario_t** out);
void EPS_FN(scenario_destroy)(eps_scenario_t* cfg);
int EPS_FN(scenario_to_json)(const eps_scenario_t* cfg, char* buf, size_t cap, size_t* len);
/* simulate_run (runner.cpp:94-305). */
int EPS_FN(simulate_run)(const eps_scenario_t* cfg, eps_epoch_row_t* rows, int cap,
                         eps_run_summary_t* summary);
/* Report writers (runner.cpp:340-418): kind 0 csv, 1 timeline json,
 * 2 summary json, 3 transitions jsonl. */
int EPS_FN(simulate_report)(const eps_scenario_t* cfg, int kind, char* buf, size_t cap,
                            size_t* len);
/* speedup_breakdown (runner.cpp:307-338): 6 rungs. */
int EPS_FN(speedup_breakdown)(const eps_scenario_t* cfg, double* total_seconds,
                              double* avg_throughput, double* speedup);
int EPS_FN(parse_flags)(const char* list, int* freeze, int* autopipe, int* autodp,
                        int* autocache);

#ifndef EPS_REFERENCE_BUILD
/* ---- B200 additions: executor-facing control plane -------------------- */

/* EpochPlanner: runner.cpp's decision order for the real training loop. */
typedef struct eps_planner eps_planner_t;
typedef struct {
  int epoch;
  int l_frozen;
  int pipeline_length;
  int replica_width;
  int micro_batches;
  int plan_changed;
  int cache_enabled;
  int cache_boundary;
  int cache_old_boundary;
  int cache_moved;
  int n_messages;
  eps_plan_t plan;
} eps_epoch_decision_t;

int eps_planner_create(const eps_scenario_t* cfg, eps_planner_t** out);
void eps_planner_destroy(eps_planner_t* p);
/* norms_prev: the per-layer norms observed in epoch-1 (length = layers), or
 * NULL to draw them from the scenario's own grad_norms source. */
int eps_planner_begin_epoch(eps_planner_t* p, int epoch, const double* norms_prev,
                            int n_norms, eps_epoch_decision_t* out);
int eps_scenario_model(const eps_scenario_t* cfg, int64_t* attention_params,
                       int64_t* mlp_params, int64_t* activation_bytes, int cap_layers,
                       int* layers, int* bytes_per_param);

/* profile_from_dims for ViT-style frontends (model.hpp additions). */
int eps_vit_profile(int layers, int64_t hidden, int64_t mlp_dim, int image, int patch,
                    int channels, int64_t classes, int64_t* attention_params,
                    int64_t* mlp_params, int64_t* activation_bytes);
int eps_bert_profile(int layers, int64_t hidden, int64_t mlp_dim, int64_t seq_len,
                     int64_t position_table, int64_t vocab, int64_t head_params,
                     int64_t* attention_params, int64_t* mlp_params,
                     int64_t* activation_bytes);
/* Integer micro-batch split (schedule.cpp:28-33). */
int eps_microbatch_sizes(int per_pipeline_batch, int micro_batches, int* sizes);
/* Real DDP bucket plan (schedule.cpp:137-162 order): per bucket, a list of
 * (stage, offset, count) slices.  slice_bucket[i] = bucket of slice i. */
int eps_plan_buckets(const int64_t* stage_params, int n_stages, int bytes_per_param,
                     double bucket_bytes, int* slice_bucket, int* slice_stage,
                     int64_t* slice_offset, int64_t* slice_count, int cap, int* n_slices,
                     int* n_buckets);
/* Grid coordinate of a global rank under K (replica, stage). */
int eps_grid_coord(const eps_cluster_t* cluster, int pipeline_length, int global_rank,
                   int* replica, int* stage);

/* ---- data plane (sm_100a; stream-ordered; device pointers) ------------ */
/* All kernels: bf16 = uint16 storage of bfloat16.  `stream` is a
 * cudaStream_t.  No allocation; no host synchronisation.  Returns EPS_ECUDA
 * on launch failure.  There is no CPU fallback. */

/* GEMM C[M,N] = sum_k A(m,k) B(n,k), bf16 in, fp32 accumulate (tcgen05 +
 * TMEM + TMA).  a_mn_major: A stored [K][M] (M contiguous) instead of
 * [M][K]; b_mn_major: B stored [K][N] instead of [N][K].  lda/ldb/ldc in
 * elements.  epilogue: see EPS_EPI_*.  aux/aux2 per epilogue.  split_k: K
 * splits for EPS_EPI_ACCUM_F32 (0 = choose from the tile count: ~3 units
 * per SM, each split >= 8 k-blocks). */
enum {
  EPS_EPI_STORE_BF16 = 0,     /* C = acc                                     */
  EPS_EPI_BIAS_BF16 = 1,      /* C = acc + bias[n]                           */
  EPS_EPI_BIAS_GELU_BF16 = 2, /* aux = acc + bias (pre-act), C = gelu(aux)   */
  EPS_EPI_BIAS_RESID_BF16 = 3,/* C = acc + bias[n] + aux[m,n] (C may == aux) */
  EPS_EPI_DGELU_BF16 = 4,     /* C = acc * gelu'(aux[m,n]); colsum -> bias   */
  EPS_EPI_STORE_F32 = 5,      /* Cf32 = acc (beta 0)                         */
  EPS_EPI_ACCUM_F32 = 6,      /* Cf32 += acc (split-K / micro-batch accum)   */
  EPS_EPI_RESID_BF16 = 7,     /* C = acc + aux[m,n] (residual-gradient add)  */
  EPS_EPI_ROWDOT_BF16 = 8,    /* C = acc; colsum[m*(N/64) + n/64] += sum over
                                 each 64-column group of bf16(acc)*aux[m,n]
                                 (attention D = rowsum(dO * O) per head, fused
                                 into the dO-producing GEMM; colsum pre-zeroed) */
  EPS_EPI_BIAS_GELU2_BF16 = 9,/* u = acc + bias: C = gelu(u), aux = gelu'(u)
                                 (one tanh for both; the backward then needs
                                 only a product, EPS_EPI_MUL_BF16)             */
  EPS_EPI_MUL_BF16 = 10       /* C = acc * aux[m,n]; colsum -> bias (dGELU
                                 with gelu' stored by EPS_EPI_BIAS_GELU2_BF16) */
};
int eps_gemm_bf16(int a_mn_major, int b_mn_major, int epilogue, const void* A, const void* B,
                  void* C, const float* bias, void* aux, float* colsum, int64_t M, int64_t N,
                  int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int split_k, void* stream);

/* CTA-pair (cta_group::2, 256-row) GEMM tiles: mode 1 on (default), 0 off;
 * mode < 0 only queries.  Returns the mode in effect. */
int eps_gemm_pair_mode(int mode);
/* Diagnostics: every GEMM launch adds its per-role wait cycles to
 * `counters` (device, 7 x uint64: MMA-warp span, its accumulator-empty and
 * operand-full waits, producer slot waits, epilogue warp 0 accumulator-full
 * and store-slot waits, epilogue span; leader CTAs / all CTAs summed).
 * NULL turns it off (the default). */
int eps_gemm_prof(void* counters);
/* Programmatic dependent launch of the GEMM / attention / LayerNorm kernels
 * (each overlaps its launch and prologue with its predecessor's tail): mode
 * 1 on (default), 0 off; mode < 0 only queries. */
int eps_pdl_mode(int mode);

/* LayerNorm over rows of width d (fp32 statistics). */
int eps_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y,
                      float* mean, float* rstd, int64_t rows, int64_t d, float eps,
                      void* stream);
/* dx (+)= LN'(dy); dgamma/dbeta accumulate (fp32).  If dres != NULL the
 * result is dres + LN'(dy) (residual branch fused).  colsum_dx (optional)
 * accumulates column sums of the produced dx (bias grad of the producer). */
int eps_layernorm_bwd(const void* dy, const void* x, const float* gamma, const float* mean,
                      const float* rstd, const void* dres, void* dx, float* dgamma,
                      float* dbeta, float* colsum_dx, int64_t rows, int64_t d,
                      float* workspace, void* stream);

/* Multi-head attention on a packed qkv [B*T, 3*H*dh] (q | k | v, head-major
 * inside each).  out [B*T, H*dh]; lse [B, H, T] fp32. */
int eps_attn_fwd(const void* qkv, void* out, float* lse, int batch, int tokens, int heads,
                 int head_dim, float scale, void* stream);
/* dqkv (bf16, same layout as qkv) is fully overwritten; dbias_qkv (fp32
 * [3*H*dh], optional) accumulates its column sums; dsum_workspace: fp32
 * [batch*heads*tokens] scratch. */
int eps_attn_bwd_ws(const void* qkv, const void* out, const void* dout, const float* lse,
                    void* dqkv, float* dbias_qkv, float* dsum_workspace, int batch, int tokens,
                    int heads, int head_dim, float scale, void* stream);

/* Backward with D = rowsum(dO * O) precomputed per (row, head) as fp32
 * [batch*tokens, heads] (e.g. by EPS_EPI_ROWDOT_BF16 on the GEMM producing
 * dout).  Used by the fused persistent kernel (head_dim 64, tokens <= 256);
 * other shapes ignore dsum_rows and use dsum_workspace as eps_attn_bwd_ws. */
int eps_attn_bwd_rowdot(const void* qkv, const void* out, const void* dout, const float* lse,
                        const float* dsum_rows, void* dqkv, float* dbias_qkv,
                        float* dsum_workspace, int batch, int tokens, int heads, int head_dim,
                        float scale, void* stream);
/* 1 if eps_attn_bwd_rowdot consumes dsum_rows for this shape. */
int eps_attn_bwd_uses_rowdot(int tokens, int head_dim);

/* Profiling aid: clock64 phase stamps of CTA 0 of the fused attention
 * backward (layout documented in attention_tc.cu); off unless enabled. */
int eps_attn_trace_enable(int on);
int eps_attn_trace_read(long long* out, int n);

/* Flat-arena form: segment s = flat[seg_offsets[s], seg_offsets[s+1]) (host
 * offsets, <= 64 segments); out: device double[n_segments]; workspace >=
 * 8 * ceil(total / 65536) bytes. */
int eps_grad_sqnorm_flat(const float* flat, const int64_t* seg_offsets, int n_segments,
                         double* out, void* workspace, size_t workspace_bytes, void* stream);
/* Per-layer sum of squares of fp32 gradient tensors (freeze test).  Tensor i
 * (length n[i]) belongs to segment seg[i]; out[s] = sum over its tensors
 * (fp64 accumulation, fixed order => deterministic). */
int eps_grad_sqnorm_segmented(const float* const* tensors, const int64_t* n, const int* seg,
                              int n_tensors, double* out, int n_segments, void* workspace,
                              size_t workspace_bytes, void* stream);

/* AutoCache store: rows of row_bytes, keyed by sample id. */
int eps_cache_gather(const void* store, const int64_t* ids, int n, int64_t row_bytes,
                     void* dst, void* stream);
/* Same gather on `ctas` CTAs (grid-stride, four 16-byte loads in flight per
 * thread): the host tier's prefetch window runs it on a copy stream beside the
 * compute kernels. */
int eps_cache_gather_bg(const void* store, const int64_t* ids, int n, int64_t row_bytes,
                        void* dst, int ctas, void* stream);
int eps_cache_scatter(void* store, const int64_t* ids, int n, int64_t row_bytes,
                      const void* src, void* stream);
/* Store sharded over the GPUs of a node (autodp.cpp:113-151:
 * redistribute moves samples between replicas every epoch): `shards` is a
 * device array of n base pointers (local or CUDA-IPC-mapped peer HBM), shard
 * r holding sample rows [r * rows_per_shard, (r + 1) * rows_per_shard).  The
 * gather reads (the scatter writes) the owning GPU's HBM over NVLink. */
int eps_cache_gather_sharded(const uint64_t* shards, int64_t rows_per_shard, const int64_t* ids,
                             int n, int64_t row_bytes, void* dst, void* stream);
int eps_cache_scatter_sharded(const uint64_t* shards, int64_t rows_per_shard, const int64_t* ids,
                              int n, int64_t row_bytes, const void* src, void* stream);

/* Fused SGD-momentum over an fp32 master copy + bf16 working copy:
 * v = mu*v + g (+wd*p); p -= lr*v; p_bf16 = bf16(p); g = 0. */
int eps_sgd_momentum(float* param, uint16_t* param_bf16, float* grad, float* momentum,
                     int64_t n, float lr, float mu, float weight_decay, void* stream);
/* Fused AdamW over the same layout (step is 1-based). */
int eps_adamw(float* param, uint16_t* param_bf16, float* grad, float* m, float* v, int64_t n,
              float lr, float beta1, float beta2, float eps, float weight_decay, int step,
              void* stream);

/* ViT frontend / head helpers.  eps_patchify: `image` = model side, or
 * (stored side << 16) | model side to nearest-upsample a smaller stored
 * image (CIFAR-shaped 32x32 -> 224) inside the same pass. */
int eps_patchify(const float* images, void* patches, int batch, int channels, int image,
                 int patch, void* stream);
int eps_vit_assemble(const void* patch_tokens, const float* cls, const float* pos, void* x,
                     int batch, int tokens, int64_t d, void* stream);
int eps_vit_assemble_bwd(const void* dx, float* dcls, float* dpos, void* dpatch_tokens,
                         int batch, int tokens, int64_t d, void* stream);
/* Softmax cross-entropy over logits [B, C] (bf16): loss_sum += sum_b
 * -log p(label); dlogits = (p - onehot)/B in bf16. */
int eps_softmax_xent(const void* logits, const int64_t* labels, void* dlogits, float* loss_sum,
                     int batch, int classes, void* stream);
/* Same with an explicit gradient scale (1/global batch under micro-batching)
 * plus column sums of dlogits into dbias (fp32 [classes]). */
int eps_softmax_xent_bias(const void* logits, const int64_t* labels, void* dlogits,
                          float* loss_sum, float* dbias, int batch, int classes, int ld,
                          float grad_scale, void* stream);
int eps_gather_rows(const void* src, int64_t src_stride_rows, void* dst, int rows, int64_t d,
                    int64_t offset_rows, void* stream);
int eps_scatter_rows(const void* src, void* dst, int64_t dst_stride_rows, int rows, int64_t d,
                     int64_t offset_rows, void* stream);
int eps_colsum_bf16(const void* x, float* out, int64_t rows, int64_t cols, void* stream);
/* Seeded synthetic data: dst[i] ~ N(0, 1) / uniform in [0, classes), a pure
 * function of (seed, i) (SplitMix64 finaliser + Box-Muller). */
int eps_fill_normal(float* dst, int64_t n, uint64_t seed, void* stream);
int eps_fill_labels(int64_t* dst, int64_t n, int64_t classes, uint64_t seed, void* stream);

/* ---- peer memory (csrc/runtime/peer.cu) ---------------------------------- */
/* CUDA IPC export of the allocation holding dev_ptr: 64-byte handle + byte
 * offset of dev_ptr inside it. */
int eps_ipc_export(const void* dev_ptr, void* handle, int64_t* offset);
/* Map a peer allocation: *base for eps_ipc_close, *dev_ptr = base + offset. */
int eps_ipc_open(const void* handle, int64_t offset, void** base, void** dev_ptr);
int eps_ipc_close(void* base);
/* Stream-ordered flag protocol: signal = system-scope release store of
 * `value` to `flag` (may be a peer address) after all prior work on the
 * stream; wait = the stream blocks (cuStreamWaitValue32, GEQ) until the local
 * `flag` reaches `value`. */
int eps_peer_signal(void* flag, uint32_t value, void* stream);
int eps_peer_wait(const void* flag, uint32_t value, void* stream);
/* Stream-ordered device copy (peer addresses allowed, UVA). */
int eps_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Stream-ordered 2D copy (UVA, any direction): `height` rows of `width`
 * bytes with row pitches dpitch / spitch (disk-tier window -> HBM staging). */
int eps_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                     int64_t height, void* stream);
/* Page-lock / release an existing host range (cudaHostRegister, portable +
 * mapped): the node-wide shared-memory host tier of the AutoCache store. */
int eps_host_register(void* ptr, int64_t bytes);
int eps_host_unregister(void* ptr);

/* ---- AutoCache disk tier (csrc/runtime/disk_tier.cpp) ---------------------
 * Replaces the reference's modeled disk -> host sliding window,
 * CacheTierSim (autocache.cpp:69-150; CacheTierParams autocache.hpp:11-20:
 * window_batches, block_batches), with real I/O: a backing file of `rows`
 * cached samples (row_bytes each, padded to 4 KiB, O_DIRECT when the
 * filesystem allows) and a page-locked host window of
 * window_batches / block_batches block slots filled by `threads` I/O threads
 * in the epoch's consumption order.  Host memory only, no CUDA calls on the
 * data path; the window is cudaHostRegister'ed when a device is present.
 *   open: create != 0 makes / truncates the file (one node-wide file; ranks
 *         open it after the creator);
 *   write: rows `ids` from host rows `src` (src_stride bytes apart);
 *   begin_epoch: the epoch's sample order; batches of batch_rows rows (last
 *         ragged) or, with batch_offsets (n_batches + 1 entries, each batch <=
 *         batch_rows), explicit ones; stages the leading window
 *         (CacheTierSim constructor);
 *   acquire: blocks until batch `batch` (batch_rows rows of the order) is
 *         resident; *rows = its first row (rows `stride` bytes apart,
 *         eps_disk_tier_info), *stall_s = the wait (WindowStep::stall_seconds);
 *         EPS_ELOGIC if the batch lies beyond the window (release earlier
 *         batches first, batches are consumed in order as in
 *         CacheTierSim::advance);
 *   release: the batch is consumed; fully consumed blocks are evicted and
 *         their slots refilled with the next blocks (issue_prefetches);
 *   stats: [bytes read, I/O-thread read seconds, stall seconds, max resident
 *         window bytes, prefetches, evictions, bytes written, O_DIRECT]. */
typedef struct eps_disk_tier eps_disk_tier_t;
int eps_disk_tier_open(const char* path, int64_t rows, int64_t row_bytes, int64_t batch_rows,
                       int block_batches, int window_batches, int threads, int create,
                       eps_disk_tier_t** out);
int eps_disk_tier_close(eps_disk_tier_t* h);
int eps_disk_tier_info(eps_disk_tier_t* h, int64_t* stride, int* direct, int* window_blocks,
                       void** window);
int eps_disk_tier_write(eps_disk_tier_t* h, const int64_t* ids, int64_t n, const void* src,
                        int64_t src_stride);
int eps_disk_tier_begin_epoch(eps_disk_tier_t* h, const int64_t* order, int64_t n,
                              const int64_t* batch_offsets, int64_t n_batches);
int eps_disk_tier_acquire(eps_disk_tier_t* h, int64_t batch, const void** rows,
                          int64_t* n_rows, double* stall_s);
int eps_disk_tier_release(eps_disk_tier_t* h, int64_t batch);
int eps_disk_tier_stats(eps_disk_tier_t* h, double* out);

/* ---- communicator plane (csrc/runtime/comm.cpp; NCCL) ----
 * The reference's message group (every rank) and training group (active
 * pipeline heads), autodp.hpp:17-21 / autodp.cpp:31-37, as NCCL
 * communicators: a world communicator from a 128-byte unique id (rank 0
 * creates it, the host exchanges it out of band), per-stage data-parallel
 * communicators split from it (color = stage, key = pipeline; color < 0 =
 * not a member, *out = NULL), rebuilt when freezing changes K.  Every
 * operation is stream-ordered on `stream` (cudaStream_t) and never
 * synchronises the host.  NCCL is loaded at run time; without it every entry
 * returns EPS_ENCCL (eps_last_error names the cause). */
typedef struct eps_comm eps_comm_t;
enum { EPS_DT_F32 = 0, EPS_DT_F64 = 1, EPS_DT_BF16 = 2, EPS_DT_U8 = 3, EPS_DT_I64 = 4 };
enum { EPS_OP_SUM = 0, EPS_OP_AVG = 1, EPS_OP_MAX = 2 };
int eps_comm_version(int* version);
int eps_comm_unique_id(void* id /* 128 bytes */);
int eps_comm_world_init(const void* id, int nranks, int rank, eps_comm_t** out);
int eps_comm_split(eps_comm_t* parent, int color, int key, eps_comm_t** out);
int eps_comm_free(eps_comm_t* comm);
int eps_comm_rank(const eps_comm_t* comm, int* rank, int* size);
/* In-place all-reduce of `count` elements of `dtype` with `op`. */
int eps_allreduce(eps_comm_t* comm, void* buf, int64_t count, int dtype, int op, void* stream);
/* One DDP gradient bucket (schedule.cpp:137-178): fp32 in place, average =
 * ncclAvg (the 1/R mean inside the collective, no extra scaling pass). */
int eps_allreduce_bucket(eps_comm_t* comm, float* grads, int64_t count, int average,
                         void* stream);
/* Byte broadcast from comm rank `root` (parameter / momentum migration on a
 * transition, autodp.cpp:81-111). */
int eps_broadcast(eps_comm_t* comm, void* buf, int64_t bytes, int root, void* stream);
/* Stage-to-stage cut activations / gradients (schedule.cpp:60-68, 97-105);
 * pair sends and receives inside eps_comm_group_start / _end. */
int eps_p2p_send(eps_comm_t* comm, const void* buf, int64_t bytes, int peer, void* stream);
int eps_p2p_recv(eps_comm_t* comm, void* buf, int64_t bytes, int peer, void* stream);
int eps_comm_group_start(void);
int eps_comm_group_end(void);

/* Kernels launched by this library in this process (launch accounting). */
unsigned long long eps_launch_count(void);

/* ---- ViT stage executor (csrc/runtime/vit.cu) --------------------------- */
/* geom = {layers, d, mlp_dim, heads, tokens, classes, image, stored_image,
 *         patch, channels, max_batch}. */
typedef struct eps_vit eps_vit_t;
int eps_vit_layout(const int* geom, int64_t* param_total, int64_t* workspace_bytes,
                   int64_t* segments, int64_t* tensors);
int eps_vit_create(const int* geom, float* params, uint16_t* params_bf16, float* grads,
                   float* momentum, void* workspace, eps_vit_t** out);
void eps_vit_destroy(eps_vit_t* h);
int eps_vit_train_step(eps_vit_t* h, const float* images, const int64_t* labels, int batch,
                       int micro_batches, int l_frozen, int cache_mode, int cache_old,
                       void* store, const int64_t* ids, float* loss_sum, void* stream);
int eps_vit_sgd(eps_vit_t* h, int l_frozen, float lr, float momentum, float weight_decay,
                void* stream);
int eps_vit_layer_sqnorms(eps_vit_t* h, int l_frozen, double* out, void* stream);
int eps_vit_forward_logits(eps_vit_t* h, const float* images, int batch, void* logits,
                           void* stream);
void* eps_vit_activation(eps_vit_t* h, int which, int layer);

/* ---- native single-GPU training loop (csrc/runtime/trainer.cpp) --------
 * The reference's epoch loop (runner.cpp:139-298 decision order through
 * EpochPlanner, redistribute, AutoCache modes, ragged last iteration) run on
 * one GPU by the ViT executor with device gradient norms feeding the freeze
 * decision -- the C++ host path of trainer.py:Trainer for a 1 x 1 cluster.
 * kind: EPS_MODEL_VIT (geom as eps_vit_layout) or EPS_MODEL_BERT (geom as
 * eps_bert_layout).  init_params_host: fp32 [param_total] in the executor's
 * layout (NULL: seeded trunc-normal init); inputs_dev / labels_dev: the dataset
 * (N = iterations x per_pipeline_batch samples; ViT fp32 images [N, C, H, W],
 * BERT int64 [2, N, T] token then segment ids; labels int64 [N], SQuAD head
 * [2, N] start then end) or NULL for seeded synthetic data.  EPS_EINVAL for
 * clusters other than 1 x 1. */
typedef struct eps_trainer eps_trainer_t;
enum { EPS_MODEL_VIT = 0, EPS_MODEL_BERT = 1 };
typedef struct {
  int epoch, l_frozen, pipeline_length, replica_width, micro_batches;
  int cache_enabled, cache_moved, cache_mode; /* cache_mode: 0 off, 1 gather, 2 move, 3 trailing */
  int iterations;
  double epoch_time_s, iteration_time_s, throughput_sps, samples, mean_loss;
  double cache_transition_time_s;
} eps_train_epoch_t;
int eps_trainer_create(const eps_scenario_t* scenario, int kind, const int* geom,
                       int iterations_per_epoch, uint64_t seed, float lr, float momentum,
                       int device_norms, const float* init_params_host, const void* inputs_dev,
                       const int64_t* labels_dev, eps_trainer_t** out);
/* One epoch; norms_out (host double[L], may be NULL) receives the per-layer
 * gradient L2 norms the next epoch's freeze test reads. */
int eps_trainer_run_epoch(eps_trainer_t* t, int epoch, eps_train_epoch_t* out, double* norms_out);
void eps_trainer_destroy(eps_trainer_t* t);

/* Pipeline-stage operations (AutoPipe executor).  Global sublayer g in
 * [0, 2L): layer g/2, ATT if even, MLP if odd (SublayerSeq order,
 * model.hpp:56-74); a stage owns global sublayers [g0, g1) with
 * g0 >= 2*l_frozen (PartitionPlan spans shifted by 2*l_frozen).  The host
 * drives the GPipe order of schedule.cpp:54-117 and moves the cut
 * activations (eps_vit_cut) between stages.
 * front = 1 on pipeline stage 0: frozen prefix / AutoCache / embedding first.
 * cache_mode (AutoCache, autocache.cpp:45-67 / runner.cpp:180-213):
 *   0 recompute the frozen prefix [0, l_frozen);
 *   1 gather X[l_frozen] from store rows `ids` (prefix skipped);
 *   2 boundary move cache_old -> l_frozen: gather X[cache_old] (cache_old > 0)
 *     or embed, forward [cache_old, l_frozen), scatter X[l_frozen];
 *   3 trailing boundary: gather X[cache_old] (0 < cache_old < l_frozen),
 *     forward [cache_old, l_frozen), write nothing. */
int eps_vit_stage_forward(eps_vit_t* h, const float* images, int b0, int b, int g0, int g1,
                          int l_frozen, int front, int cache_mode, int cache_old, void* store,
                          const int64_t* ids, void* stream);
/* Last stage: final LN + head forward, softmax-xent loss (grad scale
 * 1/global_batch), head backward; leaves dL/dX[L] in the dX rows. */
int eps_vit_stage_head(eps_vit_t* h, const int64_t* labels, int b0, int b, int global_batch,
                       float* loss_sum, void* stream);
/* Backward of [g0, g1) with dL/d(output of g1-1) in the dX rows; leaves
 * dL/d(input of g0) there.  cut_out = 1 when that gradient came from the next
 * stage (this stage then adds its column sum into sublayer g1-1's bias grad). */
int eps_vit_stage_backward(eps_vit_t* h, int b0, int b, int g0, int g1, int l_frozen,
                           int cut_out, void* stream);
/* Same over a piece [g0, g1) of a stage whose lowest sublayer is stage_g0
 * (pieces walked top-down; cut_out only on the topmost piece) -- lets the
 * host launch a gradient bucket's all-reduce as soon as its sublayers are done. */
int eps_vit_stage_backward_part(eps_vit_t* h, int b0, int b, int g0, int g1, int stage_g0,
                                int l_frozen, int cut_out, void* stream);
/* Residual-stream buffer [max_batch*T, d] bf16 at the cut before global
 * sublayer g (g == 2L: the stack output), or (grad = 1) the dX scratch. */
void* eps_vit_cut(eps_vit_t* h, int g, int grad);
/* Stage hand-off over peer memory: write the output cut `out_g` into
 * out_ptr (the next stage's cut buffer, IPC-mapped) and the gradient at the
 * input cut `dx_g` into dx_ptr (the previous stage's dX buffer) directly from
 * the producing kernel.  NULL pointers restore local writes. */
/* AutoCache store sharded over the node (see eps_cache_gather_sharded):
 * `table` = device uint64[n] of shard bases, `rows_per_shard` rows each; the
 * stage calls' store argument is then only a non-null marker.  null reverts. */
int eps_vit_set_cache_shards(eps_vit_t* h, const uint64_t* table, int64_t rows_per_shard);
int eps_vit_set_redirect(eps_vit_t* h, int out_g, void* out_ptr, int dx_g, void* dx_ptr);
/* Parameter elements [begin, end) of global sublayers [g0, g1) (embedding in
 * sublayer 0, final LN + head in sublayer 2L-1); contiguous by layout. */
int eps_vit_param_range(eps_vit_t* h, int g0, int g1, int64_t* begin, int64_t* end);
int eps_vit_sgd_range(eps_vit_t* h, int64_t begin, int64_t end, float lr, float momentum,
                      float weight_decay, void* stream);
/* Sum of squares of the fp32 gradient arena over n consecutive ranges
 * offsets[i]..offsets[i+1] (host offsets) into device double out[n]. */
int eps_vit_sqnorm_ranges(eps_vit_t* h, const int64_t* offsets, int n, double* out,
                          void* stream);
/* Per-kernel-class CUDA-event timing of the executor's launches (bench /
 * roofline).  While enabled every launch is bracketed by events on its
 * stream.  eps_vit_timing_read synchronises the recorded events and returns,
 * per class c (EPS_TC_*), ms[c] total device time, flops[c] algorithmic
 * FLOPs (2MNK per GEMM; 4T^2 d per attention forward, 2x backward), bytes[c]
 * algorithmic HBM bytes, count[c] launches; then clears the record. */
enum {
  EPS_TC_GEMM = 0,
  EPS_TC_ATTN = 1,
  EPS_TC_NORM = 2,
  EPS_TC_ELTWISE = 3,
  EPS_TC_CACHE = 4,
  EPS_TC_OPTIM = 5,
  EPS_TC_SQNORM = 6,
  EPS_TC_COUNT = 7
};
/* Weight-gradient GEMMs on a side stream beside the input-gradient chain
 * (default on; EPS_SIDE_STREAM=0 disables the stream at creation). */
int eps_vit_set_side_stream(eps_vit_t* h, int on);
int eps_vit_timing_enable(eps_vit_t* h, int on);
int eps_vit_timing_read(eps_vit_t* h, double* ms, double* flops, double* bytes, int64_t* count);
/* ---- BERT front end / heads (csrc/kernels/bert_ops.cu) ------------------ */
/* E[b*T+t] = word[tok] + pos[t] + type[seg] (fp32 tables -> bf16 rows). */
int eps_bert_embed_fwd(const int64_t* tokens, const int64_t* segments, const float* word,
                       const float* pos, const float* type, void* out, int batch,
                       int tokens_per_sample, int64_t d, void* stream);
/* Scatter-add of dE rows into the fp32 word / position / type gradients. */
int eps_bert_embed_bwd(const void* d_embed, const int64_t* tokens, const int64_t* segments,
                       float* dword, float* dpos, float* dtype, int batch,
                       int tokens_per_sample, int64_t d, void* stream);
/* SQuAD span loss over logits [batch*T, ld] (columns 0 start, 1 end):
 * loss_sum += sum_b (CE_start + CE_end)/2; dlogits scaled by grad_scale;
 * dbias[0..1] += column sums of dlogits. */
int eps_span_xent(const void* logits, const int64_t* start, const int64_t* end, void* dlogits,
                  float* loss_sum, float* dbias, int batch, int tokens_per_sample, int ld,
                  float grad_scale, void* stream);
int eps_tanh_fwd(const void* x, void* y, int64_t n, void* stream);
int eps_tanh_bwd(const void* dy, const void* y, void* dx, int64_t n, void* stream);

/* ---- BERT stage executor (csrc/runtime/bert.cu) -------------------------- */
/* Same contract as eps_vit_*; geom = {layers, d, mlp_dim, heads, tokens,
 * classes, vocab, positions, head_kind (0 pooled CLS, 1 SQuAD span), pooler,
 * max_batch}.  `state` holds the optimizer state: momentum (SGD) or m | v
 * (AdamW, 2 x param_total).  Front-stage inputs: int64 tokens [batch_rows*T]
 * followed by segment ids [batch_rows*T]; labels: class [gb] (head 0) or
 * start [gb] followed by end [gb] (head 1). */
typedef struct eps_bert eps_bert_t;
int eps_bert_layout(const int* geom, int64_t* param_total, int64_t* workspace_bytes,
                    int64_t* segments, int64_t* tensors);
int eps_bert_create(const int* geom, float* params, uint16_t* params_bf16, float* grads,
                    float* state, void* workspace, eps_bert_t** out);
void eps_bert_destroy(eps_bert_t* h);
int eps_bert_stage_forward(eps_bert_t* h, const int64_t* inputs, int batch_rows, int b0, int b,
                           int g0, int g1, int l_frozen, int front, int cache_mode, int cache_old,
                           void* store, const int64_t* ids, void* stream);
int eps_bert_stage_head(eps_bert_t* h, const int64_t* labels, int b0, int b, int global_batch,
                        float* loss_sum, void* stream);
int eps_bert_stage_backward(eps_bert_t* h, int b0, int b, int g0, int g1, int l_frozen,
                            int cut_out, void* stream);
int eps_bert_stage_backward_part(eps_bert_t* h, int b0, int b, int g0, int g1, int stage_g0,
                                 int l_frozen, int cut_out, void* stream);
void* eps_bert_cut(eps_bert_t* h, int g, int grad);
/* AutoCache store sharded over the node (see eps_cache_gather_sharded):
 * `table` = device uint64[n] of shard bases, `rows_per_shard` rows each; the
 * stage calls' store argument is then only a non-null marker.  null reverts. */
int eps_bert_set_cache_shards(eps_bert_t* h, const uint64_t* table, int64_t rows_per_shard);
int eps_bert_set_redirect(eps_bert_t* h, int out_g, void* out_ptr, int dx_g, void* dx_ptr);
int eps_bert_param_range(eps_bert_t* h, int g0, int g1, int64_t* begin, int64_t* end);
int eps_bert_sgd_range(eps_bert_t* h, int64_t begin, int64_t end, float lr, float momentum,
                       float weight_decay, void* stream);
int eps_bert_adamw_range(eps_bert_t* h, int64_t begin, int64_t end, float lr, float beta1,
                         float beta2, float eps, float weight_decay, int step, void* stream);
int eps_bert_sqnorm_ranges(eps_bert_t* h, const int64_t* offsets, int n, double* out,
                           void* stream);
int eps_bert_timing_enable(eps_bert_t* h, int on);
int eps_bert_timing_read(eps_bert_t* h, double* ms, double* flops, double* bytes,
                         int64_t* count);
#endif /* EPS_REFERENCE_BUILD */

#ifdef __cplusplus
}
#endif

#endif /* EPS_CAPI_H_ */
