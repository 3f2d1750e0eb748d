/*
 * dwdp.h — C-ABI of the B200-native DWDP MoE hot path.
 *
 * Plain C types only (no torch, no CUDA headers): device pointers are
 * `void*`, CUDA streams are passed as `void*` (a cudaStream_t / CUstream).
 * Every entry point that can fail returns a status code; the message of the
 * last failure on the calling thread is available from dwdp_last_error().
 *
 * Each declaration names the reference interface it replaces
 * (/root/reference/proj/<file>:<line>). The planners are pure and
 * reentrant; a dwdp_ctx is owned by one host thread driving one GPU.
 */
#ifndef DWDP_H
#define DWDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------
 * Replaces the exception convention of include/dwdpsim/errors.hpp:11-28
 * (ConfigError -> CLI exit 2, InvariantViolation -> exit 3, mapped in
 * tools/dwdpsim_main.cpp:328-337). */
#define DWDP_OK 0
#define DWDP_ERR_CONFIG 2    /* ConfigError: invalid user input           */
#define DWDP_ERR_INVARIANT 3 /* InvariantViolation: internal bug          */
#define DWDP_ERR_CUDA 4      /* CUDA / driver failure, or no sm_100 device */

const char* dwdp_last_error(void);
/* Library build string (arch, CUDA version). */
const char* dwdp_version(void);

/* ======================================================================
 * Expert placement table — include/dwdpsim/placement.hpp:13-43.
 * ==================================================================== */
typedef struct dwdp_placement dwdp_placement;

/* build_placement(num_experts, group_size, extra_redundancy)
 * (placement.hpp:30-34, src/placement.cpp:75-111). */
int dwdp_placement_build(int num_experts, int group_size, int extra_redundancy,
                         dwdp_placement** out);
void dwdp_placement_free(dwdp_placement* p);
/* PlacementPlan fields (placement.hpp:13-25). */
int dwdp_placement_info(const dwdp_placement* p, int* group_size,
                        int* num_experts, int* local_count, int* redundancy);
/* local_sets[rank] (sorted), `experts` holds local_count entries. */
int dwdp_placement_local_set(const dwdp_placement* p, int rank, int* experts);
/* fetch_lists[rank] = (expert, source rank), E - local_count entries. */
int dwdp_placement_fetch_list(const dwdp_placement* p, int rank, int* experts,
                              int* sources);
/* PlacementPlan::holds (src/placement.cpp:10-13). */
int dwdp_placement_holds(const dwdp_placement* p, int rank, int expert,
                         int* holds);
/* PlacementPlan::validate (src/placement.cpp:15-45): 0 or 3. */
int dwdp_placement_validate(const dwdp_placement* p);
/* A placement handle from a plan held as plain tables (the value type of
 * the C++/Python mirrors, possibly edited by the caller), checked with
 * PlacementPlan::validate: status 3 on a broken invariant. local_sets[r] =
 * local_flat[local_offsets[r] .. local_offsets[r+1]); fetch_lists[r] =
 * (fetch_experts, fetch_sources)[fetch_offsets[r] .. fetch_offsets[r+1]). */
int dwdp_placement_from_tables(int group_size, int num_experts, int local_count,
                               int redundancy, const int* local_offsets,
                               const int* local_flat, const int* fetch_offsets,
                               const int* fetch_experts,
                               const int* fetch_sources,
                               dwdp_placement** out);
/* prefetch_bytes = (E - c) * expert_shard_bytes (src/placement.cpp:113-116). */
int dwdp_prefetch_bytes(const dwdp_placement* p, double expert_shard_bytes,
                        double* bytes);
/* describe_placement (src/placement.cpp:118-150). *len in: capacity, out:
 * bytes needed including the terminator. */
int dwdp_placement_describe(const dwdp_placement* p, char* buf, size_t* len);
/* assign_fetch_sources(num_experts, local_sets) (src/placement.cpp:47-73).
 * local_sets is ragged: rank r owns local_flat[local_offsets[r] ..
 * local_offsets[r+1]). Output per rank r: fetch_counts[r] entries starting
 * at r * num_experts in fetch_experts / fetch_sources. */
int dwdp_assign_fetch_sources(int num_experts, int group_size,
                              const int* local_offsets, const int* local_flat,
                              int* fetch_counts, int* fetch_experts,
                              int* fetch_sources);

/* ======================================================================
 * TDM copy plan — include/dwdpsim/copyplan.hpp:15-51.
 * ==================================================================== */
typedef struct { /* ShardRef (copyplan.hpp:17-22) */
  int32_t peer;
  int32_t reserved;
  uint64_t param_id;
  uint64_t size;
  uint64_t src_offset;
} dwdp_shard_ref;

typedef struct { /* Slice (copyplan.hpp:24-30) */
  uint64_t param_id;
  int32_t src_rank;
  int32_t reserved;
  uint64_t src_offset;
  uint64_t dst_offset; /* relative to the per-(peer, param) buffer */
  uint64_t length;
} dwdp_slice;

/* build_copy_plan(shards, slice_size, dst_rank) (src/copyplan.cpp:25-80).
 * Size query when out == NULL: *n_inout receives the slice count. */
int dwdp_copy_plan_build(const dwdp_shard_ref* shards, size_t n_shards,
                         uint64_t slice_size, int dst_rank, dwdp_slice* out,
                         size_t* n_inout);
/* source_queues(plans, source) (src/copyplan.cpp:82-92): for each plan (in
 * ascending dst order, one queue per distinct dst even if empty) the slices
 * served by `source`, plan order preserved. out_dsts/out_counts receive
 * *n_queues entries (capacity n_plans); `out` the concatenated slices. */
int dwdp_source_queues(size_t n_plans, const int* dst_ranks,
                       const dwdp_slice* const* plans, const size_t* plan_lens,
                       int source, int* out_dsts, size_t* out_counts,
                       size_t* n_queues, dwdp_slice* out, size_t* n_inout);

/* ======================================================================
 * Workload generator — include/dwdpsim/workload.hpp:14-79, rng.hpp.
 * ==================================================================== */
#define DWDP_ISL_FIXED 0
#define DWDP_ISL_UNIFORM_RATIO 1
#define DWDP_ISL_NORMAL 2

typedef struct { /* WorkloadSpec + IslDist (workload.hpp:14-43) */
  int32_t isl_kind;
  int32_t batch_per_rank;
  double length; /* Fixed: length; UniformRatio: max; Normal: mean */
  double ratio;
  double stddev;
  int64_t max_num_tokens;
  double routing_skew;
  uint64_t seed;
} dwdp_workload_spec;

/* Rng::mix (rng.hpp:60-69). */
uint64_t dwdp_rng_mix(uint64_t a, uint64_t b);
/* route_tokens (src/workload.cpp:85-111): counts[num_experts]. */
int dwdp_route_tokens(int64_t tokens, int num_experts, int top_k,
                      double routing_skew, uint64_t seed, int64_t* counts);
/* sample_batches (src/workload.cpp:137-173): tokens/requests
 * [iterations][num_ranks]; routed (nullable) [iterations][num_ranks][E]. */
int dwdp_sample_batches(const dwdp_workload_spec* spec, int num_experts,
                        int top_k, int num_ranks, int iterations,
                        int64_t* tokens, int64_t* requests, int64_t* routed);
/* WorkloadSpec::validate + IslDist::validate (src/workload.cpp:10-22, 66-77). */
int dwdp_workload_validate(const dwdp_workload_spec* spec);
/* batches_to_csv (src/workload.cpp:191-208): the reference's replay format.
 * routed (nullable) [iterations][num_ranks][num_experts]; *len_inout =
 * capacity in, bytes needed (incl. NUL) out. */
int dwdp_batches_to_csv(const int64_t* tokens, const int64_t* requests,
                        const int64_t* routed, int iterations, int num_ranks,
                        int num_experts, char* buf, size_t* len_inout);
/* batches_from_csv (src/workload.cpp:210-247). First call with NULL arrays
 * returns the shape: *iterations, *num_ranks, *num_experts (the longest
 * expert-count row; 0 if the file carries no routing). Second call fills
 * tokens/requests [it][rank] and routed [it][rank][num_experts] (rows shorter
 * than num_experts zero-padded; routed_len[it][rank] = their length). */
int dwdp_batches_from_csv(const char* csv, int* iterations, int* num_ranks,
                          int* num_experts, int64_t* tokens, int64_t* requests,
                          int64_t* routed, int32_t* routed_len);
/* imbalance_cv (src/workload.cpp:175-189). */
int dwdp_imbalance_cv(const int64_t* tokens, int n, double* cv);
/* IslDist::cv (src/workload.cpp:24-36). */
int dwdp_isl_cv(const dwdp_workload_spec* spec, double* cv);

/* ======================================================================
 * Cost model — include/dwdpsim/modelspec.hpp:22-75, hwmodel.hpp:29-52.
 * ==================================================================== */
typedef struct { /* MoeModelSpec + CostCalibration (modelspec.hpp:13-40) */
  int32_t num_layers;
  int32_t num_experts;
  int64_t hidden_dim;
  int32_t top_k;
  int32_t reserved;
  int64_t expert_ffn_dim;
  int64_t shared_ffn_dim;
  double weight_bytes_per_param;
  double act_bytes_per_element;
  double attn_proj_params;             /* attention block (layer_costs)   */
  double kv_bytes_per_token_per_layer;
  double others_bytes_factor;          /* Others = factor x one act pass  */
  double calib_attention;              /* CostCalibration: 1.0 = neutral  */
  double calib_grouped_gemm;
  double calib_dense_gemm;
} dwdp_model_spec;

typedef struct { /* GpuSpec (hwmodel.hpp:29-38) */
  double peak_flops;
  double mem_bw;
  double link_bw;
} dwdp_gpu_spec;

#define DWDP_CAT_GROUPED_GEMM 1 /* Category (hwmodel.hpp:14-23) */
#define DWDP_CAT_DENSE_GEMM 2
#define DWDP_CAT_OTHERS 3
#define DWDP_CAT_COMMUNICATION 4
#define DWDP_CAT_D2D_COPY 5
#define DWDP_CAT_P2P_COPY 6
#define DWDP_CAT_SYNC_WAIT 7

typedef struct { /* OpCost (modelspec.hpp:37-41) + measured time */
  int32_t category;
  int32_t layer;
  double flops;
  double bytes;
  double ns;
} dwdp_op_cost;

/* Category::name (src/hwmodel.cpp:9-29); NULL for an unknown id. */
const char* dwdp_category_name(int category);
/* MoeModelSpec::validate (src/modelspec.cpp:6-23). */
int dwdp_model_validate(const dwdp_model_spec* m);
/* expert_shard_bytes (src/modelspec.cpp:32-36). */
int dwdp_expert_shard_bytes(const dwdp_model_spec* m, double* bytes);
/* attention_entries (src/modelspec.cpp:38-55): Attention (+ Others);
 * out capacity 2. */
int dwdp_attention_entries(const dwdp_model_spec* m, double tokens,
                           double mean_seq_len, dwdp_op_cost* out, int* n_out);
/* moe_entries (src/modelspec.cpp:57-86): GroupedGemm (+ DenseGemm)
 * (+ Others); out capacity 3. */
int dwdp_moe_entries(const dwdp_model_spec* m, double tokens,
                     double routed_pairs, int experts_touched,
                     dwdp_op_cost* out, int* n_out);
/* layer_costs (src/modelspec.cpp:88-98): validates the model; attn capacity
 * 2, moe capacity 3. */
int dwdp_layer_costs(const dwdp_model_spec* m, int64_t tokens,
                     int64_t mean_seq_len, dwdp_op_cost* attn, int* n_attn,
                     dwdp_op_cost* moe, int* n_moe);
/* roofline_time (src/hwmodel.cpp:68-73). */
int dwdp_roofline_time(double flops, double bytes, const dwdp_gpu_spec* g,
                       double* seconds);

typedef struct { /* AnalyticResult (simcore.hpp:218-225) */
  double t_compute_s;
  double t_prefetch_s;
  double t_all2all_s;
  double compute_prefetch_ratio;
  double dep_dwdp_speedup;
  int32_t prefetch_saturated;
  int32_t reserved;
} dwdp_analytic_result;

/* analytic_compare (src/simcore.cpp:882-905) over layer_costs. With
 * mean_seq_len == 0 the layer is the MoE block alone (the measured stack
 * without the attention block) and the model is checked on its MoE fields
 * only. */
int dwdp_analytic_compare(const dwdp_model_spec* m, const dwdp_gpu_spec* g,
                          const dwdp_placement* p, int64_t tokens,
                          int64_t mean_seq_len, dwdp_analytic_result* out);

/* ======================================================================
 * Per-GPU runtime: split-weight manager, prefetch engine, MoE forward.
 * Replaces the simulated execution of simulate_dwdp / simulate_dep
 * (include/dwdpsim/simcore.hpp:159-172, src/simcore.cpp:519-761) and the
 * cost-only moe_entries with real sm_100a kernels.
 * ==================================================================== */
#define DWDP_SCORING_SOFTMAX 0
#define DWDP_SCORING_SIGMOID 1
#define DWDP_WEIGHT_BF16 0
#define DWDP_WEIGHT_FP8 1
#define DWDP_WEIGHT_NVFP4 2 /* W4A4 NVFP4: e2m1 codes, e4m3 scales per 16
                               elements, fp32 row scales (kind::mxf4nvf4) */
#define DWDP_ENGINE_COPY 0 /* copy-engine peer copies on a side stream  */
#define DWDP_ENGINE_PULL 1 /* one-launch SM pull kernel over NVLink      */
#define DWDP_ENGINE_HYBRID 2 /* odd TDM slices on the pull kernel, even ones
                                on the copy engines, both at once          */

typedef struct {
  /* model */
  int32_t num_layers;     /* L: layers of the MoE stack                   */
  int32_t num_experts;    /* E                                            */
  int64_t hidden;         /* h (multiple of 64)                           */
  int64_t ffn;            /* f (multiple of 128)                          */
  int64_t shared_ffn;     /* fs: 0 or == f                                */
  int32_t top_k;
  int32_t scoring;        /* DWDP_SCORING_*                               */
  int32_t n_group;
  int32_t topk_group;
  int32_t norm_topk;
  float routed_scale;
  /* DWDP group */
  int32_t rank;
  int32_t group_size;     /* 1 = all experts local (no prefetch)          */
  int32_t extra_redundancy;
  int32_t device;         /* CUDA ordinal                                 */
  /* DwdpOptions (simcore.hpp:64-71) */
  int32_t merge_elim;     /* 1: GEMM reads split receive buffers in place  */
  int32_t tdm;            /* 1: sliced round-robin plan, 0: monolithic     */
  uint64_t slice_size;
  int32_t engine;         /* DWDP_ENGINE_*                                 */
  int32_t pull_ctas;      /* CTAs of the pull kernel                       */
  int32_t ce_inflight;    /* copy-engine transfers in flight per plan
                             (GpuSpec::ce_inflight, hwmodel.hpp:33)       */
  int32_t weight_dtype;   /* DWDP_WEIGHT_BF16 / DWDP_WEIGHT_FP8 (e4m3 with
                             per-output-channel fp32 scales; activations
                             quantised per row, W8A8 on tcgen05 f8f6f4)
                             or DWDP_WEIGHT_NVFP4 (W4A4, block scales)    */
  /* synthetic weights */
  uint64_t weight_seed;
  int32_t weight_layers;  /* distinct weight sets; layer l uses l % this   */
  int32_t kernel_timing;  /* 1: CUDA events between the layer's kernels    */
  int64_t max_tokens;     /* workspace sizing (tokens per forward)         */
} dwdp_ctx_config;

typedef struct dwdp_ctx dwdp_ctx;
typedef int64_t dwdp_prefetch; /* plan handle (CopyEngineSim plan id)     */

int dwdp_ctx_create(const dwdp_ctx_config* cfg, dwdp_ctx** out);
int dwdp_ctx_destroy(dwdp_ctx* ctx);
/* Device bytes the context holds (weights + receive buffers + workspace). */
int dwdp_ctx_memory(const dwdp_ctx* ctx, uint64_t* weight_bytes,
                    uint64_t* recv_bytes, uint64_t* workspace_bytes);

/* Multi-process peer wiring (one process per GPU): export this rank's
 * weight-arena IPC handles, then hand every rank's blob to every rank. */
#define DWDP_IPC_BLOB_BYTES 1024
int dwdp_ctx_export_ipc(dwdp_ctx* ctx, void* blob /*DWDP_IPC_BLOB_BYTES*/);
int dwdp_ctx_open_peers(dwdp_ctx* ctx, const void* blobs /*N x BLOB*/);
/* Single-process alternative: share arenas of contexts on other devices. */
int dwdp_ctx_link_local(dwdp_ctx* const* ctxs, int n);

/* Deterministic counter-hash init of the owned experts, shared expert,
 * router (and e_score_correction_bias = bias_scale * U(-1,1)); then stages
 * layer 0 (simcore.cpp:640-645, "layer 0 preloaded"). Synchronous. */
int dwdp_ctx_init_weights(dwdp_ctx* ctx, float bias_scale);
/* Overwrite the per-expert selection bias of every layer (e.g. a Zipf
 * popularity tilt); host array [E] fp32. */
int dwdp_ctx_set_bias(dwdp_ctx* ctx, const float* bias);
/* Copy expert `e` tensor t (0 gate, 1 up, 2 down; e == E: shared) of
 * layer `layer` as currently resident for that layer into host memory
 * (raw storage: bf16, or e4m3 bytes for fp8). For fp8, t = 3, 4, 5 read the
 * fp32 per-row scales of gate, up, down. For nvfp4, t = 0-2 read packed
 * e2m1 codes (rows x K/2 bytes), t = 3-5 the row scales and t = 6-8 the
 * e4m3 block scales in the GEMM's 512-byte atom layout. */
int dwdp_ctx_read_expert(dwdp_ctx* ctx, int layer, int expert, int t,
                         void* host_bf16);

/* ---- prefetch handles: CopyEngineSim (simcore.hpp:87-151) -------------
 * issue_plan(dst, transfers, now) -> handle: enqueue the copy plan that
 * pulls every non-local expert of global layer g into receive buffer
 * g % 2, after the MoE of global layer g-1 released it (event-only
 * ordering, never blocks the host, no collective). */
int dwdp_prefetch_issue(dwdp_ctx* ctx, int64_t global_layer, dwdp_prefetch* h);
/* plan_done */
int dwdp_prefetch_query(dwdp_ctx* ctx, dwdp_prefetch h, int* done);
/* MoeGate: make `stream` wait for the plan (cudaStreamWaitEvent). */
int dwdp_prefetch_wait(dwdp_ctx* ctx, dwdp_prefetch h, void* stream);
/* plan_start_time / plan_complete_time / plan_bytes, ns relative to the
 * context's epoch event; -1 while pending. */
int dwdp_prefetch_times(dwdp_ctx* ctx, dwdp_prefetch h, int64_t* start_ns,
                        int64_t* end_ns, double* bytes);
/* Switch the prefetch engine for plans issued from now on (DWDP_ENGINE_*);
 * both engines are wired at peer-open time, so the choice can follow the
 * GB/s measured during warm-up. */
int dwdp_ctx_set_engine(dwdp_ctx* ctx, int engine);
/* Copy plan of this rank (dst offsets relative to per-(peer,param) buffers). */
int dwdp_ctx_copy_plan(dwdp_ctx* ctx, dwdp_slice* out, size_t* n_inout);

/* ---- MoE forward -------------------------------------------------------
 * moe_entries (src/modelspec.cpp:57-86) made real: router + top-k, permute,
 * grouped GEMM1 + SwiGLU, grouped GEMM2, weighted combine (+ shared expert).
 * x, y: device bf16 [T][h]. Weights of `layer` must be resident. */
int dwdp_moe_forward(dwdp_ctx* ctx, int layer, const void* x, int64_t T,
                     void* y, void* stream);
/* One DWDP layer (simcore.cpp:676-710): MoeGate(g) = wait plan(g) and time
 * the weight wait, issue plan(g+1), then the MoE of layer g % L. If
 * `residual`, y = x + MoE(x). */
int dwdp_layer_forward(dwdp_ctx* ctx, int64_t global_layer, const void* x,
                       int64_t T, void* y, int residual, void* stream);
/* L consecutive layers from the context's global layer cursor (one
 * iteration of the stack); x and y may alias. */
int dwdp_stack_forward(dwdp_ctx* ctx, const void* x, int64_t T, void* y,
                       void* stream);
/* Router + permutation only, for parity: idx/wts [T][k] (device),
 * counts [E] and row_of [T][k] (device int32); *rows = padded rows. */
int dwdp_route(dwdp_ctx* ctx, int layer, const void* x, int64_t T, void* idx,
               void* wts, void* counts, void* row_of, int64_t* rows,
               void* stream);

/* ---- accounting: SimEvent / RunReport (simcore.hpp:29-61) --------------
 * Per global layer measured after the fact from CUDA events. */
typedef struct {
  int64_t global_layer;
  int64_t tokens;
  double gate_wait_ns;   /* SyncWait "weight_wait": exposed prefetch  */
  double moe_ns;         /* GroupedGemm+DenseGemm+Others of the layer */
  double prefetch_ns;    /* P2PCopy of this layer's plan              */
  double prefetch_bytes;
  double merge_ns;       /* D2DCopy (merge_elim == 0 only)            */
  /* per-kernel split of moe_ns (kernel_timing == 1, else 0):         */
  double router_ns;      /* router logits + scoring/top-k             */
  double permute_ns;     /* count/scan/scatter+gather                 */
  double gemm1_ns;       /* grouped GEMM gate/up + SwiGLU             */
  double gemm2_ns;       /* grouped GEMM down                         */
  double combine_ns;     /* weighted combine (+ shared, residual)     */
  int64_t routed_rows;   /* padded expert-major rows of the layer     */
  double comm_ns;        /* DEP: dispatch + combine all-to-alls (incl.
                            the waits for the slowest rank)            */
  double dispatch_ns;    /* DEP: the dispatch part of comm_ns          */
  /* absolute times on the context's clock (ns since its creation): */
  double start_ns;       /* MoeGate entry (before the weight wait)     */
  double end_ns;         /* end of the layer's last kernel             */
  double prefetch_start_ns, prefetch_end_ns; /* this layer's plan, -1 if none */
} dwdp_layer_record;
/* Drain completed layer records (synchronises the context's streams). */
int dwdp_ctx_records(dwdp_ctx* ctx, dwdp_layer_record* out, size_t* n_inout);

/* ---- RunReport / breakdown / compare_reports (simcore.hpp:29-61, 177-213;
 * simcore.cpp:18-63, 766-876) over measured events. Categories keep the
 * reference's Category order (hwmodel.hpp:14-23). */
#define DWDP_CAT_ATTENTION 0
#define DWDP_CAT_GROUPED_GEMM 1
#define DWDP_CAT_DENSE_GEMM 2
#define DWDP_CAT_OTHERS 3
#define DWDP_CAT_COMMUNICATION 4
#define DWDP_CAT_D2D_COPY 5
#define DWDP_CAT_P2P_COPY 6
#define DWDP_CAT_SYNC_WAIT 7
#define DWDP_NUM_CATEGORIES 8
/* SimEvent::detail strings as codes */
#define DWDP_DETAIL_NONE 0
#define DWDP_DETAIL_WEIGHT_WAIT 1
#define DWDP_DETAIL_DISPATCH 2
#define DWDP_DETAIL_COMBINE 3
#define DWDP_DETAIL_BARRIER 4
typedef struct {
  int32_t rank;
  int32_t stream;   /* 0 compute, 1 copy engine (Stream) */
  int32_t category; /* DWDP_CAT_* */
  int32_t layer;
  int32_t iteration;
  int32_t detail;   /* DWDP_DETAIL_* */
  int64_t start_ns, end_ns;
  double bytes;
} dwdp_sim_event;
typedef struct {
  double compute_us[DWDP_NUM_CATEGORIES]; /* mean us per rank and steady iteration */
  double copy_us[DWDP_NUM_CATEGORIES];
  int32_t compute_present[DWDP_NUM_CATEGORIES]; /* category has an entry (map key) */
  int32_t copy_present[DWDP_NUM_CATEGORIES];
  double iteration_latency_us;
  int32_t p2p_fully_overlapped;
  int32_t reserved;
  double tokens_per_s; /* RunReport::throughput_tokens_per_s */
} dwdp_breakdown;
typedef struct {
  double a_us[DWDP_NUM_CATEGORIES], b_us[DWDP_NUM_CATEGORIES];
  double delta_frac[DWDP_NUM_CATEGORIES]; /* (a - b) / a_latency */
  int32_t has_delta[DWDP_NUM_CATEGORIES]; /* 0 for P2PCopy (off the critical path) */
  double a_latency_us, b_latency_us, overall_frac, gross_sync_comm_pct;
} dwdp_comparison;
/* breakdown(RunReport) over an explicit event list; iter_* are
 * [num_ranks][iterations] row-major. Validates per-(rank, stream) overlap. */
int dwdp_report_breakdown(const dwdp_sim_event* events, size_t n, int num_ranks,
                          int iterations, int warmup_iterations,
                          const int64_t* iter_start, const int64_t* iter_end,
                          const int64_t* iter_tokens, dwdp_breakdown* out);
/* Measured run: per-rank layer records (whole iterations of num_layers
 * layers, as drained by dwdp_ctx_records) -> events -> breakdown. recs is
 * the concatenation of the ranks' records, counts[r] records each. If
 * events != NULL, up to *n_events events are written (total in *n_events). */
int dwdp_report_from_records(const dwdp_layer_record* recs, const size_t* counts,
                             int num_ranks, int num_layers, int warmup_iterations,
                             dwdp_breakdown* out, dwdp_sim_event* events,
                             size_t* n_events);
int dwdp_compare_reports(const dwdp_breakdown* a, const dwdp_breakdown* b,
                         dwdp_comparison* out);
/* BreakdownTable::to_csv / ComparisonTable::to_csv; *len_inout = capacity in,
 * bytes needed (incl. NUL) out. */
int dwdp_breakdown_csv(const dwdp_breakdown* b, char* buf, size_t* len_inout);
int dwdp_comparison_csv(const dwdp_comparison* c, char* buf, size_t* len_inout);
/* Kernels launched by this context so far (for the bench's launch count). */
int dwdp_ctx_launch_count(const dwdp_ctx* ctx, int64_t* n);

/* ---- DEP baseline: simulate_dep (simcore.hpp:152-157, simcore.cpp:346-478)
 * made real: the same kernels with the dispatch and combine all-to-alls
 * (NCCL grouped send/recv after a counts all-gather). Requires
 * group_size | num_experts (contiguous EP blocks == the DWDP placement). */
#define DWDP_NCCL_ID_BYTES 128
int dwdp_nccl_unique_id(void* id /*DWDP_NCCL_ID_BYTES*/);
int dwdp_dep_init(dwdp_ctx* ctx, const void* nccl_id);
/* DEP variant: 0 (default) = the reference's semantics, every (token,
 * expert) pair's row sent to the expert's rank (simcore.cpp:321-324) with
 * per-expert counts exchanged per layer; 1 = token-deduplicated dispatch
 * (each token row once per peer rank, with its routing), receive-side
 * permute merging each expert's rows across sources, per-rank partial
 * combine so one row per (token, rank) returns, token counts exchanged once
 * per stack; 2 = each token row only to the ranks owning one of its experts
 * (own rank first), row counts exchanged per layer. Quantised experts (fp8,
 * nvfp4): modes 1 and 2 send the rows quantised once by the sender (codes +
 * scales). Modes 1 and 2 are within bf16 rounding of mode 0 (the per-rank
 * partial sums are rounded to bf16 before the final sum). */
int dwdp_dep_set_mode(dwdp_ctx* ctx, int mode);
int dwdp_dep_layer_forward(dwdp_ctx* ctx, int layer, const void* x, int64_t T,
                           void* y, int residual, void* stream);
int dwdp_dep_stack_forward(dwdp_ctx* ctx, const void* x, int64_t T, void* y,
                           void* stream);

/* ---- MLA attention block of the prefetch window -----------------------
 * The paper's window is MoE(l) + Attention(l+1); the
 * reference costs the attention block as attention_entries
 * (src/modelspec.cpp:38-55). DeepSeek-V3 MLA prefill on sm_100a kernels:
 * the five projections on the tcgen05 GEMM, RMSNorm / RoPE / K-V assembly,
 * and a tcgen05 causal flash-attention core (qk 128 nope + 64 rope, v 128).
 * Weights are caller-owned device bf16 [out][in]; wkv_a has its
 * kv_lora + rope rows zero-padded to a multiple of 256. x, y: [T][hidden];
 * seq_lens: host array of n_seqs back-to-back sequence lengths summing to T
 * (RoPE positions and the causal mask restart per sequence). */
typedef struct {
  int32_t hidden, heads, q_lora, kv_lora, nope, rope, v_dim, device;
  int64_t max_tokens;
  float rope_theta, softmax_scale;
} dwdp_mla_config;
typedef struct {
  const void *wq_a, *wq_b, *wkv_a, *wkv_b, *wo;
} dwdp_mla_weights;
typedef struct dwdp_mla dwdp_mla;
int dwdp_mla_create(const dwdp_mla_config* cfg, dwdp_mla** out);
int dwdp_mla_destroy(dwdp_mla* m);
int dwdp_mla_forward(dwdp_mla* m, const dwdp_mla_weights* w, const void* x, int64_t T,
                     const int64_t* seq_lens, int n_seqs, void* y, void* stream);
int dwdp_mla_launch_count(const dwdp_mla* m, int64_t* n);

/* ---- kernel-level entry points (tests / microbenchmarks) --------------- */
/* D[M][N] = A[M][K] . B[N][K]^T, bf16 in, fp32 accumulate, bf16 out, on the
 * tcgen05 grouped-GEMM kernel with one group. */
int dwdp_gemm_bf16(const void* A, const void* B, void* D, int64_t M, int64_t N,
                   int64_t K, void* stream);
/* NVFP4 quantisation of `rows` bf16 rows of length K (K % 256 == 0):
 * codes [rows][K/2] (element 2i in the low nibble), e4m3 block scales in
 * the 512-byte atom layout (ceil(rows/128)*128*K/16 bytes) and fp32 row
 * scales -- the activation recipe of the nvfp4 MoE path. */
int dwdp_quant_nvfp4(const void* src, int64_t rows, int64_t K, void* codes,
                     void* sf, float* row_scale, void* stream);
/* D[M][N] = (A . B^T) * sa[m] * sb[n] over NVFP4 operands as produced by
 * dwdp_quant_nvfp4 (N % 256 == 0), bf16 out, on the kind::mxf4nvf4 grouped
 * GEMM with one group. */
int dwdp_gemm_nvfp4(const void* A, const void* A_sf, const float* A_scale,
                    const void* B, const void* B_sf, const float* B_scale,
                    void* D, int64_t M, int64_t N, int64_t K, void* stream);
/* Fill a device bf16 buffer with the counter hash (oracle_fill_bf16). */
int dwdp_fill_bf16(void* dst, int64_t n, uint64_t seed, float scale,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DWDP_H */
