// Per-GPU DWDP runtime: split-weight arenas, prefetch engine, layer loop.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dwdp.h"
#include "kernels.hpp"
#include "plan.hpp"

namespace dwdp {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void nccl_unique_id(void* out);  // dep.cpp
// The C-ABI's exception -> status mapping (capi.cpp), for entry points
// defined in other translation units (mla.cpp).
int capi_guard(const std::function<void()>& f);
void nccl_destroy(void* comm);

#define DWDP_CUDA(x)                                                                         \
  do {                                                                                       \
    const cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                                   \
      throw ::dwdp::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " at " +     \
                              __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

// One fetched shard: a run of `count` consecutive expert slots of tensor
// `tensor` held by `peer` (ShardRef of the reference, simcore.cpp:500-507).
struct ShardRun {
  int peer, tensor, count;
  int src_slot0;  // first slot inside the peer's local region of a weight layer
  int dst_slot0;  // first slot inside this rank's receive region
  uint64_t param_id;
};

struct Plan {  // one issued prefetch (CopyEngineSim::Plan)
  int64_t g = -1;
  cudaEvent_t start = nullptr, done = nullptr;
  double bytes = 0;
  int refs = 0;  // undrained layer records that read this plan's times
};

struct LayerRec {
  int64_t g, tokens;
  cudaEvent_t gate0, gate1, moe_end, merge_end;
  int64_t plan;  // index into plans_ or -1
  cudaEvent_t k[4] = {nullptr, nullptr, nullptr, nullptr};  // after router/permute/gemm1/gemm2
  int meta_slot = -1;                                       // pinned copy of meta[2]
  // DEP: [0] dispatch start, [1] dispatch end, [2] return start, [3] return end
  cudaEvent_t comm[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t rows = -1;                                        // host-known routed rows (DEP)
};

class Ctx {
 public:
  explicit Ctx(const dwdp_ctx_config& cfg);
  ~Ctx();

  void export_ipc(void* blob);
  void open_peers(const void* blobs);
  void link_local(const std::vector<Ctx*>& all);
  void init_weights(float bias_scale);
  void set_bias(const float* host);
  void read_expert(int layer, int expert, int t, void* host);

  int64_t prefetch_issue(int64_t g);
  bool prefetch_done(int64_t h);
  void prefetch_wait(int64_t h, cudaStream_t st);
  void prefetch_times(int64_t h, int64_t* s, int64_t* e, double* bytes);

  void moe_forward(int layer, int parity, const uint16_t* x, int64_t T, uint16_t* y,
                   const uint16_t* resid, cudaStream_t st, LayerRec* rec = nullptr);
  // Public MoE forward of `layer` (dwdp_moe_forward): the remote experts must
  // be resident -- a receive buffer holds a prefetched global layer g with
  // g % L == layer; the stream waits for that plan and the read is recorded
  // so a later prefetch into the buffer waits for it (WAR).
  void moe_forward_resident(int layer, const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st);
  void layer_forward(int64_t g, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                     cudaStream_t st);
  void stack_forward(const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st);
  void route(int layer, const uint16_t* x, int64_t T, int32_t* idx, float* wts,
             int32_t* counts, int32_t* row_of, int64_t* rows, cudaStream_t st);
  size_t drain_records(dwdp_layer_record* out, size_t cap);
  std::vector<Slice> copy_plan() const { return plan_slices_; }

  void gemm_nvfp4(const uint8_t* A, const uint8_t* Asf, const float* As, const uint8_t* B,
                  const uint8_t* Bsf, const float* Bs, uint16_t* D, int64_t M, int64_t N, int64_t K,
                  cudaStream_t st);
  void gemm_bf16(const uint16_t* A, const uint16_t* B, uint16_t* D, int64_t M, int64_t N,
                 int64_t K, cudaStream_t st);

  // DEP baseline (dep.cpp): expert parallelism over the same contiguous
  // blocks, dispatch + combine all-to-alls over NCCL (simcore.cpp:346-478).
  void dep_init(const void* nccl_unique_id);
  void dep_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                         cudaStream_t st);
  void dep_stack_forward(const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st);
  // DEP variant (dwdp_dep_set_mode(1)): token-deduplicated dispatch (each
  // token row goes once to every peer rank, with its routing), receive-side
  // permute that merges each local expert's rows across sources (no
  // per-(source, expert) padding), per-rank partial combine, one row per
  // (token, rank) back, final sum at the source; message sizes are the ranks'
  // token counts, exchanged once per stack instead of per-expert counts per
  // layer (bf16 experts).
  int dep_mode = 0;
  void dep2_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                          cudaStream_t st, const std::vector<int64_t>& Ts);
  std::vector<int64_t> dep2_exchange_tokens(int64_t T, cudaStream_t st);
  int dep2_experts(int layer, const uint16_t* x, int64_t T, int64_t Tall, cudaStream_t st, LayerRec& rec);
  // DEP mode 2: each token row only to the ranks that own one of its experts
  void dep3_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                          cudaStream_t st);

  dwdp_ctx_config cfg;
  uint64_t weight_bytes = 0, recv_bytes = 0, workspace_bytes = 0;
  std::atomic<int64_t> launches{0};

 private:
  void* dalloc(size_t bytes, uint64_t* account);
  void build_layout();
  void build_copy_plan();
  int slot_of(int layer, int parity, int expert) const;
  void* peer_src(int peer, int t, int wl, uint64_t src_offset) const;
  uint8_t* dst_addr(int t, int parity, const ShardRun& r, uint64_t dst_offset) const;

  int E_, k_, L_, WL_, N_, rank_, c_ = 0, nrecv_ = 0;
  int64_t h_, f_;
  bool shared_;
  Placement pl_;
  std::vector<int> local_index_;  // expert -> index in local set, -1 if remote
  std::vector<int> recv_index_;   // expert -> slot in receive region, -1 if local
  // arenas: 0 gate [slots][f][h], 1 up [slots][f][h], 2 down [slots][h][f]
  // (bf16, or e4m3 bytes when fp8); fp8 adds per-row fp32 scale arenas
  // 3 gate [slots][f], 4 up [slots][f], 5 down [slots][h]. Every tensor
  // arena is one IPC object and one prefetched "param" of the copy plan.
  uint16_t* arena_[3] = {nullptr, nullptr, nullptr};
  float* sarena_[3] = {nullptr, nullptr, nullptr};
  // nvfp4 (fp4_): arenas 0-2 hold packed e2m1 codes, 3-5 fp32 row scales and
  // 6-8 the e4m3 block scales (512-byte atoms, kernels.hpp nvfp4_sf_offset)
  uint8_t* sfarena_[3] = {nullptr, nullptr, nullptr};
  bool fp8_ = false, fp4_ = false;
  int esz_ = 2, ntens_ = 3;
  int64_t slot_elems_ = 0;
  int nslots_ = 0, shared_base_ = 0, recv_base_ = 0, merge_base_ = 0;
  std::vector<void*> peer_arena_[9];   // per tensor arena, per peer rank (nullptr for self)
  uint8_t* tbase(int t) const {
    return t < 3   ? reinterpret_cast<uint8_t*>(arena_[t])
           : t < 6 ? reinterpret_cast<uint8_t*>(sarena_[t - 3])
                   : sfarena_[t - 6];
  }
  int64_t trows(int t) const { return (t % 3) == 2 ? h_ : f_; }  // rows per slot
  uint64_t tsb(int t) const {  // bytes per slot of tensor arena t
    if (t < 3) return fp4_ ? uint64_t(slot_elems_) / 2 : uint64_t(slot_elems_) * uint64_t(esz_);
    if (t < 6) return uint64_t(trows(t)) * 4;
    return uint64_t(slot_elems_) / 16;  // one e4m3 scale per 16 elements
  }
  // W8A8 activations
  uint8_t* h8_ = nullptr;               // e4m3 H [max_rows][f] (nvfp4: [max_rows][f/2])
  uint8_t *xsf_ = nullptr, *hsf_ = nullptr;  // nvfp4 block scales of X_perm4 / H4 (atoms)
  uint8_t* sfl_ = nullptr;                   // nvfp4 linear block-scale scratch [rows][h/16]
  int fp4_pair_ = 0;                         // nvfp4 GEMMs on CTA pairs (DWDP_FP4_PAIR)
  CUtensorMap tm_sf_x_, tm_sf_h_, tm_sf_w_[3];  // nvfp4 scale atoms for the CTA-pair kernel
  CUtensorMap tm_dep_sfx_, tm_dep_sfh_;
  CUtensorMap tm_o_, tm_dep_o_;                 // nvfp4 GEMM2 output maps (TMA store)
  CUtensorMap tm_h_o_, tm_dep_h_o_;             // nvfp4 GEMM1 (CTA pair) output maps
  int fp4_pair2_ = 0;                           // GEMM2 on CTA pairs too (DWDP_FP4_PAIR2)
  float *xs_ = nullptr, *hs_ = nullptr;  // per-row scales of X_perm8 / H8
  CUtensorMap tm_x8_, tm_h8_;
  std::vector<void*> ipc_opened_;
  uint16_t* router_w_ = nullptr;       // [WL][E][h]
  float* bias_ = nullptr;              // [WL][E]
  // exact int8 router: weight digit planes [WL][3][E][h] + row exponents
  int8_t* router_wq_ = nullptr;
  int32_t* router_we_ = nullptr;
  std::vector<CUtensorMap> tm_rw_, tm_rw_p_;  // router weight planes (256 / 128-row boxes)
  std::vector<CUtensorMap> tm_rw64_;          // 64-row boxes (fused router GEMM)
  std::vector<CUtensorMap> tm_rw32_;          // 32-row boxes (fused router GEMM on CTA pairs)
  bool router_pair_ = false;
  bool router_fused_ = false;
  int8_t* xq_ = nullptr;               // activation digit planes [3][T][h]
  int32_t* xe_ = nullptr;              // activation row exponents [T]
  int32_t* rC_ = nullptr;              // int32 plane products [3T][3E]
  int32_t* rmeta_ = nullptr;           // single-group GEMM table
  int32_t* zeros_ = nullptr;
  void route_logits(int wl, const uint16_t* x, int64_t T, cudaStream_t st);
  int32_t* slot_tab_ = nullptr;        // [L][2][E+1]
  // workspace
  int64_t max_tokens_ = 0, max_rows_ = 0, max_mb_ = 0;
  float* logits_ = nullptr;
  int32_t *idx_ = nullptr, *counts_ = nullptr, *row_of_ = nullptr, *mblock_ = nullptr,
          *meta_ = nullptr, *scratch_ = nullptr;
  float* wts_ = nullptr;
  int2* mbseg_ = nullptr;               // [max_mb] expert segment of each m-block
  int32_t* mbrows_ = nullptr;           // [max_mb] real rows of each m-block
  int32_t* srcrow_ = nullptr;           // [max_rows] source token of each routed row
  uint16_t *xperm_ = nullptr, *hbuf_ = nullptr;
  CUtensorMap tm_gate_, tm_up_, tm_down_, tm_xperm_, tm_h_;
  CUtensorMap tm_down_p_;          // down arena with 128-row boxes (CTA-pair GEMM2)
  int gemm_pair_ = 0;              // any GEMM on CTA pairs (256-row segments, half-n-block maps)
  int gemm1_pair_ = 0;             // GemmArgs::pair for GEMM1: 0 1-SM, 1 CTA pair
  int gemm2_pair_ = 0;             // GEMM2 and the router GEMM on CTA pairs too
  int row_align_ = 128;            // expert segment padding (256 with pairs)
  // split layout (DWDP_GEMM_PAIR=4): GEMM1 1-SM on 128-row segments, H in
  // 256-row segments, GEMM2 on CTA pairs (launch_split_layout)
  bool split2_ = false;
  int32_t *mblock2_ = nullptr, *mbrows2_ = nullptr, *meta2_ = nullptr, *d1_ = nullptr,
          *d2_ = nullptr;
  int2* mbseg2_ = nullptr;
  int64_t max_mb2_ = 0;
  int64_t mb_bound256(int64_t T) const {
    return (T * k_ + int64_t(E_) * 255) / 128 + 2 + (shared_ ? (T + 255) / 256 * 2 : 0);
  }
  int raster_ = 0;                 // GemmArgs::raster (DWDP_RASTER experiments)
  bool gather_ = false;            // GEMM1 gathers routed rows from x (DWDP_GATHER=1)
  // upper bound on the m-blocks of T tokens (routed segments + shared block)
  int64_t mb_bound(int64_t T) const {
    return (T * k_ + int64_t(E_) * (row_align_ - 1)) / 128 + 2 +
           (shared_ ? (T + row_align_ - 1) / row_align_ * (row_align_ / 128) : 0);
  }
  // prefetch engine
  std::vector<ShardRun> runs_;
  std::vector<Slice> plan_slices_;
  double plan_bytes_ = 0;
  cudaStream_t copy_st_ = nullptr;
  std::vector<cudaStream_t> ce_st_;    // extra copy streams: ce_inflight - 1
  std::vector<cudaEvent_t> ce_fork_, ce_join_;
  cudaEvent_t epoch_ = nullptr;
  cudaEvent_t moe_done_[2] = {nullptr, nullptr};
  bool moe_done_recorded_[2] = {false, false};
  // Receive-buffer ownership: buffer p holds the experts of global layer
  // buf_owner_[p] (-1: never filled); buf_read_[p] once an MoE reading them
  // is enqueued (moe_done_[p] recorded after it). A plan may only overwrite
  // a buffer whose owner has been read.
  int64_t buf_owner_[2] = {-1, -1};
  bool buf_read_[2] = {false, false};
  int64_t last_issued_g_ = -1;
  // Live plans: handle h lives at plans_[h - plan_base_]; done plans that no
  // undrained record references and that no buffer can still be waiting on
  // are retired (their events recycled), so serving loops hold O(1) state.
  std::deque<Plan> plans_;
  int64_t plan_base_ = 0;
  std::map<int64_t, int64_t> plan_of_g_;  // live global layer -> plan handle
  Plan* plan_at(int64_t h);
  void retire_plans();
  int resident_buffer(int layer) const;  // parity holding `layer`, -1 if none
  void push_record(const LayerRec& rec);
  void release_record(const LayerRec& r);
  static constexpr size_t kMaxRecords = 2048;  // undrained records kept (oldest dropped)
  PullItem* pull_items_ = nullptr;  // device [WL][2][n_slices]
  PullItem* pull_items_odd_ = nullptr;  // hybrid: device [WL][2][n_slices / 2] (odd slices)
  size_t n_odd_ = 0;
  uint64_t pull_max_len_ = 0;          // longest slice (pull-kernel chunk grid)
  int64_t cursor_ = 0;              // next global layer of stack_forward
  std::deque<LayerRec> recs_;
  std::vector<cudaEvent_t> free_events_;
  cudaEvent_t take_event();
  int32_t* meta_ring_ = nullptr;  // pinned host ring for per-layer routed rows
  int meta_ring_pos_ = 0;
  static constexpr int kMetaRing = 4096;
  // DEP state
  void* nccl_ = nullptr;                 // ncclComm_t
  uint16_t* dep_recv_ = nullptr;         // received X, then O, + shared rows
  uint16_t* dep_h_ = nullptr;            // H of the received rows
  int64_t dep_cap_rows_ = 0;
  int32_t* dep_counts_all_ = nullptr;    // device [N][E]
  int32_t* dep_counts_host_ = nullptr;   // pinned [N][E]
  int32_t* dep_tab_ = nullptr;           // device m-block table + meta
  int32_t* dep_tab_host_ = nullptr;      // pinned staging
  int2* dep_seg_ = nullptr;              // device (source, expert) segment table
  int2* dep_seg_host_ = nullptr;
  int32_t* dep_mbrows_ = nullptr;        // device real rows per m-block
  int32_t* dep_mbrows_host_ = nullptr;
  int64_t dep_tab_cap_ = 0;
  CUtensorMap tm_dep_recv_, tm_dep_h_;
  // fp8 DEP: received e4m3 rows live in dep_recv_ (bytes), their scales in
  // dep_xs_; H is re-quantised into dep_h8_ / dep_hs_
  uint8_t* dep_h8_ = nullptr;
  float *dep_xs_ = nullptr, *dep_hs_ = nullptr;
  // nvfp4 DEP: received codes in dep_recv_ (bytes), linear block scales in
  // dep_sfl_ (also the H quantiser's scratch), atoms in dep_xsf_ / dep_hsf_
  uint8_t *dep_sfl_ = nullptr, *dep_xsf_ = nullptr, *dep_hsf_ = nullptr;
  CUtensorMap tm_dep_x8_, tm_dep_h8_;
  void dep_reserve(int64_t rows);
  // layer-output ping-pong buffer [max_tokens][h] bf16: the stacks alternate
  // y / ping so a layer's residual input never aliases its output
  uint16_t* ping_ = nullptr;
  uint16_t* ping();
  // combine into y, or (when resid aliases y: in-place single-layer calls)
  // into ping and copy back
  void combine_into(const uint16_t* O, const int32_t* row_of, const float* wts, const uint16_t* S,
                    const int32_t* s_meta, const uint16_t* resid, uint16_t* y, int64_t T, int k,
                    cudaStream_t st);
  // DEP mode 1 buffers: all ranks' token rows (then the partial rows sent
  // back), their routing, local row_of, permute scratch, final-combine tables
  uint16_t* dep2_x_ = nullptr;
  int32_t *dep2_idx_ = nullptr, *dep2_loc_ = nullptr, *dep2_rowof_ = nullptr, *dep2_scratch_ = nullptr,
          *dep2_rowf_ = nullptr, *dep2_tok_ = nullptr, *dep2_flag_host_ = nullptr;
  float *dep2_wts_ = nullptr, *dep2_wf_ = nullptr;
  // receive-side expert-major rows / H / m-block tables, sized for 1.3x the
  // balanced load (routing skew across expert blocks); overflow is detected
  // on the device and raised on every rank at the next token exchange
  uint16_t *dep2_xperm_ = nullptr, *dep2_h_ = nullptr;
  int32_t *dep2_mblock_ = nullptr, *dep2_mbrows_ = nullptr, *dep2_meta_ = nullptr;
  int2* dep2_mbseg_ = nullptr;
  int64_t dep2_cap_rows_ = 0, dep2_max_mb_ = 0;
  CUtensorMap tm_dep2_xperm_, tm_dep2_h_;
  // fp8 / nvfp4 experts: e4m3 / e2m1 copies of the received rows live in the
  // dep2_xperm_ bytes (as X_perm8 in the DWDP path), H re-quantised into dep2_h8_
  uint8_t *dep2_h8_ = nullptr, *dep2_sfl_ = nullptr, *dep2_xsf_ = nullptr, *dep2_hsf_ = nullptr;
  float *dep2_xs_ = nullptr, *dep2_hs_ = nullptr;
  CUtensorMap tm_dep2_x8_, tm_dep2_h8_, tm_dep2_sfx_, tm_dep2_sfh_, tm_dep2_o_, tm_dep2_h_o_;
  // quantised rows on the wire (modes 1 and 2): the own tokens' codes, row
  // scales and linear block scales; the received rows' scales (codes in the
  // dep2_x_ bytes); mode 2's send rows' scales
  uint8_t *dq_x_ = nullptr, *dq_sfl_ = nullptr, *dq_sflr_ = nullptr, *dq_sfl_send_ = nullptr;
  float *dq_xs_ = nullptr, *dq_xsr_ = nullptr, *dq_xs_send_ = nullptr;
  int64_t qrow_bytes() const { return fp4_ ? h_ / 2 : h_; }
  void dq_quantize_own(const uint16_t* x, int64_t T, cudaStream_t st);
  int64_t* dep2_tok_host_ = nullptr;
  int64_t dep2_rowf_T_ = -1;
  void dep2_alloc();
  // DEP mode 2 send side: destination ranks [T][k+1], the permute by rank
  // (send rows in rank segments), the rows' routing, per-rank counts
  int32_t *dep3_idx2_ = nullptr, *dep3_rowof2_ = nullptr, *dep3_sidx_ = nullptr, *dep3_counts_ = nullptr,
          *dep3_counts_host_ = nullptr, *dep3_meta_ = nullptr, *dep3_scratch_ = nullptr, *dep3_mblock_ = nullptr;
  int2* dep3_mbseg_ = nullptr;
  float *dep3_swts_ = nullptr, *dep3_ones_ = nullptr;
  uint16_t* dep3_xsend_ = nullptr;
  int64_t dep3_cap_rows_ = 0;
  void dep3_alloc();
  int num_sms_ = 148;
};

}  // namespace dwdp
