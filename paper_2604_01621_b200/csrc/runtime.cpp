// Per-GPU DWDP runtime. Reference semantics (paths under /root/reference/proj):
//   split-weight placement  — north-star item 1; experts of placement.cpp:75-111
//   prefetch engine/handles — CopyEngineSim, simcore.cpp:72-283 / simcore.hpp:87-151
//   per-rank layer loop     — simulate_dwdp MoeGate/MoeOps, simcore.cpp:640-733
//   static transfer list    — prefetch_transfers, simcore.cpp:486-515
#include <mutex>

#include "runtime.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>

#include "gemm_sm100.hpp"

namespace dwdp {

namespace {
constexpr uint32_t kIpcMagic = 0x44574450;  // "DWDP"
struct IpcBlob {
  uint32_t magic;
  int32_t rank, nslots, c;
  int64_t slot_elems;
  int32_t ntens, weight_layers;
  int32_t weight_dtype, group_size;
  cudaIpcMemHandle_t h[9];
};
static_assert(sizeof(IpcBlob) <= DWDP_IPC_BLOB_BYTES, "ipc blob too large");

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DWDP_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

uint64_t tensor_seed(uint64_t base, int layer, int expert, int t) {
  return Rng::mix(Rng::mix(base, 0x1000ULL + uint64_t(layer)), uint64_t(expert) * 8ULL + uint64_t(t));
}
}  // namespace

// ===================================================================== //
// construction

Ctx::Ctx(const dwdp_ctx_config& c) : cfg(c) {
  E_ = c.num_experts;
  k_ = c.top_k;
  L_ = c.num_layers;
  WL_ = c.weight_layers > 0 ? std::min(c.weight_layers, c.num_layers) : c.num_layers;
  N_ = c.group_size;
  rank_ = c.rank;
  h_ = c.hidden;
  f_ = c.ffn;
  shared_ = c.shared_ffn > 0;
  require(c.weight_dtype == DWDP_WEIGHT_BF16 || c.weight_dtype == DWDP_WEIGHT_FP8 ||
              c.weight_dtype == DWDP_WEIGHT_NVFP4,
          "ctx: unknown weight_dtype");
  fp8_ = c.weight_dtype == DWDP_WEIGHT_FP8;
  fp4_ = c.weight_dtype == DWDP_WEIGHT_NVFP4;
  esz_ = fp8_ || fp4_ ? 1 : 2;
  // GEMM1 runs on the 1-SM kernel by default. With GEMM1 on the CTA-pair
  // kernel too (cta_group::2, 256-row segments; DWDP_GEMM_PAIR=1) each GEMM
  // is 2-10% faster per SM clock, but on the power-capped B200 it drew the
  // clock down from ~1.3 to ~0.94 GHz and the full step measured 9% slower
  // on the same box (scripts/gpu/r1/r1_ab_pair.sh: 144K vs 158K tokens/s).
  {
    const char* env = std::getenv("DWDP_GEMM_PAIR");
    // DWDP_GEMM_PAIR=1: every GEMM on CTA pairs; =2: GEMM1 only; =3: GEMM2
    // and the router GEMM only (GEMM1 on the 1-SM kernel, 256-row segments);
    // unset or 0: every GEMM on the 1-SM kernel. =3 cut GEMM2 from 17.0 to
    // 13.3 ms per layer (half the B bytes per CTA; the 1-SM GEMM2 is L2-feed
    // bound at 73% tensor-pipe active) but the step moved +1.3/+3.9% on one
    // box and -3.3/-2.2% on another, where the SM clock fell from 1.24 to
    // 1.0 GHz under sw_power_cap (scripts/gpu/r1/r1_ab_pair3.sh,
    // r1_pair3_confirm.sh), so it stays opt-in.
    gemm1_pair_ = env && (env[0] == '1' || env[0] == '2') ? 1 : 0;
    gemm2_pair_ = env && (env[0] == '1' || env[0] == '3') ? 1 : 0;
    gemm_pair_ = gemm1_pair_ || gemm2_pair_;
    row_align_ = gemm_pair_ ? 256 : 128;
    // =4: split layout -- GEMM1 keeps the 1-SM kernel and 128-row segments,
    // its epilogue writes H into 256-row segments and GEMM2 alone runs on CTA
    // pairs (bf16 experts)
    split2_ = env && env[0] == '4' && !fp8_ && !fp4_;
    const char* r = std::getenv("DWDP_RASTER");  // experiments: m / n (default auto)
    raster_ = r ? (r[0] == 'm' ? 1 : r[0] == 'n' ? 2 : 0) : 0;
    const char* g = std::getenv("DWDP_GATHER");  // GEMM1 gathers routed rows from x
    gather_ = g && g[0] == '1';
    // NVFP4 GEMM1 on CTA pairs: 38 instead of 54 KB of L2->SM traffic per
    // k-block (the 1-SM fp4 kernel is L2-bandwidth bound): 9.45 -> 7.93 ms
    // per layer. GEMM2 (K = 2048, drain-bound) stays on the 1-SM kernel,
    // where the pair measured 6.04 -> 7.95 ms. DWDP_FP4_PAIR=0 disables.
    const char* f4 = std::getenv("DWDP_FP4_PAIR");
    fp4_pair_ = fp4_ && (f4 ? f4[0] == '1' : true) ? 1 : 0;
    const char* f42 = std::getenv("DWDP_FP4_PAIR2");
    fp4_pair2_ = fp4_pair_ && f42 && f42[0] == '1' ? 1 : 0;
    if (fp4_pair_) row_align_ = 256;
  }
  ntens_ = fp4_ ? 9 : fp8_ ? 6 : 3;
  require(L_ >= 1, "ctx: num_layers must be >= 1");
  require(E_ >= 1 && E_ <= 512, "ctx: num_experts must be in [1, 512]");
  require(k_ >= 1 && k_ <= 16 && k_ <= E_, "ctx: top_k must be in [1, min(16, E)]");
  require(h_ > 0 && h_ % 256 == 0, "ctx: hidden must be a positive multiple of 256");
  require(!fp4_ || f_ % 256 == 0, "ctx: nvfp4 needs ffn to be a multiple of 256");
  require(f_ > 0 && f_ % 128 == 0, "ctx: ffn must be a positive multiple of 128");
  require(c.shared_ffn == 0 || c.shared_ffn == c.ffn, "ctx: shared_ffn must be 0 or == ffn");
  require(c.scoring == 0 || c.scoring == 1, "ctx: unknown scoring");
  const int G = c.n_group > 0 ? c.n_group : 1;
  require(G <= 32 && E_ % G == 0, "ctx: n_group must divide E and be <= 32");
  require(c.topk_group >= 1 && c.topk_group <= G, "ctx: topk_group must be in [1, n_group]");
  require(N_ >= 1, "ctx: group_size must be >= 1");
  require(rank_ >= 0 && rank_ < N_, "ctx: rank out of range");
  require(c.max_tokens >= 1, "ctx: max_tokens must be >= 1");
  require(c.engine == DWDP_ENGINE_COPY || c.engine == DWDP_ENGINE_PULL || c.engine == DWDP_ENGINE_HYBRID,
          "ctx: unknown engine");
  require(!c.tdm || c.slice_size > 0, "dwdp.slice_size must be > 0 with tdm");
  require(!c.tdm || c.slice_size % 16 == 0, "dwdp.slice_size must be a multiple of 16 bytes");
  DeviceGuard dg(c.device);
  int cc = 0;
  cudaDeviceProp prop;
  DWDP_CUDA(cudaGetDeviceProperties(&prop, c.device));
  cc = prop.major * 10 + prop.minor;
  if (cc < 100 || cc >= 110)
    throw CudaError("dwdp: device " + std::to_string(c.device) + " is sm_" + std::to_string(cc) +
                    "; this build targets sm_100a only");
  num_sms_ = prop.multiProcessorCount;
  configure_max_shared_carveout_kernels(N_ > 1 && c.engine != DWDP_ENGINE_COPY);
  if (N_ >= 2) pl_ = build_placement(E_, N_, c.extra_redundancy);
  build_layout();

  // ---- arenas (one allocation per tensor kind so each is an IPC object)
  slot_elems_ = f_ * h_;
  for (int t = 0; t < 3; ++t)
    arena_[t] = static_cast<uint16_t*>(dalloc(tsb(t) * uint64_t(nslots_), nullptr));
  if (fp8_ || fp4_)
    for (int t = 0; t < 3; ++t)
      sarena_[t] = static_cast<float*>(dalloc(tsb(3 + t) * uint64_t(nslots_), nullptr));
  if (fp4_)
    for (int t = 0; t < 3; ++t)
      sfarena_[t] = static_cast<uint8_t*>(dalloc(tsb(6 + t) * uint64_t(nslots_), nullptr));
  for (int t = 0; t < ntens_; ++t) {
    weight_bytes += tsb(t) * uint64_t(recv_base_);
    recv_bytes += tsb(t) * uint64_t(nslots_ - recv_base_);
  }
  router_w_ = static_cast<uint16_t*>(dalloc(size_t(WL_) * E_ * h_ * 2, &weight_bytes));
  bias_ = static_cast<float*>(dalloc(size_t(WL_) * E_ * 4, &weight_bytes));
  DWDP_CUDA(cudaMemset(bias_, 0, size_t(WL_) * E_ * 4));

  // ---- slot tables [L][2][E+1]
  std::vector<int32_t> tab(size_t(L_) * 2 * (E_ + 1));
  for (int l = 0; l < L_; ++l)
    for (int p = 0; p < 2; ++p)
      for (int e = 0; e <= E_; ++e) tab[(size_t(l) * 2 + p) * (E_ + 1) + e] = slot_of(l, p, e);
  slot_tab_ = static_cast<int32_t*>(dalloc(tab.size() * 4, &workspace_bytes));
  DWDP_CUDA(cudaMemcpy(slot_tab_, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));

  // ---- workspace sized for max_tokens
  max_tokens_ = c.max_tokens;
  max_mb_ = mb_bound(max_tokens_);
  max_rows_ = max_mb_ * 128;
  logits_ = static_cast<float*>(dalloc(size_t(max_tokens_) * E_ * 4, &workspace_bytes));
  idx_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * k_ * 4, &workspace_bytes));
  wts_ = static_cast<float*>(dalloc(size_t(max_tokens_) * k_ * 4, &workspace_bytes));
  row_of_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * k_ * 4, &workspace_bytes));
  counts_ = static_cast<int32_t*>(dalloc(size_t(E_) * 4, &workspace_bytes));
  mblock_ = static_cast<int32_t*>(dalloc(size_t(max_mb_) * 4, &workspace_bytes));
  mbseg_ = static_cast<int2*>(dalloc(size_t(max_mb_) * sizeof(int2), &workspace_bytes));
  mbrows_ = static_cast<int32_t*>(dalloc(size_t(max_mb_) * 4, &workspace_bytes));
  srcrow_ = static_cast<int32_t*>(dalloc(size_t(max_rows_) * 4, &workspace_bytes));
  meta_ = static_cast<int32_t*>(dalloc(16 * 4, &workspace_bytes));
  scratch_ = static_cast<int32_t*>(
      dalloc(size_t(permute_scratch_ints(max_tokens_, E_)) * 4, &workspace_bytes));
  xperm_ = static_cast<uint16_t*>(dalloc(size_t(max_rows_) * h_ * 2, &workspace_bytes));
  int64_t h_rows = max_rows_;
  if (split2_) {
    max_mb2_ = mb_bound256(max_tokens_);
    h_rows = std::max(h_rows, max_mb2_ * 128);
    mblock2_ = static_cast<int32_t*>(dalloc(size_t(max_mb2_) * 4, &workspace_bytes));
    mbseg2_ = static_cast<int2*>(dalloc(size_t(max_mb2_) * sizeof(int2), &workspace_bytes));
    mbrows2_ = static_cast<int32_t*>(dalloc(size_t(max_mb2_) * 4, &workspace_bytes));
    d2_ = static_cast<int32_t*>(dalloc(size_t(max_mb2_) * 4, &workspace_bytes));
    d1_ = static_cast<int32_t*>(dalloc(size_t(max_mb_) * 4, &workspace_bytes));
    meta2_ = static_cast<int32_t*>(dalloc(16 * 4, &workspace_bytes));
  }
  hbuf_ = static_cast<uint16_t*>(dalloc(size_t(h_rows) * f_ * 2, &workspace_bytes));
  router_wq_ = static_cast<int8_t*>(dalloc(size_t(WL_) * 3 * E_ * h_, &weight_bytes));
  router_we_ = static_cast<int32_t*>(dalloc(size_t(WL_) * E_ * 4, &weight_bytes));
  // fused router GEMM (E % 64 == 0, the contiguous-lane top-k for E = 256,
  // h % 128 == 0); DWDP_ROUTER=planes keeps the plane-product GEMM + top-k
  {
    const char* rt = std::getenv("DWDP_ROUTER");
    const int G = c.n_group > 0 ? c.n_group : 1;
    router_fused_ = !(rt && std::string(rt) == "planes") && E_ == 256 && h_ % 128 == 0 &&
                    (G == 1 || (E_ / G) % 8 == 0);
    // the fused GEMM on CTA pairs (default; DWDP_ROUTER_PAIR=0: the 1-SM kernel)
    const char* rp = std::getenv("DWDP_ROUTER_PAIR");
    router_pair_ = router_fused_ && !(rp != nullptr && std::atoi(rp) == 0);
  }
  for (int wl = 0; wl < WL_; ++wl) {
    tm_rw64_.push_back(make_tmap_i8(router_wq_ + size_t(wl) * 3 * E_ * h_, 3 * int64_t(E_), h_, 64));
    tm_rw32_.push_back(make_tmap_i8(router_wq_ + size_t(wl) * 3 * E_ * h_, 3 * int64_t(E_), h_, 32));
    tm_rw_.push_back(make_tmap_i8(router_wq_ + size_t(wl) * 3 * E_ * h_, 3 * int64_t(E_), h_, 256));
    tm_rw_p_.push_back(make_tmap_i8(router_wq_ + size_t(wl) * 3 * E_ * h_, 3 * int64_t(E_), h_, 128));
  }
  xq_ = static_cast<int8_t*>(dalloc(size_t(max_tokens_) * 3 * h_, &workspace_bytes));
  xe_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * 4, &workspace_bytes));
  if (!router_fused_)  // int32 plane products: only the unfused router needs them
    rC_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * 9 * E_ * 4, &workspace_bytes));
  rmeta_ = static_cast<int32_t*>(dalloc(16, &workspace_bytes));
  const size_t nz = size_t((3 * max_tokens_ + 127) / 128 + 8);
  zeros_ = static_cast<int32_t*>(dalloc(nz * 4, &workspace_bytes));
  DWDP_CUDA(cudaMemset(zeros_, 0, nz * 4));

  auto tmap = fp8_ || fp4_ ? make_tmap_i8 : make_tmap_bf16;  // e4m3 / e2m1 tiles use the byte map
  const int64_t kdiv = fp4_ ? 2 : 1;  // nvfp4: two elements per byte
  tm_gate_ = tmap(arena_[0], int64_t(nslots_) * f_, h_ / kdiv, 128);
  tm_up_ = tmap(arena_[1], int64_t(nslots_) * f_, h_ / kdiv, 128);
  tm_down_ = tmap(arena_[2], int64_t(nslots_) * h_, f_ / kdiv, 256);
  if (gemm_pair_ || fp4_pair_ || split2_)  // half n-block per CTA
    tm_down_p_ = tmap(arena_[2], int64_t(nslots_) * h_, f_ / kdiv, 128);
  tm_xperm_ = make_tmap_bf16(xperm_, max_rows_, h_, 128);
  tm_h_ = make_tmap_bf16(hbuf_, h_rows, f_, 128);
  if (fp8_) {
    h8_ = static_cast<uint8_t*>(dalloc(size_t(max_rows_) * f_, &workspace_bytes));
    xs_ = static_cast<float*>(dalloc(size_t(max_rows_) * 4, &workspace_bytes));
    hs_ = static_cast<float*>(dalloc(size_t(max_rows_) * 4, &workspace_bytes));
    tm_x8_ = make_tmap_i8(xperm_, max_rows_, h_, 128);  // X_perm8 reuses the xperm_ bytes
    tm_h8_ = make_tmap_i8(h8_, max_rows_, f_, 128);
  }
  if (fp4_) {
    h8_ = static_cast<uint8_t*>(dalloc(size_t(max_rows_) * f_ / 2, &workspace_bytes));
    hsf_ = static_cast<uint8_t*>(dalloc(size_t(max_rows_) * f_ / 16, &workspace_bytes));
    xsf_ = static_cast<uint8_t*>(dalloc(size_t(max_rows_) * h_ / 16, &workspace_bytes));
    sfl_ = static_cast<uint8_t*>(dalloc(size_t(max_rows_) * std::max(h_, f_) / 16, &workspace_bytes));
    xs_ = static_cast<float*>(dalloc(size_t(max_rows_) * 4, &workspace_bytes));
    hs_ = static_cast<float*>(dalloc(size_t(max_rows_) * 4, &workspace_bytes));
    tm_x8_ = make_tmap_i8(xperm_, max_rows_, h_ / 2, 128);  // X_perm4 reuses the xperm_ bytes
    tm_h8_ = make_tmap_i8(h8_, max_rows_, f_ / 2, 128);
    tm_sf_x_ = make_tmap_sf(xsf_, int64_t(max_rows_) * h_ / 16);
    tm_sf_h_ = make_tmap_sf(hsf_, int64_t(max_rows_) * f_ / 16);
    for (int t = 0; t < 3; ++t) tm_sf_w_[t] = make_tmap_sf(sfarena_[t], int64_t(tsb(6 + t)) * nslots_);
    tm_o_ = make_tmap_out(xperm_, max_rows_, h_);  // O (bf16) overwrites X_perm4
    tm_h_o_ = make_tmap_out(hbuf_, max_rows_, f_);
  }

  DWDP_CUDA(cudaStreamCreateWithFlags(&copy_st_, cudaStreamNonBlocking));
  for (int i = 1; i < std::max(1, c.ce_inflight); ++i) {
    cudaStream_t s;
    cudaEvent_t a, b;
    DWDP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DWDP_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    DWDP_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    ce_st_.push_back(s);
    ce_fork_.push_back(a);
    ce_join_.push_back(b);
  }
  DWDP_CUDA(cudaEventCreate(&epoch_));
  DWDP_CUDA(cudaEventRecord(epoch_, copy_st_));
  for (auto& ev : moe_done_) DWDP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  for (int t = 0; t < 9; ++t) peer_arena_[t].assign(size_t(N_), nullptr);
  build_copy_plan();
  DWDP_CUDA(cudaDeviceSynchronize());
}

Ctx::~Ctx() {
  DeviceGuard dg(cfg.device);
  cudaDeviceSynchronize();
  for (auto& r : recs_)
    for (cudaEvent_t e : {r.gate0, r.gate1, r.moe_end, r.merge_end, r.k[0], r.k[1], r.k[2], r.k[3],
                          r.comm[0], r.comm[1], r.comm[2], r.comm[3]})
      if (e) cudaEventDestroy(e);
  nccl_destroy(nccl_);
  for (void* b : {static_cast<void*>(dep_recv_), static_cast<void*>(dep_h_),
                  static_cast<void*>(dep_counts_all_), static_cast<void*>(dep_tab_),
                  static_cast<void*>(dep_mbrows_), static_cast<void*>(dep_h8_),
                  static_cast<void*>(dep_xs_), static_cast<void*>(dep_hs_), static_cast<void*>(dep_sfl_),
                  static_cast<void*>(dep_xsf_), static_cast<void*>(dep_hsf_)})
    if (b) cudaFree(b);
  if (dep_counts_host_) cudaFreeHost(dep_counts_host_);
  for (void* b : {static_cast<void*>(dep2_xperm_), static_cast<void*>(dep2_h_), static_cast<void*>(dep2_mblock_),
                  static_cast<void*>(dep2_mbrows_), static_cast<void*>(dep2_mbseg_), static_cast<void*>(dep2_meta_)})
    if (b) cudaFree(b);
  for (void* b : {static_cast<void*>(dep2_x_), static_cast<void*>(dep2_idx_), static_cast<void*>(dep2_loc_),
                  static_cast<void*>(dep2_rowof_), static_cast<void*>(dep2_wts_), static_cast<void*>(dep2_scratch_),
                  static_cast<void*>(dep2_rowf_), static_cast<void*>(dep2_wf_), static_cast<void*>(dep2_tok_)})
    if (b) cudaFree(b);
  if (dep2_tok_host_) cudaFreeHost(dep2_tok_host_);
  if (dep2_flag_host_) cudaFreeHost(dep2_flag_host_);
  if (dep_mbrows_host_) cudaFreeHost(dep_mbrows_host_);
  if (dep_tab_host_) cudaFreeHost(dep_tab_host_);
  for (auto& p : plans_) {
    if (p.start) cudaEventDestroy(p.start);
    if (p.done) cudaEventDestroy(p.done);
  }
  for (cudaEvent_t e : free_events_) cudaEventDestroy(e);
  if (meta_ring_) cudaFreeHost(meta_ring_);
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  for (void* b : {static_cast<void*>(mblock2_), static_cast<void*>(mbseg2_), static_cast<void*>(mbrows2_),
                  static_cast<void*>(meta2_), static_cast<void*>(d1_), static_cast<void*>(d2_)})
    if (b) cudaFree(b);
  if (ping_) cudaFree(ping_);
  void* bufs[] = {arena_[0], arena_[1], arena_[2], router_w_, bias_, slot_tab_, logits_, idx_,
                  wts_, row_of_, counts_, mblock_, meta_, scratch_, xperm_, hbuf_, pull_items_, pull_items_odd_,
                  router_wq_, router_we_, xq_, xe_, rC_, rmeta_, zeros_, mbseg_, mbrows_, dep_seg_, srcrow_,
                  sarena_[0], sarena_[1], sarena_[2], h8_, xs_, hs_, sfarena_[0], sfarena_[1],
                  sfarena_[2], xsf_, hsf_, sfl_};
  if (dep_seg_host_) cudaFreeHost(dep_seg_host_);
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& ev : moe_done_)
    if (ev) cudaEventDestroy(ev);
  if (epoch_) cudaEventDestroy(epoch_);
  if (copy_st_) cudaStreamDestroy(copy_st_);
  for (size_t i = 0; i < ce_st_.size(); ++i) {
    cudaStreamDestroy(ce_st_[i]);
    cudaEventDestroy(ce_fork_[i]);
    cudaEventDestroy(ce_join_[i]);
  }
}

void* Ctx::dalloc(size_t bytes, uint64_t* account) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  DWDP_CUDA(cudaMalloc(&p, bytes));
  if (account) *account += bytes;
  return p;
}

// Arena slot layout (per tensor kind, all three identical):
//   [0, WL*c)                  owned experts, weight layer wl at wl*c
//   [WL*c, WL*c + WL)          shared expert of each weight layer
//   [recv, recv + 2*(E-c))     DWDP receive buffers, parity g % 2
//   [merge, merge + (E-c))     merged copy (merge_elim == 0 baseline only)
void Ctx::build_layout() {
  local_index_.assign(size_t(E_), -1);
  recv_index_.assign(size_t(E_), -1);
  if (N_ >= 2) {
    c_ = pl_.local_count;
    const auto& mine = pl_.local_sets[size_t(rank_)];
    for (int i = 0; i < c_; ++i) local_index_[size_t(mine[size_t(i)])] = i;
    int j = 0;
    for (const auto& f : pl_.fetch_lists[size_t(rank_)]) recv_index_[size_t(f.first)] = j++;
    nrecv_ = E_ - c_;
  } else {
    c_ = E_;
    for (int e = 0; e < E_; ++e) local_index_[size_t(e)] = e;
    nrecv_ = 0;
  }
  shared_base_ = WL_ * c_;
  recv_base_ = shared_base_ + (shared_ ? WL_ : 0);
  merge_base_ = recv_base_ + 2 * nrecv_;
  nslots_ = merge_base_ + (cfg.merge_elim ? 0 : nrecv_);
}

int Ctx::slot_of(int layer, int parity, int e) const {
  const int wl = layer % WL_;
  if (e == E_) return shared_ ? shared_base_ + wl : 0;
  if (local_index_[size_t(e)] >= 0) return wl * c_ + local_index_[size_t(e)];
  if (!cfg.merge_elim) return merge_base_ + recv_index_[size_t(e)];
  return recv_base_ + parity * nrecv_ + recv_index_[size_t(e)];
}

// Static per-rank transfer list (prefetch_transfers, simcore.cpp:486-515):
// for each tensor, one ShardRef per (peer, contiguous run of slots); the
// reference emits one per (peer, tensor) with src_offset 0, which is the
// single-run case (every divisible placement).
void Ctx::build_copy_plan() {
  runs_.clear();
  plan_slices_.clear();
  plan_bytes_ = 0;
  if (nrecv_ == 0) return;
  std::vector<ShardRun> base;  // tensor-independent runs
  std::map<int, int> runs_per_peer;
  for (const auto& [e, src] : pl_.fetch_lists[size_t(rank_)]) {
    const auto& ls = pl_.local_sets[size_t(src)];
    const int sslot = int(std::lower_bound(ls.begin(), ls.end(), e) - ls.begin());
    const int dslot = recv_index_[size_t(e)];
    if (!base.empty() && base.back().peer == src &&
        base.back().src_slot0 + base.back().count == sslot &&
        base.back().dst_slot0 + base.back().count == dslot) {
      ++base.back().count;
    } else {
      base.push_back({src, 0, 1, sslot, dslot, uint64_t(runs_per_peer[src]++)});
    }
  }
  std::stable_sort(base.begin(), base.end(),
                   [](const ShardRun& a, const ShardRun& b) { return a.peer < b.peer; });
  std::vector<ShardRef> shards;
  uint64_t max_size = 0;
  for (int t = 0; t < ntens_; ++t)  // 3 weight tensors (+ 3 fp8 scale tensors)
    for (const auto& b : base) {
      ShardRun r = b;
      r.tensor = t;
      r.param_id = uint64_t(t) + uint64_t(ntens_) * b.param_id;  // b.param_id = run index within peer
      runs_.push_back(r);
      shards.push_back({r.peer, r.param_id, uint64_t(r.count) * tsb(t),
                        uint64_t(r.src_slot0) * tsb(t)});
      max_size = std::max(max_size, uint64_t(r.count) * tsb(t));
    }
  const uint64_t slice = cfg.tdm ? cfg.slice_size : max_size;
  plan_slices_ = dwdp::build_copy_plan(shards, slice, rank_);
  for (const auto& s : plan_slices_) plan_bytes_ += double(s.length);
}

void* Ctx::peer_src(int peer, int t, int wl, uint64_t src_offset) const {
  return static_cast<uint8_t*>(peer_arena_[t][size_t(peer)]) + uint64_t(wl) * c_ * tsb(t) +
         src_offset;
}

uint8_t* Ctx::dst_addr(int t, int parity, const ShardRun& r, uint64_t dst_offset) const {
  return tbase(t) + uint64_t(recv_base_ + parity * nrecv_ + r.dst_slot0) * tsb(t) + dst_offset;
}

// ===================================================================== //
// peers

void Ctx::export_ipc(void* out) {
  DeviceGuard dg(cfg.device);
  IpcBlob b{};
  b.magic = kIpcMagic;
  b.rank = rank_;
  b.nslots = nslots_;
  b.c = c_;
  b.slot_elems = slot_elems_;
  b.ntens = ntens_;
  b.weight_layers = WL_;
  b.weight_dtype = cfg.weight_dtype;
  b.group_size = N_;
  for (int t = 0; t < ntens_; ++t) DWDP_CUDA(cudaIpcGetMemHandle(&b.h[t], tbase(t)));
  std::memset(out, 0, DWDP_IPC_BLOB_BYTES);
  std::memcpy(out, &b, sizeof b);
}

void Ctx::open_peers(const void* blobs) {
  DeviceGuard dg(cfg.device);
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    IpcBlob b;
    std::memcpy(&b, static_cast<const uint8_t*>(blobs) + size_t(p) * DWDP_IPC_BLOB_BYTES, sizeof b);
    require(b.magic == kIpcMagic && b.rank == p, "open_peers: malformed blob");
    // peer_src() indexes the peer's owned region with this rank's geometry
    require(b.c == c_ && b.slot_elems == slot_elems_ && b.ntens == ntens_ && b.nslots == nslots_ &&
                b.weight_layers == WL_ && b.weight_dtype == cfg.weight_dtype && b.group_size == N_,
            "open_peers: peer arena geometry differs");
    for (int t = 0; t < ntens_; ++t) {
      void* ptr = nullptr;
      DWDP_CUDA(cudaIpcOpenMemHandle(&ptr, b.h[t], cudaIpcMemLazyEnablePeerAccess));
      peer_arena_[t][size_t(p)] = ptr;
      ipc_opened_.push_back(ptr);
    }
  }
  link_local({});
}

void Ctx::link_local(const std::vector<Ctx*>& all) {
  DeviceGuard dg(cfg.device);
  for (Ctx* o : all) {
    if (o == this) continue;
    if (o->cfg.device != cfg.device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(o->cfg.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DWDP_CUDA(e);
      cudaGetLastError();
    }
    for (int t = 0; t < ntens_; ++t) peer_arena_[t][size_t(o->rank_)] = o->tbase(t);
  }
  // Pull-kernel work lists for every (weight layer, parity).
  if (nrecv_ == 0) return;
  const size_t n = plan_slices_.size();
  std::vector<PullItem> items(size_t(WL_) * 2 * n);
  std::map<std::pair<int, uint64_t>, const ShardRun*> by_shard;
  for (const auto& r : runs_) by_shard[{r.peer, r.param_id}] = &r;
  for (int wl = 0; wl < WL_; ++wl)
    for (int par = 0; par < 2; ++par)
      for (size_t i = 0; i < n; ++i) {
        const Slice& s = plan_slices_[i];
        const ShardRun* r = by_shard.at({s.src_rank, s.param_id});
        if (!peer_arena_[r->tensor][size_t(r->peer)]) return;  // peers not wired yet
        items[(size_t(wl) * 2 + size_t(par)) * n + i] = {
            peer_src(r->peer, r->tensor, wl, s.src_offset), dst_addr(r->tensor, par, *r, s.dst_offset),
            s.length};
      }
  if (!pull_items_) pull_items_ = static_cast<PullItem*>(dalloc(items.size() * sizeof(PullItem), &workspace_bytes));
  DWDP_CUDA(cudaMemcpy(pull_items_, items.data(), items.size() * sizeof(PullItem), cudaMemcpyHostToDevice));
  pull_max_len_ = 0;
  for (const Slice& sl : plan_slices_) pull_max_len_ = std::max<uint64_t>(pull_max_len_, sl.length);
  // hybrid engine: the odd slices of every (weight layer, parity) list
  n_odd_ = n / 2;
  std::vector<PullItem> odd(size_t(WL_) * 2 * std::max<size_t>(n_odd_, 1));
  for (size_t lp = 0; lp < size_t(WL_) * 2; ++lp)
    for (size_t i = 0; i < n_odd_; ++i) odd[lp * n_odd_ + i] = items[lp * n + 2 * i + 1];
  if (!pull_items_odd_)
    pull_items_odd_ = static_cast<PullItem*>(dalloc(odd.size() * sizeof(PullItem), &workspace_bytes));
  DWDP_CUDA(cudaMemcpy(pull_items_odd_, odd.data(), odd.size() * sizeof(PullItem), cudaMemcpyHostToDevice));
}

// ===================================================================== //
// weights

void Ctx::init_weights(float bias_scale) {
  DeviceGuard dg(cfg.device);
  const uint64_t base = cfg.weight_seed;
  const int owned = recv_base_;  // local + shared slots
  std::vector<uint64_t> seeds(static_cast<size_t>(owned));
  uint64_t* dseeds = static_cast<uint64_t*>(dalloc(size_t(owned) * 8 + 8, nullptr));
  const float sh = 1.0f / std::sqrt(float(h_)), sf = 1.0f / std::sqrt(float(f_));
  const std::vector<int> ident = [&] {
    std::vector<int> v(static_cast<size_t>(E_));
    for (int e = 0; e < E_; ++e) v[size_t(e)] = e;
    return v;
  }();
  const std::vector<int>& mine = N_ >= 2 ? pl_.local_sets[size_t(rank_)] : ident;
  for (int t = 0; t < 3; ++t) {
    for (int wl = 0; wl < WL_; ++wl) {
      for (int i = 0; i < c_; ++i) seeds[size_t(wl * c_ + i)] = tensor_seed(base, wl, mine[size_t(i)], t);
      if (shared_) seeds[size_t(shared_base_ + wl)] = tensor_seed(base, wl, E_, t);
    }
    DWDP_CUDA(cudaMemcpy(dseeds, seeds.data(), size_t(owned) * 8, cudaMemcpyHostToDevice));
    if (fp4_)  // e2m1 codes + block scales + row scales over the same bf16 values
      launch_nvfp4_fill_rows(tbase(t), sfarena_[t], sarena_[t], dseeds, owned, int(trows(t)),
                             t == 2 ? f_ : h_, t == 2 ? sf : sh, nullptr);
    else if (fp8_)  // e4m3 rows + per-row scales over the same bf16 values
      launch_fp8_fill_rows(tbase(t), sarena_[t], dseeds, owned, int(trows(t)), t == 2 ? f_ : h_,
                           t == 2 ? sf : sh, nullptr);
    else
      launch_fill_slots(arena_[t], dseeds, owned, slot_elems_, t == 2 ? sf : sh, nullptr);
    ++launches;
    DWDP_CUDA(cudaGetLastError());
  }
  for (int wl = 0; wl < WL_; ++wl) {
    launch_fill(router_w_ + size_t(wl) * E_ * h_, int64_t(E_) * h_, tensor_seed(base, wl, E_ + 1, 0),
                sh, nullptr);
    if (bias_scale != 0.0f)
      launch_fill_f32(bias_ + size_t(wl) * E_, E_, tensor_seed(base, wl, E_ + 1, 1), bias_scale, nullptr);
    launch_router_quant(router_w_ + size_t(wl) * E_ * h_, E_, h_, router_wq_ + size_t(wl) * 3 * E_ * h_,
                        router_we_ + size_t(wl) * E_, nullptr, nullptr);
    launches += 3;
  }
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaDeviceSynchronize());
  cudaFree(dseeds);
}

void Ctx::set_bias(const float* host) {
  DeviceGuard dg(cfg.device);
  for (int wl = 0; wl < WL_; ++wl)
    DWDP_CUDA(cudaMemcpy(bias_ + size_t(wl) * E_, host, size_t(E_) * 4, cudaMemcpyHostToDevice));
}

void Ctx::read_expert(int layer, int expert, int t, void* host) {
  DeviceGuard dg(cfg.device);
  require(layer >= 0 && layer < L_ && expert >= 0 && expert <= E_ && t >= 0 && t < ntens_,
          "read_expert: index out of range");
  require(expert < E_ || shared_, "read_expert: no shared expert");
  int par = 0;
  if (expert < E_ && recv_index_[size_t(expert)] >= 0) {  // remote: a receive buffer
    par = resident_buffer(layer);
    require(par >= 0, "read_expert: the layer's remote experts are not resident");
    // the copy stream fills the buffer asynchronously: wait for its plan
    DWDP_CUDA(cudaEventSynchronize(plan_at(plan_of_g_.at(buf_owner_[par]))->done));
  }
  const int slot = slot_of(layer, par, expert);
  DWDP_CUDA(cudaMemcpy(host, tbase(t) + uint64_t(slot) * tsb(t), tsb(t), cudaMemcpyDeviceToHost));
}

// ===================================================================== //
// prefetch engine: issue_plan / plan_done / plan_*_time

cudaEvent_t Ctx::take_event() {
  if (!free_events_.empty()) {
    cudaEvent_t e = free_events_.back();
    free_events_.pop_back();
    return e;
  }
  cudaEvent_t e;
  DWDP_CUDA(cudaEventCreate(&e));
  return e;
}

int64_t Ctx::prefetch_issue(int64_t g) {
  DeviceGuard dg(cfg.device);
  if (nrecv_ == 0) return -1;  // full replication: nothing to fetch (simcore.cpp:625-628)
  require(g >= 0, "prefetch_issue: negative layer");
  invariant(plan_of_g_.count(g) == 0, "dwdp: plan double issue");
  require(g > last_issued_g_, "prefetch_issue: global layers are prefetched in increasing order");
  for (int p = 0; p < N_; ++p)
    require(p == rank_ || peer_arena_[0][size_t(p)] != nullptr, "prefetch_issue: peers not wired");
  const int par = int(g & 1), l = int(g % L_), wl = l % WL_;
  // The buffer's current owner (layer g-2 in the double-buffer protocol)
  // must have been read before it is overwritten; the copy stream then waits
  // for that read (WAR, simcore.cpp:694-696).
  require(buf_owner_[par] < 0 || buf_read_[par],
          "prefetch_issue: receive buffer " + std::to_string(par) + " still holds global layer " +
              std::to_string(buf_owner_[par]) + ", whose MoE has not been enqueued");
  if (moe_done_recorded_[par]) DWDP_CUDA(cudaStreamWaitEvent(copy_st_, moe_done_[par], 0));
  Plan pl;
  pl.g = g;
  pl.start = take_event();
  pl.done = take_event();
  pl.bytes = plan_bytes_;
  DWDP_CUDA(cudaEventRecord(pl.start, copy_st_));
  if (cfg.engine == DWDP_ENGINE_PULL) {
    require(pull_items_ != nullptr, "prefetch_issue: pull lists not built (peers not wired)");
    const size_t n = plan_slices_.size();
    launch_pull(pull_items_ + (size_t(wl) * 2 + size_t(par)) * n, int(n), pull_max_len_,
                cfg.pull_ctas > 0 ? cfg.pull_ctas : num_sms_, copy_st_);
    ++launches;
    DWDP_CUDA(cudaGetLastError());
  } else if (cfg.engine == DWDP_ENGINE_HYBRID) {
    // Both engines at once: odd slices through the pull kernel on the copy
    // stream, even slices as copy-engine copies on the side streams.
    require(pull_items_odd_ != nullptr, "prefetch_issue: pull lists not built (peers not wired)");
    require(!ce_st_.empty(), "prefetch_issue: hybrid engine needs ce_inflight >= 2");
    const size_t ns = ce_st_.size();
    for (size_t i = 0; i < ns; ++i) {
      DWDP_CUDA(cudaEventRecord(ce_fork_[i], copy_st_));
      DWDP_CUDA(cudaStreamWaitEvent(ce_st_[i], ce_fork_[i], 0));
    }
    if (n_odd_ > 0) {
      launch_pull(pull_items_odd_ + (size_t(wl) * 2 + size_t(par)) * n_odd_, int(n_odd_), pull_max_len_,
                  cfg.pull_ctas > 0 ? cfg.pull_ctas : num_sms_, copy_st_);
      ++launches;
      DWDP_CUDA(cudaGetLastError());
    }
    std::map<std::pair<int, uint64_t>, const ShardRun*> by_shard;
    for (const auto& r : runs_) by_shard[{r.peer, r.param_id}] = &r;
    for (size_t i = 0; i < plan_slices_.size(); i += 2) {
      const Slice& s = plan_slices_[i];
      const ShardRun* r = by_shard.at({s.src_rank, s.param_id});
      DWDP_CUDA(cudaMemcpyAsync(dst_addr(r->tensor, par, *r, s.dst_offset),
                                peer_src(r->peer, r->tensor, wl, s.src_offset), s.length,
                                cudaMemcpyDeviceToDevice, ce_st_[(i / 2) % ns]));
    }
    for (size_t i = 0; i < ns; ++i) {
      DWDP_CUDA(cudaEventRecord(ce_join_[i], ce_st_[i]));
      DWDP_CUDA(cudaStreamWaitEvent(copy_st_, ce_join_[i], 0));
    }
  } else {
    // ce_inflight copy streams: slice i of the TDM plan goes to stream
    // i mod ce_inflight, so consecutive slices (different peers in the plan's
    // rotation) are in flight together (CopyEngineSim admit, simcore.cpp:134-161).
    const size_t ns = ce_st_.size() + 1;
    for (size_t i = 0; i + 1 < ns; ++i) {
      DWDP_CUDA(cudaEventRecord(ce_fork_[i], copy_st_));
      DWDP_CUDA(cudaStreamWaitEvent(ce_st_[i], ce_fork_[i], 0));
    }
    std::map<std::pair<int, uint64_t>, const ShardRun*> by_shard;
    for (const auto& r : runs_) by_shard[{r.peer, r.param_id}] = &r;
    for (size_t i = 0; i < plan_slices_.size(); ++i) {
      const Slice& s = plan_slices_[i];
      const ShardRun* r = by_shard.at({s.src_rank, s.param_id});
      const cudaStream_t cs = (i % ns) == 0 ? copy_st_ : ce_st_[i % ns - 1];
      DWDP_CUDA(cudaMemcpyAsync(dst_addr(r->tensor, par, *r, s.dst_offset),
                                peer_src(r->peer, r->tensor, wl, s.src_offset), s.length,
                                cudaMemcpyDeviceToDevice, cs));
    }
    for (size_t i = 0; i + 1 < ns; ++i) {
      DWDP_CUDA(cudaEventRecord(ce_join_[i], ce_st_[i]));
      DWDP_CUDA(cudaStreamWaitEvent(copy_st_, ce_join_[i], 0));
    }
  }
  DWDP_CUDA(cudaEventRecord(pl.done, copy_st_));
  const int64_t h = plan_base_ + int64_t(plans_.size());
  plans_.push_back(pl);
  plan_of_g_[g] = h;
  buf_owner_[par] = g;
  buf_read_[par] = false;
  last_issued_g_ = g;
  retire_plans();
  return h;
}

Plan* Ctx::plan_at(int64_t h) {
  require(h >= 0 && h < plan_base_ + int64_t(plans_.size()), "prefetch: unknown handle");
  if (h < plan_base_) return nullptr;  // retired: completed, events recycled
  return &plans_[size_t(h - plan_base_)];
}

// Drop completed plans from the front that nothing can reference any more:
// no undrained record reads their times and neither receive buffer is (or
// will be) waited on through them (the two newest plans stay).
void Ctx::retire_plans() {
  while (plans_.size() > 2) {
    Plan& p = plans_.front();
    if (p.refs > 0 || p.g == buf_owner_[0] || p.g == buf_owner_[1]) break;
    const cudaError_t q = cudaEventQuery(p.done);
    if (q == cudaErrorNotReady) break;
    DWDP_CUDA(q);
    free_events_.push_back(p.start);
    free_events_.push_back(p.done);
    plan_of_g_.erase(p.g);
    plans_.pop_front();
    ++plan_base_;
  }
}

int Ctx::resident_buffer(int layer) const {
  int best = -1;
  for (int p = 0; p < 2; ++p)
    if (buf_owner_[p] >= 0 && buf_owner_[p] % L_ == layer && (best < 0 || buf_owner_[p] > buf_owner_[best]))
      best = p;
  return best;
}

bool Ctx::prefetch_done(int64_t h) {
  if (h < 0) return true;
  const Plan* p = plan_at(h);
  if (!p) return true;
  const cudaError_t e = cudaEventQuery(p->done);
  if (e == cudaErrorNotReady) return false;
  DWDP_CUDA(e);
  return true;
}

void Ctx::prefetch_wait(int64_t h, cudaStream_t st) {
  if (h < 0) return;
  const Plan* p = plan_at(h);
  if (p) DWDP_CUDA(cudaStreamWaitEvent(st, p->done, 0));
}

void Ctx::prefetch_times(int64_t h, int64_t* s, int64_t* e, double* bytes) {
  *s = *e = -1;
  *bytes = 0;
  if (h < 0) return;
  const Plan* pp = plan_at(h);
  require(pp != nullptr, "prefetch_times: plan retired (times are kept for the two newest plans "
                         "and for plans of undrained layer records)");
  const Plan& p = *pp;
  *bytes = p.bytes;
  if (!prefetch_done(h)) return;
  float ms0 = 0, ms1 = 0;
  DWDP_CUDA(cudaEventElapsedTime(&ms0, epoch_, p.start));
  DWDP_CUDA(cudaEventElapsedTime(&ms1, epoch_, p.done));
  *s = int64_t(std::llround(double(ms0) * 1e6));
  *e = int64_t(std::llround(double(ms1) * 1e6));
}

// ===================================================================== //
// MoE forward

// Exact router: digit planes of x (quant kernel), int8 tensor-core products
// against the weight planes, exact recombination + scoring + top-k.
void Ctx::route_logits(int wl, const uint16_t* x, int64_t T, cudaStream_t st) {
  launch_router_quant(x, T, h_, xq_, xe_, rmeta_, st);
  RouterCfg rc{E_, k_, cfg.scoring, cfg.n_group, cfg.topk_group, cfg.norm_topk, cfg.routed_scale};
  if (router_fused_) {
    // one GEMM over the 3 x 3 digit-plane products with the exact
    // recombination in its epilogue -> fp32 logits; top-k reads them
    const CUtensorMap tx = make_tmap_i8(xq_, 3 * T, h_, 128);
    if (router_pair_)
      launch_router_gemm_pair(tx, tm_rw32_[size_t(wl)], xe_, router_we_ + size_t(wl) * E_, logits_, T, E_, h_, st);
    else
      launch_router_gemm(tx, tm_rw64_[size_t(wl)], xe_, router_we_ + size_t(wl) * E_, logits_, T, E_, h_, st);
    launch_topk(nullptr, xe_, router_we_ + size_t(wl) * E_, bias_ + size_t(wl) * E_, logits_, idx_, wts_, T, rc,
                st);
    return;
  }
  const CUtensorMap tx = make_tmap_i8(xq_, 3 * T, h_, 128);
  GemmArgs ga{int(h_), 3 * E_, 0, -1, zeros_, zeros_, rmeta_,
              reinterpret_cast<uint16_t*>(rC_), 3 * int64_t(E_), 3 * T, 0, nullptr,
              nullptr, nullptr, nullptr, nullptr, gemm2_pair_, 0};
  const int64_t tiles = (3 * T + 127) / 128 * ((3 * E_ + 255) / 256);
  const CUtensorMap& tb = gemm2_pair_ ? tm_rw_p_[size_t(wl)] : tm_rw_[size_t(wl)];
  launch_grouped_gemm(GEMM_INT8, tx, tx, tb, tb, ga, int(std::min<int64_t>(tiles, 1 << 30)), st);
  launch_topk(rC_, xe_, router_we_ + size_t(wl) * E_, bias_ + size_t(wl) * E_, logits_, idx_, wts_,
              T, rc, st);
}

void Ctx::moe_forward(int layer, int parity, const uint16_t* x, int64_t T, uint16_t* y,
                      const uint16_t* resid, cudaStream_t st, LayerRec* rec) {
  require(layer >= 0 && layer < L_, "moe_forward: layer out of range");
  require(T >= 0 && T <= max_tokens_, "moe_forward: T exceeds max_tokens");
  if (T == 0) return;
  const bool timed = rec != nullptr && cfg.kernel_timing != 0;
  auto mark = [&](int i) {
    if (!timed) return;
    rec->k[i] = take_event();
    DWDP_CUDA(cudaEventRecord(rec->k[i], st));
  };
  const int wl = layer % WL_;
  route_logits(wl, x, T, st);
  mark(0);
  const int64_t mb_ub = mb_bound(T);
  const int32_t* stab = slot_tab_ + (size_t(layer) * 2 + size_t(parity)) * (E_ + 1);
  // CTA pairs need 256-row expert segments. Below one 128-row m-block per
  // expert on average (decode batches) the padding would double the MMA and
  // A-tile work of every expert, so such calls use 128-row segments and the
  // 1-SM kernel. (Rank-local choice: the DEP layout keeps row_align_.)
  const bool pair = gemm_pair_ && T * k_ >= int64_t(E_) * 128;
  const int align = pair ? row_align_ : 128;
  const bool pair2 = pair && gemm2_pair_;
  const CUtensorMap& tmdown = pair2 ? tm_down_p_ : tm_down_;
  if (fp4_) {
    // W4A4 NVFP4: the permute writes e2m1 copies of every routed row and of
    // the shared-expert rows (after meta[2]) with block + row scales; GEMM1
    // emits bf16 H, which is re-quantised for GEMM2. 1-SM kernel only.
    uint8_t* x4 = reinterpret_cast<uint8_t*>(xperm_);
    const bool pair4 = fp4_pair_ && T * k_ >= int64_t(E_) * 128;  // decode batches: 1-SM kernel
    const int np = launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_,
                                  nullptr, meta_, nullptr, scratch_, st, x4, xs_, pair4 ? 256 : 128, mbrows_,
                                  sfl_);
    launch_nvfp4_sf_relayout(sfl_, xsf_, max_rows_, h_, meta_, st);
    mark(1);
    GemmArgs g1{int(h_), int(f_), int(f_), E_, mblock_, stab, meta_, hbuf_, f_, INT64_MAX, 0, mbseg_,
                nullptr, xs_, sarena_[0], sarena_[1], pair4 ? 1 : 0, raster_, mbrows_, nullptr, 0,
                xsf_, sfarena_[0], sfarena_[1]};
    const CUtensorMap sf1[4] = {tm_sf_x_, tm_sf_w_[0], tm_sf_w_[1], tm_h_o_};
    launch_grouped_gemm(GEMM_SWIGLU_FP4, tm_x8_, tm_x8_, tm_gate_, tm_up_, g1,
                        int(std::min<int64_t>(mb_ub * (f_ / 128), 1 << 30)), st, sf1);
    launch_quant_rows_nvfp4(hbuf_, max_rows_, f_, meta_, h8_, sfl_, hsf_, hs_, st);
    mark(2);
    GemmArgs g2{int(f_), int(h_), int(h_), E_, mblock_, stab, meta_, xperm_, h_, INT64_MAX, 0, mbseg_,
                nullptr, hs_, sarena_[2], nullptr, pair4 && fp4_pair2_ ? 1 : 0, raster_, mbrows_, nullptr, 0,
                hsf_, sfarena_[2], nullptr};
    const CUtensorMap sf2[4] = {tm_sf_h_, tm_sf_w_[2], tm_sf_w_[2], tm_o_};
    const CUtensorMap& tmd4 = pair4 && fp4_pair2_ ? tm_down_p_ : tm_down_;
    launch_grouped_gemm(GEMM_PLAIN_FP4, tm_h8_, tm_h8_, tmd4, tmd4, g2,
                        int(std::min<int64_t>(mb_ub * (h_ / 256), 1 << 30)), st, sf2);
    mark(3);
    combine_into(xperm_, row_of_, wts_, shared_ ? xperm_ : nullptr, meta_, resid, y, T, k_, st);
    launches += 3 + np + 1 + 4 + 1;  // router 3, permute + relayout, GEMM1 + quant 2 + GEMM2, combine
  } else if (fp8_) {
    // W8A8: the permute writes e4m3 copies of every routed row and of the
    // shared-expert rows (after meta[2]) with per-row scales; GEMM1 emits
    // bf16 H, which is re-quantised per row for GEMM2.
    uint8_t* x8 = reinterpret_cast<uint8_t*>(xperm_);
    const int np = launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_,
                                  nullptr, meta_, nullptr, scratch_, st, x8, xs_, align, mbrows_);
    mark(1);
    GemmArgs g1{int(h_), int(f_), int(f_), E_, mblock_, stab, meta_, hbuf_, f_, INT64_MAX, 0, mbseg_,
                nullptr, xs_, sarena_[0], sarena_[1], pair ? gemm1_pair_ : 0, raster_, mbrows_};
    launch_grouped_gemm(GEMM_SWIGLU_FP8, tm_x8_, tm_x8_, tm_gate_, tm_up_, g1,
                        int(std::min<int64_t>(mb_ub * (f_ / 128), 1 << 30)), st);
    launch_quant_rows_fp8(hbuf_, max_rows_, f_, meta_, h8_, hs_, st);
    mark(2);
    GemmArgs g2{int(f_), int(h_), int(h_), E_, mblock_, stab, meta_, xperm_, h_, INT64_MAX, 0, mbseg_,
                nullptr, hs_, sarena_[2], nullptr, pair2 ? 1 : 0, raster_, mbrows_};
    launch_grouped_gemm(GEMM_PLAIN_FP8, tm_h8_, tm_h8_, tmdown, tmdown, g2,
                        int(std::min<int64_t>(mb_ub * (h_ / 256), 1 << 30)), st);
    mark(3);
    combine_into(xperm_, row_of_, wts_, shared_ ? xperm_ : nullptr, meta_, resid, y, T, k_, st);
    launches += 3 + np + 3 + 1;  // router 3, permute, GEMM1 + quant + GEMM2, combine
  } else {
  // gather_: GEMM1's producer gathers the routed rows from x (cp.async), the
  // permute only ranks rows and writes src_row (1-SM kernel only)
  const bool gather = gather_ && !pair;
  const int np = launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_,
                                gather ? srcrow_ : nullptr, meta_, gather ? nullptr : xperm_, scratch_, st,
                                nullptr, nullptr, align, mbrows_);
  mark(1);
  const CUtensorMap tm_x = shared_ ? make_tmap_bf16(x, T, h_, 128) : tm_xperm_;
  // Routed A rows come from the materialised expert-major copy. GEMM1 can
  // also gather them from x (GemmArgs::a_rows, DWDP_GATHER=1), saving the
  // permute's 7 GB copy, but both gathers measured ~2x slower on B200: with
  // TMA tile::gather4 42.7 GB and with cp.async 91.8 GB of HBM reads per
  // GEMM1 instead of 26 GB -- the gathered rows are not reused from L2
  // across the expert's 16 n-block tiles the way the contiguous copy is.
  // split layout: GEMM2 on CTA pairs over H in 256-row segments (only when
  // experts average >= one m-block, as for `pair`)
  const bool split = split2_ && T * k_ >= int64_t(E_) * 128;
  if (split) {
    launch_split_layout(counts_, E_, T, shared_ ? 1 : 0, mblock2_, mbseg2_, mbrows2_, meta2_, d1_, d2_, st);
    ++launches;
  }
  GemmArgs g1{int(h_), int(f_), int(f_), E_, mblock_, stab, meta_, hbuf_, f_, INT64_MAX, 1, mbseg_,
              gather ? srcrow_ : nullptr, nullptr, nullptr, nullptr, pair ? gemm1_pair_ : 0, raster_, mbrows_,
              x, h_};
  if (split) g1.d_row0 = d1_;
  launch_grouped_gemm(GEMM_SWIGLU, tm_xperm_, tm_x, tm_gate_, tm_up_, g1, int(std::min<int64_t>(mb_ub * (f_ / 128), 1 << 30)), st);
  mark(2);
  GemmArgs g2{int(f_), int(h_), int(h_), E_, mblock_, stab, meta_, xperm_, h_, INT64_MAX, 0, mbseg_,
              nullptr, nullptr, nullptr, nullptr, pair2 ? 1 : 0, raster_, mbrows_};
  int64_t mb2_ub = mb_ub;
  if (split) {
    g2.mblock_expert = mblock2_;
    g2.meta = meta2_;
    g2.mb_seg = mbseg2_;
    g2.mb_rows = mbrows2_;
    g2.d_row0 = d2_;
    g2.pair = 1;
    mb2_ub = mb_bound256(T);
  }
  launch_grouped_gemm(GEMM_PLAIN, tm_h_, tm_h_, split ? tm_down_p_ : tmdown, split ? tm_down_p_ : tmdown, g2,
                      int(std::min<int64_t>(mb2_ub * (h_ / 256), 1 << 30)), st);
  mark(3);
  combine_into(xperm_, row_of_, wts_, shared_ ? xperm_ : nullptr, meta_, resid, y, T, k_, st);
  launches += 3 + np + 2 + 1;  // router 3, permute, GEMM1, GEMM2, combine
  }
  if (timed) {
    if (!meta_ring_) DWDP_CUDA(cudaHostAlloc(&meta_ring_, kMetaRing * 4 * sizeof(int32_t), 0));
    rec->meta_slot = meta_ring_pos_;
    meta_ring_pos_ = (meta_ring_pos_ + 1) % kMetaRing;
    DWDP_CUDA(cudaMemcpyAsync(meta_ring_ + rec->meta_slot * 4, meta_, 16, cudaMemcpyDeviceToHost, st));
  }
  DWDP_CUDA(cudaGetLastError());
}

// One DWDP layer: MoeGate(g) then MoeOps(g) (simcore.cpp:676-710).
void Ctx::layer_forward(int64_t g, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                        cudaStream_t st) {
  DeviceGuard dg(cfg.device);
  require(g >= 0, "layer_forward: negative global layer");
  const int l = int(g % L_), par = int(g & 1);
  if (nrecv_ > 0) {
    // A layer runs on the experts its own plan brought in: replaying a
    // global layer whose buffer was refilled since (or one that was never
    // prefetched but lies behind the prefetch cursor) would silently compute
    // with another layer's weights.
    if (plan_of_g_.count(g) == 0)
      require(g > last_issued_g_, "layer_forward: global layer " + std::to_string(g) +
                                      " is behind the prefetch cursor (" +
                                      std::to_string(last_issued_g_) + "); global layers only advance");
    else
      require(buf_owner_[par] == g, "layer_forward: receive buffer " + std::to_string(par) +
                                        " no longer holds global layer " + std::to_string(g));
  }
  // Layers the caller skipped (g jumps past a prefetched layer, e.g. a stack
  // iteration starting at the next layer 0) are abandoned: nothing reads
  // their buffer any more, so the next plan may overwrite it. (Their data
  // stays valid until then: a later moe_forward of that layer still checks
  // the buffer's owner.)
  for (int p = 0; p < 2; ++p)
    if (buf_owner_[p] >= 0 && buf_owner_[p] < g && !buf_read_[p]) buf_read_[p] = true;
  cursor_ = std::max(cursor_, g + 1);
  LayerRec rec{g, T, take_event(), take_event(), take_event(), nullptr, -1};
  DWDP_CUDA(cudaEventRecord(rec.gate0, st));
  if (nrecv_ > 0) {
    if (plan_of_g_.count(g) == 0) prefetch_issue(g);
    rec.plan = plan_of_g_.at(g);
    prefetch_wait(rec.plan, st);  // weight_wait (simcore.cpp:684-690)
  }
  DWDP_CUDA(cudaEventRecord(rec.gate1, st));
  // Double buffering: the next layer's buffer is free once this layer's
  // weights are in use (simcore.cpp:694-696): its owner g-1 was read.
  if (nrecv_ > 0 && plan_of_g_.count(g + 1) == 0 && g + 1 > last_issued_g_) prefetch_issue(g + 1);
  if (nrecv_ > 0 && !cfg.merge_elim) {  // D2D merge baseline (simcore.cpp:700-703)
    for (int t = 0; t < ntens_; ++t)
      DWDP_CUDA(cudaMemcpyAsync(tbase(t) + uint64_t(merge_base_) * tsb(t),
                                tbase(t) + uint64_t(recv_base_ + par * nrecv_) * tsb(t),
                                uint64_t(nrecv_) * tsb(t), cudaMemcpyDeviceToDevice, st));
    rec.merge_end = take_event();
    DWDP_CUDA(cudaEventRecord(rec.merge_end, st));
  }
  moe_forward(l, par, x, T, y, residual ? x : nullptr, st, &rec);
  DWDP_CUDA(cudaEventRecord(moe_done_[par], st));
  moe_done_recorded_[par] = true;
  if (buf_owner_[par] == g) buf_read_[par] = true;
  DWDP_CUDA(cudaEventRecord(rec.moe_end, st));
  push_record(rec);
}

void Ctx::moe_forward_resident(int layer, const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st) {
  DeviceGuard dg(cfg.device);
  require(layer >= 0 && layer < L_, "moe_forward: layer out of range");
  if (nrecv_ == 0) {  // every expert local
    moe_forward(layer, 0, x, T, y, nullptr, st);
    return;
  }
  const int par = resident_buffer(layer);
  require(par >= 0, "moe_forward: the remote experts of layer " + std::to_string(layer) +
                        " are not resident; prefetch a global layer of it first "
                        "(dwdp_prefetch_issue or dwdp_layer_forward)");
  prefetch_wait(plan_of_g_.at(buf_owner_[par]), st);
  moe_forward(layer, par, x, T, y, nullptr, st);
  DWDP_CUDA(cudaEventRecord(moe_done_[par], st));
  moe_done_recorded_[par] = true;
  buf_read_[par] = true;
}

void Ctx::push_record(const LayerRec& rec) {
  if (rec.plan >= 0) {
    Plan* p = plan_at(rec.plan);
    if (p) ++p->refs;
  }
  recs_.push_back(rec);
  // Nobody draining (kernel_timing off, no accounting): keep the newest
  // kMaxRecords and recycle the rest, so state stays bounded and the pinned
  // routed-rows ring (kMetaRing slots) is never reused under a live record.
  while (recs_.size() > kMaxRecords) {
    LayerRec old = recs_.front();
    recs_.pop_front();
    DWDP_CUDA(cudaEventSynchronize(old.moe_end));
    release_record(old);
  }
}

void Ctx::release_record(const LayerRec& r) {
  for (cudaEvent_t e : {r.gate0, r.gate1, r.moe_end, r.merge_end, r.k[0], r.k[1], r.k[2], r.k[3],
                        r.comm[0], r.comm[1], r.comm[2], r.comm[3]})
    if (e) free_events_.push_back(e);
  if (r.plan >= 0) {
    Plan* p = plan_at(r.plan);
    if (p) --p->refs;
  }
  retire_plans();
}

// One iteration of the stack starts at the next global layer that is layer 0
// (global layer g = iteration * L + l, simcore.cpp:711-728).
uint16_t* Ctx::ping() {
  if (!ping_) ping_ = static_cast<uint16_t*>(dalloc(size_t(max_tokens_) * h_ * 2, &workspace_bytes));
  return ping_;
}

void Ctx::combine_into(const uint16_t* O, const int32_t* row_of, const float* wts, const uint16_t* S,
                       const int32_t* s_meta, const uint16_t* resid, uint16_t* y, int64_t T, int k,
                       cudaStream_t st) {
  if (resid == nullptr || resid != y) {
    launch_combine(O, row_of, wts, S, s_meta, resid, y, T, k, h_, st);
    return;
  }
  uint16_t* tmp = ping();  // in-place call (x == y): never read and written by one kernel
  launch_combine(O, row_of, wts, S, s_meta, resid, tmp, T, k, h_, st);
  DWDP_CUDA(cudaMemcpyAsync(y, tmp, size_t(T) * h_ * 2, cudaMemcpyDeviceToDevice, st));
}

// Layer outputs alternate between y and the ping buffer, ending in y, so no
// layer's residual input aliases its output (x == y is allowed: the first
// layer then writes the ping buffer).
void Ctx::stack_forward(const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st) {
  const int64_t g0 = (cursor_ + L_ - 1) / L_ * L_;
  uint16_t* p = ping();
  const uint16_t* in = x;
  for (int l = 0; l < L_; ++l) {
    uint16_t* out = ((L_ - 1 - l) % 2 == 0) ? y : p;
    if (in == out) out = (out == y) ? p : y;  // x == y on the first layer
    layer_forward(g0 + l, in, T, out, true, st);
    in = out;
  }
  if (in != y) DWDP_CUDA(cudaMemcpyAsync(y, in, size_t(T) * h_ * 2, cudaMemcpyDeviceToDevice, st));
}

void Ctx::route(int layer, const uint16_t* x, int64_t T, int32_t* idx, float* wts,
                int32_t* counts, int32_t* row_of, int64_t* rows, cudaStream_t st) {
  DeviceGuard dg(cfg.device);
  require(T >= 1 && T <= max_tokens_, "route: T out of range");
  const int wl = layer % WL_;
  route_logits(wl, x, T, st);
  launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_, srcrow_, meta_, nullptr,
                 scratch_, st);
  launches += 5;
  const size_t tk = size_t(T) * size_t(k_);
  if (idx) DWDP_CUDA(cudaMemcpyAsync(idx, idx_, tk * 4, cudaMemcpyDeviceToDevice, st));
  if (wts) DWDP_CUDA(cudaMemcpyAsync(wts, wts_, tk * 4, cudaMemcpyDeviceToDevice, st));
  if (counts) DWDP_CUDA(cudaMemcpyAsync(counts, counts_, size_t(E_) * 4, cudaMemcpyDeviceToDevice, st));
  if (row_of) DWDP_CUDA(cudaMemcpyAsync(row_of, row_of_, tk * 4, cudaMemcpyDeviceToDevice, st));
  int32_t meta[4];
  DWDP_CUDA(cudaMemcpyAsync(meta, meta_, 16, cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaStreamSynchronize(st));
  if (rows) *rows = meta[2];
}

size_t Ctx::drain_records(dwdp_layer_record* out, size_t cap) {
  DeviceGuard dg(cfg.device);
  size_t n = 0;
  while (!recs_.empty() && n < cap) {
    LayerRec r = recs_.front();
    recs_.pop_front();
    DWDP_CUDA(cudaEventSynchronize(r.moe_end));
    float wait = 0, moe = 0, merge = 0, pf = 0;
    DWDP_CUDA(cudaEventElapsedTime(&wait, r.gate0, r.gate1));
    DWDP_CUDA(cudaEventElapsedTime(&moe, r.merge_end ? r.merge_end : r.gate1, r.moe_end));
    if (r.merge_end) DWDP_CUDA(cudaEventElapsedTime(&merge, r.gate1, r.merge_end));
    double pbytes = 0;
    const Plan* plan = r.plan >= 0 ? plan_at(r.plan) : nullptr;  // refs > 0: never retired
    if (plan) {
      DWDP_CUDA(cudaEventSynchronize(plan->done));
      DWDP_CUDA(cudaEventElapsedTime(&pf, plan->start, plan->done));
      pbytes = plan->bytes;
    }
    auto el = [](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0;
      DWDP_CUDA(cudaEventElapsedTime(&ms, a, b));
      return double(ms) * 1e6;
    };
    double kns[5] = {0, 0, 0, 0, 0}, comm = 0;
    const cudaEvent_t begin = r.merge_end ? r.merge_end : r.gate1;
    if (r.k[0] && r.k[3] && r.comm[0] && r.comm[1] && r.comm[2] && r.comm[3]) {  // DEP mode 1 layer
      // router | dispatch | permute | GEMM1 | GEMM2 | partial combine | return | final combine
      kns[0] = el(begin, r.k[0]);
      kns[1] = el(r.comm[1], r.k[1]);
      kns[2] = el(r.k[1], r.k[2]);
      kns[3] = el(r.k[2], r.k[3]);
      kns[4] = el(r.k[3], r.comm[2]) + el(r.comm[3], r.moe_end);
      comm = el(r.k[0], r.comm[1]) + el(r.comm[2], r.comm[3]);
    } else if (r.k[0] && r.k[3] && r.comm[1] && r.comm[3]) {  // DEP layer
      kns[0] = el(begin, r.k[0]);
      kns[1] = el(r.k[0], r.k[1]);
      kns[2] = el(r.comm[1], r.k[2]);
      kns[3] = el(r.k[2], r.k[3]);
      kns[4] = el(r.comm[3], r.moe_end);
      comm = el(r.k[1], r.comm[1]) + el(r.k[3], r.comm[3]);
    } else if (r.k[0] && r.k[3]) {
      const cudaEvent_t seq[6] = {begin, r.k[0], r.k[1], r.k[2], r.k[3], r.moe_end};
      for (int i = 0; i < 5; ++i) kns[i] = el(seq[i], seq[i + 1]);
    }
    const int64_t rows = r.rows >= 0 ? r.rows : r.meta_slot >= 0 ? meta_ring_[r.meta_slot * 4 + 2] : -1;
    const double dispatch = (r.comm[0] && r.comm[1]) ? el(r.k[0], r.comm[1])
                            : (r.k[1] && r.comm[1]) ? el(r.k[1], r.comm[1]) : 0.0;
    double pf0 = -1, pf1 = -1;
    if (plan) {
      pf0 = el(epoch_, plan->start);
      pf1 = el(epoch_, plan->done);
    }
    if (out)
      out[n] = {r.g,    r.tokens, double(wait) * 1e6, double(moe) * 1e6, double(pf) * 1e6, pbytes,
                double(merge) * 1e6, kns[0], kns[1], kns[2], kns[3], kns[4], rows, comm, dispatch,
                el(epoch_, r.gate0), el(epoch_, r.moe_end), pf0, pf1};
    ++n;
    release_record(r);
  }
  return n;
}

// ===================================================================== //
// single-group GEMM for kernel tests

void Ctx::gemm_bf16(const uint16_t* A, const uint16_t* B, uint16_t* D, int64_t M, int64_t N,
                    int64_t K, cudaStream_t st) {
  DeviceGuard dg(cfg.device);
  require(M >= 1 && N % 256 == 0 && K % 64 == 0 && N > 0 && K > 0, "gemm: need N%256==0, K%64==0");
  const int64_t mb = (M + 127) / 128;
  int32_t* tabs = static_cast<int32_t*>(dalloc(size_t(mb + 8) * 4, nullptr));
  DWDP_CUDA(cudaMemsetAsync(tabs, 0, size_t(mb + 8) * 4, st));
  const int32_t meta[4] = {int32_t(mb), int32_t(mb), int32_t(mb * 128), 0};
  DWDP_CUDA(cudaMemcpyAsync(tabs + mb + 4, meta, 16, cudaMemcpyHostToDevice, st));
  const CUtensorMap ta = make_tmap_bf16(A, M, K, 128);
  const CUtensorMap tb = make_tmap_bf16(B, N, K, 256);
  GemmArgs a{int(K), int(N), int(N), 1, tabs, tabs + mb, tabs + mb + 4, D, N, M, 0, nullptr};
  launch_grouped_gemm(GEMM_PLAIN, ta, ta, tb, tb, a, int(mb * (N / 256)), st);
  ++launches;
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaStreamSynchronize(st));
  cudaFree(tabs);
}

void Ctx::gemm_nvfp4(const uint8_t* A, const uint8_t* Asf, const float* As, const uint8_t* B,
                     const uint8_t* Bsf, const float* Bs, uint16_t* D, int64_t M, int64_t N,
                     int64_t K, cudaStream_t st) {
  DeviceGuard dg(cfg.device);
  require(M >= 1 && N > 0 && N % 256 == 0 && K > 0 && K % 256 == 0, "gemm: need N%256==0, K%256==0");
  // CTA pairs take m-blocks in pairs: the odd tail block reads zero-filled A
  // rows and stores nothing (m_limit). (Test entry: DWDP_FP4_PAIR=1 selects.)
  const char* f4 = std::getenv("DWDP_FP4_PAIR");
  const int pair = f4 && f4[0] == '1' ? 1 : 0;
  const int64_t mb = pair ? (M + 255) / 256 * 2 : (M + 127) / 128;
  int32_t* tabs = static_cast<int32_t*>(dalloc(size_t(mb + 8) * 4, nullptr));
  DWDP_CUDA(cudaMemsetAsync(tabs, 0, size_t(mb + 8) * 4, st));
  const int32_t meta[4] = {int32_t(mb), int32_t(mb), int32_t(mb * 128), 0};
  DWDP_CUDA(cudaMemcpyAsync(tabs + mb + 4, meta, 16, cudaMemcpyHostToDevice, st));
  const CUtensorMap ta = make_tmap_i8(A, M, K / 2, 128);
  const CUtensorMap tb = make_tmap_i8(B, N, K / 2, pair ? 128 : 256);
  // scale maps cover whole 128-row blocks; the caller's buffers are padded to 128 rows
  const CUtensorMap sf[4] = {make_tmap_sf(Asf, (M + 127) / 128 * 128 * K / 16),
                             make_tmap_sf(Bsf, (N + 127) / 128 * 128 * K / 16),
                             make_tmap_sf(Bsf, (N + 127) / 128 * 128 * K / 16), make_tmap_out(D, M, N)};
  GemmArgs a{int(K), int(N), int(N), 1, tabs, tabs + mb, tabs + mb + 4, D, N, M, 0, nullptr,
             nullptr, As, Bs, nullptr, pair, 0, nullptr, nullptr, 0, Asf, Bsf, nullptr};
  launch_grouped_gemm(GEMM_PLAIN_FP4, ta, ta, tb, tb, a, int(mb * (N / 256)), st, sf);
  ++launches;
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaStreamSynchronize(st));
  cudaFree(tabs);
}

}  // namespace dwdp
