// DEP baseline: "the same kernels with the two all-to-alls".
//
// Reference semantics: simulate_dep (/root/reference/proj/src/simcore.cpp:346-478):
// EP partition into contiguous expert blocks (:359-370), per layer barrier +
// dispatch all-to-all, expert-parallel MoE over the tokens routed to the
// rank's block (:401-451), barrier + combine all-to-all (:452-465).
//
// B200 realisation: router/top-k/permute on the rank's own tokens (shared
// kernels), an NCCL all-gather of the per-expert counts (the host needs the
// message sizes: DEP's inherent synchronisation point), grouped ncclSend /
// ncclRecv of the expert-sorted rows, the grouped GEMMs over the received
// rows (each (source, expert) segment padded to the GEMM row alignment, 128
// or 256 rows with CTA pairs, so the m-block ->
// expert table needs no regroup copy), the reverse all-to-all back into the
// send layout, and the weighted combine. NCCL is resolved at run time from
// the copy the process already loaded (torch), so libdwdp.so has no link
// dependency on it.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "gemm_sm100.hpp"
#include "runtime.hpp"

namespace dwdp {
namespace {

struct NcclId {
  char internal[DWDP_NCCL_ID_BYTES];
};
constexpr int kUint8 = 1, kInt32 = 2, kInt64 = 4, kFloat32 = 7, kBf16 = 9;

struct Nccl {
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* s) { return dlsym(h, s); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!n.CommInitRank || !n.Send || !n.Recv || !n.AllGather)
    throw CudaError("NCCL not available (libnccl.so.2 not loadable)");
  return n;
}

void nccl_check(int r, const char* what) {
  if (r != 0)
    throw CudaError(std::string(what) + ": " +
                    (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}


}  // namespace

void nccl_destroy(void* comm) {
  if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
}

void nccl_unique_id(void* out) {
  NcclId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

void Ctx::dep_init(const void* unique_id) {
  struct DG {
    int prev = -1;
    explicit DG(int d) {
      cudaGetDevice(&prev);
      cudaSetDevice(d);
    }
    ~DG() { cudaSetDevice(prev); }
  } dg(cfg.device);
  require(N_ >= 2, "dep: group_size must be >= 2");
  require(E_ % N_ == 0, "dep: group_size must divide num_experts");
  require(nccl_ == nullptr, "dep: already initialised");
  NcclId id;
  std::memcpy(&id, unique_id, sizeof id);
  nccl_check(nccl().CommInitRank(&nccl_, N_, id, rank_), "ncclCommInitRank");
  dep_counts_all_ = static_cast<int32_t*>(dalloc(size_t(N_) * E_ * 4, &workspace_bytes));
  DWDP_CUDA(cudaHostAlloc(&dep_counts_host_, size_t(N_) * E_ * 4, 0));
  dep_tab_cap_ = max_mb_ * 2 + 16;
  dep_tab_ = static_cast<int32_t*>(dalloc(size_t(dep_tab_cap_) * 4, &workspace_bytes));
  DWDP_CUDA(cudaHostAlloc(&dep_tab_host_, size_t(dep_tab_cap_) * 4, 0));
  dep_seg_ = static_cast<int2*>(dalloc(size_t(dep_tab_cap_) * sizeof(int2), &workspace_bytes));
  DWDP_CUDA(cudaHostAlloc(&dep_seg_host_, size_t(dep_tab_cap_) * sizeof(int2), 0));
  dep_mbrows_ = static_cast<int32_t*>(dalloc(size_t(dep_tab_cap_) * 4, &workspace_bytes));
  DWDP_CUDA(cudaHostAlloc(&dep_mbrows_host_, size_t(dep_tab_cap_) * 4, 0));
  dep_reserve(max_rows_);
}

void Ctx::dep_reserve(int64_t rows) {
  if (rows <= dep_cap_rows_) return;
  rows = rows + rows / 4;  // headroom for routing imbalance across ranks
  DWDP_CUDA(cudaDeviceSynchronize());
  if (dep_recv_) cudaFree(dep_recv_);
  if (dep_h_) cudaFree(dep_h_);
  dep_recv_ = static_cast<uint16_t*>(dalloc(size_t(rows) * h_ * 2, nullptr));
  dep_h_ = static_cast<uint16_t*>(dalloc(size_t(rows) * f_ * 2, nullptr));
  dep_cap_rows_ = rows;
  tm_dep_recv_ = make_tmap_bf16(dep_recv_, rows, h_, 128);
  tm_dep_h_ = make_tmap_bf16(dep_h_, rows, f_, 128);
  if (fp8_ || fp4_) {
    for (void* b : {static_cast<void*>(dep_h8_), static_cast<void*>(dep_xs_), static_cast<void*>(dep_hs_),
                    static_cast<void*>(dep_sfl_), static_cast<void*>(dep_xsf_), static_cast<void*>(dep_hsf_)})
      if (b) cudaFree(b);
    const int64_t kd = fp4_ ? 2 : 1;  // elements per byte
    dep_h8_ = static_cast<uint8_t*>(dalloc(size_t(rows) * f_ / kd, nullptr));
    dep_xs_ = static_cast<float*>(dalloc(size_t(rows) * 4, nullptr));
    dep_hs_ = static_cast<float*>(dalloc(size_t(rows) * 4, nullptr));
    tm_dep_x8_ = make_tmap_i8(dep_recv_, rows, h_ / kd, 128);
    tm_dep_h8_ = make_tmap_i8(dep_h8_, rows, f_ / kd, 128);
    if (fp4_) {
      dep_sfl_ = static_cast<uint8_t*>(dalloc(size_t(rows) * std::max(h_, f_) / 16, nullptr));
      dep_xsf_ = static_cast<uint8_t*>(dalloc(size_t(rows) * h_ / 16, nullptr));
      dep_hsf_ = static_cast<uint8_t*>(dalloc(size_t(rows) * f_ / 16, nullptr));
      tm_dep_sfx_ = make_tmap_sf(dep_xsf_, rows * h_ / 16);
      tm_dep_sfh_ = make_tmap_sf(dep_hsf_, rows * f_ / 16);
      tm_dep_o_ = make_tmap_out(dep_recv_, rows, h_);
      tm_dep_h_o_ = make_tmap_out(dep_h_, rows, f_);
    }
  }
  const int64_t need_tab = rows / 128 + 16;
  if (need_tab > dep_tab_cap_) {
    cudaFree(dep_tab_);
    cudaFreeHost(dep_tab_host_);
    cudaFree(dep_seg_);
    cudaFreeHost(dep_seg_host_);
    cudaFree(dep_mbrows_);
    cudaFreeHost(dep_mbrows_host_);
    dep_tab_cap_ = need_tab;
    dep_tab_ = static_cast<int32_t*>(dalloc(size_t(dep_tab_cap_) * 4, nullptr));
    DWDP_CUDA(cudaHostAlloc(&dep_tab_host_, size_t(dep_tab_cap_) * 4, 0));
    dep_seg_ = static_cast<int2*>(dalloc(size_t(dep_tab_cap_) * sizeof(int2), nullptr));
    DWDP_CUDA(cudaHostAlloc(&dep_seg_host_, size_t(dep_tab_cap_) * sizeof(int2), 0));
    dep_mbrows_ = static_cast<int32_t*>(dalloc(size_t(dep_tab_cap_) * 4, nullptr));
    DWDP_CUDA(cudaHostAlloc(&dep_mbrows_host_, size_t(dep_tab_cap_) * 4, 0));
  }
}

void Ctx::dep_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                            cudaStream_t st) {
  struct DG {
    int prev = -1;
    explicit DG(int d) {
      cudaGetDevice(&prev);
      cudaSetDevice(d);
    }
    ~DG() { cudaSetDevice(prev); }
  } dg(cfg.device);
  require(nccl_ != nullptr, "dep: call dep_init first");
  require(layer >= 0 && layer < L_, "dep: layer out of range");
  require(T >= 0 && T <= max_tokens_, "dep: T exceeds max_tokens");
  if (dep_mode == 1) {  // standalone layer: its own token-count exchange
    const auto Ts = dep2_exchange_tokens(T, st);
    dep2_layer_forward(layer, x, T, y, residual, st, Ts);
    return;
  }
  if (dep_mode == 2) {
    dep3_layer_forward(layer, x, T, y, residual, st);
    return;
  }
  const Nccl& n = nccl();
  const int wl = layer % WL_;
  const int per = E_ / N_;
  LayerRec rec{int64_t(layer), T, take_event(), take_event(), take_event(), nullptr, -1};
  DWDP_CUDA(cudaEventRecord(rec.gate0, st));
  DWDP_CUDA(cudaEventRecord(rec.gate1, st));
  auto mark = [&](cudaEvent_t* slot) {
    *slot = take_event();
    DWDP_CUDA(cudaEventRecord(*slot, st));
  };
  // 1. router + top-k + permute of the rank's own tokens (send layout)
  if (T > 0) route_logits(wl, x, T, st);
  mark(&rec.k[0]);
  // fp8: e4m3 send rows + scales, the shared-expert rows after the routed ones
  uint8_t* x8 = reinterpret_cast<uint8_t*>(xperm_);
  int np = 0;
  if (T > 0 && fp4_)  // codes + linear block scales + row scales, shared rows after the routed ones
    np = launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_, nullptr, meta_,
                        nullptr, scratch_, st, x8, xs_, row_align_, nullptr, sfl_);
  else if (T > 0 && fp8_)
    np = launch_permute(idx_, x, T, E_, k_, h_, shared_ ? 1 : 0, counts_, row_of_, mblock_, mbseg_, nullptr, meta_,
                   nullptr, scratch_, st, x8, xs_, row_align_);  // send side: padding unused
  else if (T > 0)
    np = launch_permute(idx_, x, T, E_, k_, h_, 0, counts_, row_of_, mblock_, mbseg_, nullptr, meta_, xperm_, scratch_, st,
                   nullptr, nullptr, row_align_);
  else
    DWDP_CUDA(cudaMemsetAsync(counts_, 0, size_t(E_) * 4, st));
  mark(&rec.k[1]);
  // 2. counts exchange (host needs every message size)
  nccl_check(n.AllGather(counts_, dep_counts_all_, size_t(E_), kInt32, nccl_, st), "ncclAllGather");
  DWDP_CUDA(cudaMemcpyAsync(dep_counts_host_, dep_counts_all_, size_t(N_) * E_ * 4,
                            cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaStreamSynchronize(st));
  const int32_t* ca = dep_counts_host_;
  // segments padded like the permute's send layout (256 rows with CTA pairs)
  auto padr = [&](int64_t n) { return (n + row_align_ - 1) / row_align_ * row_align_; };
  const size_t nr = static_cast<size_t>(N_);
  std::vector<int64_t> send_off(nr), send_rows(nr), recv_off(nr), recv_rows(nr);
  int64_t acc = 0;
  for (int d = 0; d < N_; ++d) {
    send_off[size_t(d)] = acc;
    int64_t r = 0;
    for (int e = d * per; e < (d + 1) * per; ++e) r += padr(ca[size_t(rank_) * E_ + e]);
    send_rows[size_t(d)] = r;
    acc += r;
  }
  acc = 0;
  int64_t nblocks = 0;
  for (int s = 0; s < N_; ++s) {
    recv_off[size_t(s)] = acc;
    int64_t r = 0;
    for (int e = rank_ * per; e < (rank_ + 1) * per; ++e) r += padr(ca[size_t(s) * E_ + e]);
    recv_rows[size_t(s)] = r;
    acc += r;
  }
  const int64_t routed_rows = acc;
  const int64_t send_total = send_off[nr - 1] + send_rows[nr - 1];
  const int64_t shared_blocks = shared_ ? padr(T) / 128 : 0;
  dep_reserve(routed_rows + shared_blocks * 128);
  // m-block -> expert over the receive layout, then the shared expert blocks
  // (each (source, expert) run of m-blocks is one raster segment)
  for (int s = 0; s < N_; ++s)
    for (int e = rank_ * per; e < (rank_ + 1) * per; ++e) {
      const int32_t cnt = ca[size_t(s) * E_ + e];
      const int2 seg = make_int2(int(nblocks), int(padr(cnt) / 128));
      for (int b = 0; b < seg.y; ++b) {
        dep_seg_host_[nblocks] = seg;
        dep_mbrows_host_[nblocks] = std::max(0, std::min(128, cnt - 128 * b));
        dep_tab_host_[4 + nblocks++] = e;
      }
    }
  const int64_t routed_mb = nblocks;
  const int2 sseg = make_int2(int(routed_mb), int(shared_blocks));
  for (int64_t b = 0; b < shared_blocks; ++b) {
    dep_seg_host_[nblocks] = sseg;
    dep_mbrows_host_[nblocks] = int32_t(std::max<int64_t>(0, std::min<int64_t>(128, T - 128 * b)));
    dep_tab_host_[4 + nblocks++] = E_;
  }
  dep_tab_host_[0] = int32_t(nblocks);
  dep_tab_host_[1] = int32_t(routed_mb);
  dep_tab_host_[2] = int32_t(routed_rows);
  dep_tab_host_[3] = int32_t(T);
  DWDP_CUDA(cudaMemcpyAsync(dep_tab_, dep_tab_host_, size_t(4 + nblocks) * 4,
                            cudaMemcpyHostToDevice, st));
  DWDP_CUDA(cudaMemcpyAsync(dep_seg_, dep_seg_host_, size_t(nblocks + 1) * sizeof(int2),
                            cudaMemcpyHostToDevice, st));
  DWDP_CUDA(cudaMemcpyAsync(dep_mbrows_, dep_mbrows_host_, size_t(nblocks + 1) * 4,
                            cudaMemcpyHostToDevice, st));
  // 3. dispatch all-to-all (bf16 rows, e4m3 rows + their fp32 scales, or
  // e2m1 codes + linear block scales + fp32 row scales)
  const size_t rowel = size_t(h_);
  uint8_t* r8 = reinterpret_cast<uint8_t*>(dep_recv_);
  const size_t cb = size_t(h_ / 2), sb = size_t(h_ / 16);  // nvfp4 bytes per row: codes, scales
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    const size_t so = size_t(send_off[size_t(p)]), sr = size_t(send_rows[size_t(p)]);
    const size_t ro = size_t(recv_off[size_t(p)]), rr = size_t(recv_rows[size_t(p)]);
    if (fp4_) {
      if (sr) {
        nccl_check(n.Send(x8 + so * cb, sr * cb, kUint8, p, nccl_, st), "ncclSend");
        nccl_check(n.Send(sfl_ + so * sb, sr * sb, kUint8, p, nccl_, st), "ncclSend");
        nccl_check(n.Send(xs_ + so, sr, kFloat32, p, nccl_, st), "ncclSend");
      }
      if (rr) {
        nccl_check(n.Recv(r8 + ro * cb, rr * cb, kUint8, p, nccl_, st), "ncclRecv");
        nccl_check(n.Recv(dep_sfl_ + ro * sb, rr * sb, kUint8, p, nccl_, st), "ncclRecv");
        nccl_check(n.Recv(dep_xs_ + ro, rr, kFloat32, p, nccl_, st), "ncclRecv");
      }
    } else if (fp8_) {
      if (sr) {
        nccl_check(n.Send(x8 + so * rowel, sr * rowel, kUint8, p, nccl_, st), "ncclSend");
        nccl_check(n.Send(xs_ + so, sr, kFloat32, p, nccl_, st), "ncclSend");
      }
      if (rr) {
        nccl_check(n.Recv(r8 + ro * rowel, rr * rowel, kUint8, p, nccl_, st), "ncclRecv");
        nccl_check(n.Recv(dep_xs_ + ro, rr, kFloat32, p, nccl_, st), "ncclRecv");
      }
    } else {
      if (sr) nccl_check(n.Send(xperm_ + so * rowel, sr * rowel, kBf16, p, nccl_, st), "ncclSend");
      if (rr) nccl_check(n.Recv(dep_recv_ + ro * rowel, rr * rowel, kBf16, p, nccl_, st), "ncclRecv");
    }
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  if (send_rows[size_t(rank_)]) {
    const size_t so = size_t(send_off[size_t(rank_)]), ro = size_t(recv_off[size_t(rank_)]);
    const size_t sr = size_t(send_rows[size_t(rank_)]);
    if (fp4_) {
      DWDP_CUDA(cudaMemcpyAsync(r8 + ro * cb, x8 + so * cb, sr * cb, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dep_sfl_ + ro * sb, sfl_ + so * sb, sr * sb, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dep_xs_ + ro, xs_ + so, sr * 4, cudaMemcpyDeviceToDevice, st));
    } else if (fp8_) {
      DWDP_CUDA(cudaMemcpyAsync(r8 + ro * rowel, x8 + so * rowel, sr * rowel, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dep_xs_ + ro, xs_ + so, sr * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      DWDP_CUDA(cudaMemcpyAsync(dep_recv_ + ro * rowel, xperm_ + so * rowel, sr * rowel * 2,
                                cudaMemcpyDeviceToDevice, st));
    }
  }
  if ((fp8_ || fp4_) && shared_ && T > 0)  // shared-row scales follow the received rows
    DWDP_CUDA(cudaMemcpyAsync(dep_xs_ + routed_rows, xs_ + send_total, size_t(T) * 4,
                              cudaMemcpyDeviceToDevice, st));
  if (fp4_ && shared_ && T > 0) {  // nvfp4: the shared rows' codes and scales too (one A operand)
    DWDP_CUDA(cudaMemcpyAsync(r8 + size_t(routed_rows) * cb, x8 + size_t(send_total) * cb, size_t(T) * cb,
                              cudaMemcpyDeviceToDevice, st));
    DWDP_CUDA(cudaMemcpyAsync(dep_sfl_ + size_t(routed_rows) * sb, sfl_ + size_t(send_total) * sb,
                              size_t(T) * sb, cudaMemcpyDeviceToDevice, st));
  }
  if (fp4_ && nblocks > 0) launch_nvfp4_sf_relayout(dep_sfl_, dep_xsf_, dep_cap_rows_, h_, dep_tab_, st);
  mark(&rec.comm[1]);
  // 4. expert-parallel grouped GEMMs (+ shared expert on own tokens)
  const int32_t* stab = slot_tab_ + size_t(layer) * 2 * (E_ + 1);
  const int32_t* dmeta = dep_tab_;
  const int32_t* dmb = dep_tab_ + 4;
  if (nblocks > 0 && fp4_) {
    GemmArgs g1{int(h_), int(f_), int(f_), E_, dmb, stab, dmeta, dep_h_, f_, INT64_MAX, 0, dep_seg_,
                nullptr, dep_xs_, sarena_[0], sarena_[1], fp4_pair_, raster_, dep_mbrows_, nullptr, 0,
                dep_xsf_, sfarena_[0], sfarena_[1]};
    const CUtensorMap sf1[4] = {tm_dep_sfx_, tm_sf_w_[0], tm_sf_w_[1], tm_dep_h_o_};  // segments padded to row_align_
    launch_grouped_gemm(GEMM_SWIGLU_FP4, tm_dep_x8_, tm_dep_x8_, tm_gate_, tm_up_, g1, int(nblocks * (f_ / 128)),
                        st, sf1);
    launch_quant_rows_nvfp4(dep_h_, dep_cap_rows_, f_, dmeta, dep_h8_, dep_sfl_, dep_hsf_, dep_hs_, st);
  } else if (nblocks > 0 && fp8_) {
    const CUtensorMap tm_x = shared_ && T > 0 ? make_tmap_i8(x8 + send_total * h_, T, h_, 128) : tm_dep_x8_;
    GemmArgs g1{int(h_), int(f_), int(f_), E_, dmb, stab, dmeta, dep_h_, f_, INT64_MAX, 1, dep_seg_,
                nullptr, dep_xs_, sarena_[0], sarena_[1], gemm1_pair_, raster_, dep_mbrows_};
    launch_grouped_gemm(GEMM_SWIGLU_FP8, tm_dep_x8_, tm_x, tm_gate_, tm_up_, g1, int(nblocks * (f_ / 128)), st);
    launch_quant_rows_fp8(dep_h_, dep_cap_rows_, f_, dmeta, dep_h8_, dep_hs_, st);
  } else if (nblocks > 0) {
    const CUtensorMap tm_x = shared_ && T > 0 ? make_tmap_bf16(x, T, h_, 128) : tm_dep_recv_;
    GemmArgs g1{int(h_), int(f_), int(f_), E_, dmb, stab, dmeta, dep_h_, f_, INT64_MAX, 1, dep_seg_,
                nullptr, nullptr, nullptr, nullptr, gemm1_pair_, raster_, dep_mbrows_};
    launch_grouped_gemm(GEMM_SWIGLU, tm_dep_recv_, tm_x, tm_gate_, tm_up_, g1, int(nblocks * (f_ / 128)), st);
  }
  mark(&rec.k[2]);
  if (nblocks > 0 && fp4_) {
    GemmArgs g2{int(f_), int(h_), int(h_), E_, dmb, stab, dmeta, dep_recv_, h_, INT64_MAX, 0, dep_seg_,
                nullptr, dep_hs_, sarena_[2], nullptr, 0, raster_, dep_mbrows_, nullptr, 0,
                dep_hsf_, sfarena_[2], nullptr};
    const CUtensorMap sf2[4] = {tm_dep_sfh_, tm_sf_w_[2], tm_sf_w_[2], tm_dep_o_};
    launch_grouped_gemm(GEMM_PLAIN_FP4, tm_dep_h8_, tm_dep_h8_, tm_down_, tm_down_, g2, int(nblocks * (h_ / 256)),
                        st, sf2);
  } else if (nblocks > 0 && fp8_) {
    GemmArgs g2{int(f_), int(h_), int(h_), E_, dmb, stab, dmeta, dep_recv_, h_, INT64_MAX, 0, dep_seg_,
                nullptr, dep_hs_, sarena_[2], nullptr, gemm2_pair_, raster_, dep_mbrows_};
    const CUtensorMap& tmd8 = gemm2_pair_ ? tm_down_p_ : tm_down_;
    launch_grouped_gemm(GEMM_PLAIN_FP8, tm_dep_h8_, tm_dep_h8_, tmd8, tmd8, g2, int(nblocks * (h_ / 256)), st);
  } else if (nblocks > 0) {
    GemmArgs g2{int(f_), int(h_), int(h_), E_, dmb, stab, dmeta, dep_recv_, h_, INT64_MAX, 0, dep_seg_,
                nullptr, nullptr, nullptr, nullptr, gemm2_pair_, raster_, dep_mbrows_};
    const CUtensorMap& tmd = gemm2_pair_ ? tm_down_p_ : tm_down_;
    launch_grouped_gemm(GEMM_PLAIN, tm_dep_h_, tm_dep_h_, tmd, tmd, g2, int(nblocks * (h_ / 256)), st);
  }
  mark(&rec.k[3]);
  // 5. combine all-to-all: results back into the send layout (xperm)
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    if (recv_rows[size_t(p)])
      nccl_check(n.Send(dep_recv_ + recv_off[size_t(p)] * h_, size_t(recv_rows[size_t(p)]) * rowel,
                        kBf16, p, nccl_, st), "ncclSend");
    if (send_rows[size_t(p)])
      nccl_check(n.Recv(xperm_ + send_off[size_t(p)] * h_, size_t(send_rows[size_t(p)]) * rowel,
                        kBf16, p, nccl_, st), "ncclRecv");
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  if (send_rows[size_t(rank_)])
    DWDP_CUDA(cudaMemcpyAsync(xperm_ + send_off[size_t(rank_)] * h_,
                              dep_recv_ + recv_off[size_t(rank_)] * h_,
                              size_t(send_rows[size_t(rank_)]) * rowel * 2, cudaMemcpyDeviceToDevice, st));
  mark(&rec.comm[3]);
  // 6. weighted combine (shared rows follow the routed rows of the receive buffer)
  combine_into(xperm_, row_of_, wts_, shared_ ? dep_recv_ + routed_rows * h_ : nullptr, nullptr,
               residual ? x : nullptr, y, T, k_, st);
  launches += (T > 0 ? 3 : 0) + np + (nblocks > 0 ? (fp4_ ? 5 : fp8_ ? 3 : 2) : 0) + 1;
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaEventRecord(rec.moe_end, st));
  rec.rows = routed_rows;
  push_record(rec);
}

void Ctx::dep_stack_forward(const uint16_t* x, int64_t T, uint16_t* y, cudaStream_t st) {
  std::vector<int64_t> Ts;
  if (dep_mode == 1) Ts = dep2_exchange_tokens(T, st);  // once per stack: every layer has the same T
  uint16_t* p = ping();  // ping-pong as in stack_forward
  const uint16_t* in = x;
  for (int l = 0; l < L_; ++l) {
    uint16_t* out = ((L_ - 1 - l) % 2 == 0) ? y : p;
    if (in == out) out = (out == y) ? p : y;
    if (dep_mode == 1)
      dep2_layer_forward(l, in, T, out, true, st, Ts);
    else if (dep_mode == 2)
      dep3_layer_forward(l, in, T, out, true, st);
    else
      dep_layer_forward(l, in, T, out, true, st);
    in = out;
  }
  if (in != y) DWDP_CUDA(cudaMemcpyAsync(y, in, size_t(T) * h_ * 2, cudaMemcpyDeviceToDevice, st));
}

// ===================================================================== //
// DEP mode 1: token-deduplicated dispatch + partial combine.

void Ctx::dep2_alloc() {
  if (dep2_x_) return;
  // mode 2 receives up to 127 padding rows per source segment
  const int64_t rows = int64_t(N_) * (max_tokens_ + 128);
  dep2_x_ = static_cast<uint16_t*>(dalloc(size_t(rows) * h_ * 2, &workspace_bytes));
  dep2_idx_ = static_cast<int32_t*>(dalloc(size_t(rows) * k_ * 4, &workspace_bytes));
  dep2_loc_ = static_cast<int32_t*>(dalloc(size_t(rows) * k_ * 4, &workspace_bytes));
  dep2_rowof_ = static_cast<int32_t*>(dalloc(size_t(rows) * k_ * 4, &workspace_bytes));
  dep2_wts_ = static_cast<float*>(dalloc(size_t(rows) * k_ * 4, &workspace_bytes));
  dep2_scratch_ = static_cast<int32_t*>(
      dalloc(size_t(permute_scratch_ints(rows, E_)) * 4, &workspace_bytes));
  dep2_rowf_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * N_ * 4, &workspace_bytes));
  dep2_wf_ = static_cast<float*>(dalloc(size_t(max_tokens_) * N_ * 4, &workspace_bytes));
  dep2_tok_ = static_cast<int32_t*>(dalloc(size_t(N_) * 8 * 4, &workspace_bytes));
  {
    const int per = E_ / N_;
    // receive-side routed rows: the worst case (every received row carries
    // min(k, per) of this rank's experts) when it fits an 8 GB budget (decode
    // batches under Zipf skew), else 1.3x a balanced rank's k T rows (large
    // prefill batches, where routing is close to balanced; an overflowing
    // layer raises on every rank)
    const int64_t balanced = max_tokens_ * k_;  // a rank's expected routed rows
    const int64_t worst = rows * std::min(k_, per);
    const int64_t budget_rows = (int64_t(8) << 30) / (2 * h_ + 3 * f_);
    const int64_t routed = std::min<int64_t>(worst, std::max<int64_t>(balanced * 13 / 10, budget_rows));
    dep2_cap_rows_ = (routed + int64_t(per) * 128 + max_tokens_ + 127) / 128 * 128 + 256;
    dep2_max_mb_ = dep2_cap_rows_ / 128 + 4;
    dep2_xperm_ = static_cast<uint16_t*>(dalloc(size_t(dep2_cap_rows_) * h_ * 2, &workspace_bytes));
    dep2_h_ = static_cast<uint16_t*>(dalloc(size_t(dep2_cap_rows_) * f_ * 2, &workspace_bytes));
    dep2_mblock_ = static_cast<int32_t*>(dalloc(size_t(dep2_max_mb_) * 4, &workspace_bytes));
    dep2_mbrows_ = static_cast<int32_t*>(dalloc(size_t(dep2_max_mb_) * 4, &workspace_bytes));
    dep2_mbseg_ = static_cast<int2*>(dalloc(size_t(dep2_max_mb_) * sizeof(int2), &workspace_bytes));
    dep2_meta_ = static_cast<int32_t*>(dalloc(16 * 4, &workspace_bytes));
    DWDP_CUDA(cudaMemset(dep2_meta_, 0, 16 * 4));
    tm_dep2_xperm_ = make_tmap_bf16(dep2_xperm_, dep2_cap_rows_, h_, 128);
    tm_dep2_h_ = make_tmap_bf16(dep2_h_, dep2_cap_rows_, f_, 128);
    if (fp8_ || fp4_) {  // quantised rows in the dep2_xperm_ bytes, as X_perm8 / X_perm4 in the DWDP path
      const int64_t kd = fp4_ ? 2 : 1, R = dep2_cap_rows_;
      dep2_h8_ = static_cast<uint8_t*>(dalloc(size_t(R * f_ / kd), &workspace_bytes));
      dep2_xs_ = static_cast<float*>(dalloc(size_t(R) * 4, &workspace_bytes));
      dep2_hs_ = static_cast<float*>(dalloc(size_t(R) * 4, &workspace_bytes));
      tm_dep2_x8_ = make_tmap_i8(dep2_xperm_, R, h_ / kd, 128);
      tm_dep2_h8_ = make_tmap_i8(dep2_h8_, R, f_ / kd, 128);
      if (fp4_) {
        dep2_sfl_ = static_cast<uint8_t*>(dalloc(size_t(R * std::max(h_, f_) / 16), &workspace_bytes));
        dep2_xsf_ = static_cast<uint8_t*>(dalloc(size_t(R * h_ / 16), &workspace_bytes));
        dep2_hsf_ = static_cast<uint8_t*>(dalloc(size_t(R * f_ / 16), &workspace_bytes));
        tm_dep2_sfx_ = make_tmap_sf(dep2_xsf_, R * h_ / 16);
        tm_dep2_sfh_ = make_tmap_sf(dep2_hsf_, R * f_ / 16);
        tm_dep2_o_ = make_tmap_out(dep2_xperm_, R, h_);
        tm_dep2_h_o_ = make_tmap_out(dep2_h_, R, f_);
      }
      const int64_t M = max_tokens_;
      dq_x_ = static_cast<uint8_t*>(dalloc(size_t(M * qrow_bytes()), &workspace_bytes));
      dq_xs_ = static_cast<float*>(dalloc(size_t(M) * 4, &workspace_bytes));
      dq_xsr_ = static_cast<float*>(dalloc(size_t(rows) * 4, &workspace_bytes));
      if (fp4_) {
        dq_sfl_ = static_cast<uint8_t*>(dalloc(size_t(M * h_ / 16), &workspace_bytes));
        dq_sflr_ = static_cast<uint8_t*>(dalloc(size_t(rows * h_ / 16), &workspace_bytes));
      }
    }
  }
  DWDP_CUDA(cudaHostAlloc(&dep2_tok_host_, size_t(N_) * 8, 0));
  DWDP_CUDA(cudaHostAlloc(&dep2_flag_host_, 16, 0));
  dep2_flag_host_[0] = 0;
  // the final parts [N][T] live in dep_recv_ (>= N * max_tokens rows)
  dep_reserve(std::max<int64_t>(max_rows_, rows));
}

std::vector<int64_t> Ctx::dep2_exchange_tokens(int64_t T, cudaStream_t st) {
  require(nccl_ != nullptr, "dep: call dep_init first");
  dep2_alloc();
  const Nccl& n = nccl();
  // (T, overflow flag of this rank's previous layers) from every rank: a
  // receive-side overflow anywhere raises on all ranks at the same point
  // (a single rank raising would leave the others waiting in NCCL)
  int64_t* dt = reinterpret_cast<int64_t*>(dep2_tok_);
  const int64_t mine[2] = {T, int64_t(dep2_flag_host_[0])};
  DWDP_CUDA(cudaMemcpyAsync(dt + 2 * N_, mine, 16, cudaMemcpyHostToDevice, st));
  nccl_check(n.AllGather(dt + 2 * N_, dt, 2, kInt64, nccl_, st), "ncclAllGather");
  std::vector<int64_t> all(size_t(2 * N_));
  DWDP_CUDA(cudaMemcpyAsync(all.data(), dt, size_t(2 * N_) * 8, cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> Ts(static_cast<size_t>(N_));
  bool over = false;
  for (int r = 0; r < N_; ++r) {
    Ts[size_t(r)] = all[size_t(2 * r)];
    over = over || all[size_t(2 * r + 1)] != 0;
  }
  invariant(!over, "dep mode 1: receive-side rows exceeded the workspace on some rank");
  return Ts;
}

// Quantised experts: the own token rows quantised once before the dispatch
// (the same per-row e4m3 scale / e2m1 codes with block and row scales the
// DWDP permute computes), so the wire carries 1 or 0.56 bytes per element.
void Ctx::dq_quantize_own(const uint16_t* x, int64_t T, cudaStream_t st) {
  if (T <= 0) return;
  if (fp4_)
    launch_quant_rows_nvfp4(x, T, h_, nullptr, dq_x_, dq_sfl_, dep2_xsf_, dq_xs_, st);
  else
    launch_quant_rows_fp8(x, T, h_, nullptr, dq_x_, dq_xs_, st);
}

// The receive side shared by DEP modes 1 and 2: the received token rows
// dep2_x_ [Tall][h] (this rank's own T tokens first) with their routing
// dep2_idx_ / dep2_wts_ -> expert outputs O in dep2_xperm_ (routed rows, then
// the own tokens' shared-expert rows from dep2_meta_[2]); rec.k[1..3] marked.
// Returns the kernel launches issued.
int Ctx::dep2_experts(int layer, const uint16_t* x, int64_t T, int64_t Tall, cudaStream_t st, LayerRec& rec) {
  const int per = E_ / N_, lo = rank_ * per;
  launch_localize_idx(dep2_idx_, Tall * k_, lo, lo + per, dep2_loc_, st);
  const int32_t* stab = slot_tab_ + size_t(layer) * 2 * (E_ + 1);
  const int64_t mb_ub = dep2_max_mb_;
  const int g1_tiles = int(std::min<int64_t>(mb_ub * (f_ / 128), 1 << 30));
  const int g2_tiles = int(std::min<int64_t>(mb_ub * (h_ / 256), 1 << 30));
  int np = 1;
  auto mark = [&](cudaEvent_t* slot) {
    *slot = take_event();
    DWDP_CUDA(cudaEventRecord(*slot, st));
  };
  if (fp8_ || fp4_) {
    // quantised experts, as the DWDP path: the permute writes e4m3 (e2m1 +
    // block scales) copies of every local (token, expert) row and of the own
    // tokens' shared-expert rows with row scales; GEMM1 emits bf16 H, which
    // is re-quantised for GEMM2; O (bf16) overwrites the quantised rows
    // the received rows are already quantised (codes in the dep2_x_ bytes,
    // row scales dq_xsr_, nvfp4 linear block scales dq_sflr_): the permute
    // moves qrow-byte code rows as bf16 pairs, qrow_meta places each row's
    // scales and the own tokens' shared-expert rows
    uint8_t* x8 = reinterpret_cast<uint8_t*>(dep2_xperm_);
    const int64_t qrow = qrow_bytes();
    if (Tall > 0) {
      np += launch_permute(dep2_loc_, dep2_x_, Tall, E_, k_, qrow / 2, shared_ ? 1 : 0, counts_, dep2_rowof_,
                           dep2_mblock_, dep2_mbseg_, nullptr, dep2_meta_, dep2_xperm_, dep2_scratch_, st, nullptr,
                           nullptr, 128, dep2_mbrows_, nullptr, T, dep2_cap_rows_);
      launch_qrow_meta(dep2_rowof_, Tall, k_, dq_xsr_, fp4_ ? dq_sflr_ : nullptr, int(h_ / 16), dep2_xs_,
                       fp4_ ? dep2_sfl_ : nullptr, dep2_meta_, shared_ ? T : 0,
                       reinterpret_cast<const uint8_t*>(dep2_x_), qrow, x8, st);
      ++np;
    }
    if (fp4_ && Tall > 0) {
      launch_nvfp4_sf_relayout(dep2_sfl_, dep2_xsf_, dep2_cap_rows_, h_, dep2_meta_, st);
      ++np;
    }
    mark(&rec.k[1]);
    if (Tall > 0 && fp4_) {
      GemmArgs g1{int(h_), int(f_), int(f_), E_, dep2_mblock_, stab, dep2_meta_, dep2_h_, f_, INT64_MAX, 0,
                  dep2_mbseg_, nullptr, dep2_xs_, sarena_[0], sarena_[1], 0, raster_, dep2_mbrows_, nullptr, 0,
                  dep2_xsf_, sfarena_[0], sfarena_[1]};
      const CUtensorMap sf1[4] = {tm_dep2_sfx_, tm_sf_w_[0], tm_sf_w_[1], tm_dep2_h_o_};
      launch_grouped_gemm(GEMM_SWIGLU_FP4, tm_dep2_x8_, tm_dep2_x8_, tm_gate_, tm_up_, g1, g1_tiles, st, sf1);
      launch_quant_rows_nvfp4(dep2_h_, dep2_cap_rows_, f_, dep2_meta_, dep2_h8_, dep2_sfl_, dep2_hsf_, dep2_hs_,
                              st);
    } else if (Tall > 0) {
      GemmArgs g1{int(h_), int(f_), int(f_), E_, dep2_mblock_, stab, dep2_meta_, dep2_h_, f_, INT64_MAX, 0,
                  dep2_mbseg_, nullptr, dep2_xs_, sarena_[0], sarena_[1], 0, raster_, dep2_mbrows_};
      launch_grouped_gemm(GEMM_SWIGLU_FP8, tm_dep2_x8_, tm_dep2_x8_, tm_gate_, tm_up_, g1, g1_tiles, st);
      launch_quant_rows_fp8(dep2_h_, dep2_cap_rows_, f_, dep2_meta_, dep2_h8_, dep2_hs_, st);
    }
    mark(&rec.k[2]);
    if (Tall > 0 && fp4_) {
      GemmArgs g2{int(f_), int(h_), int(h_), E_, dep2_mblock_, stab, dep2_meta_, dep2_xperm_, h_, INT64_MAX, 0,
                  dep2_mbseg_, nullptr, dep2_hs_, sarena_[2], nullptr, 0, raster_, dep2_mbrows_, nullptr, 0,
                  dep2_hsf_, sfarena_[2], nullptr};
      const CUtensorMap sf2[4] = {tm_dep2_sfh_, tm_sf_w_[2], tm_sf_w_[2], tm_dep2_o_};
      launch_grouped_gemm(GEMM_PLAIN_FP4, tm_dep2_h8_, tm_dep2_h8_, tm_down_, tm_down_, g2, g2_tiles, st, sf2);
    } else if (Tall > 0) {
      GemmArgs g2{int(f_), int(h_), int(h_), E_, dep2_mblock_, stab, dep2_meta_, dep2_xperm_, h_, INT64_MAX, 0,
                  dep2_mbseg_, nullptr, dep2_hs_, sarena_[2], nullptr, 0, raster_, dep2_mbrows_};
      launch_grouped_gemm(GEMM_PLAIN_FP8, tm_dep2_h8_, tm_dep2_h8_, tm_down_, tm_down_, g2, g2_tiles, st);
    }
    mark(&rec.k[3]);
  } else {
    if (Tall > 0)
      np += launch_permute(dep2_loc_, dep2_x_, Tall, E_, k_, h_, shared_ ? 1 : 0, counts_, dep2_rowof_,
                           dep2_mblock_, dep2_mbseg_, nullptr, dep2_meta_, dep2_xperm_, dep2_scratch_, st, nullptr,
                           nullptr, 128, dep2_mbrows_, nullptr, T, dep2_cap_rows_);
    mark(&rec.k[1]);
    // 4. grouped GEMMs (the rank's expert block + its shared expert)
    const CUtensorMap tm_x = shared_ && T > 0 ? make_tmap_bf16(x, T, h_, 128) : tm_dep2_xperm_;
    GemmArgs g1{int(h_), int(f_), int(f_), E_, dep2_mblock_, stab, dep2_meta_, dep2_h_, f_, INT64_MAX, 1,
                dep2_mbseg_, nullptr, nullptr, nullptr, nullptr, 0, raster_, dep2_mbrows_};
    if (Tall > 0) launch_grouped_gemm(GEMM_SWIGLU, tm_dep2_xperm_, tm_x, tm_gate_, tm_up_, g1, g1_tiles, st);
    mark(&rec.k[2]);
    GemmArgs g2{int(f_), int(h_), int(h_), E_, dep2_mblock_, stab, dep2_meta_, dep2_xperm_, h_, INT64_MAX, 0,
                dep2_mbseg_, nullptr, nullptr, nullptr, nullptr, 0, raster_, dep2_mbrows_};
    if (Tall > 0) launch_grouped_gemm(GEMM_PLAIN, tm_dep2_h_, tm_dep2_h_, tm_down_, tm_down_, g2, g2_tiles, st);
    mark(&rec.k[3]);
  }
  return np;
}

void Ctx::dep2_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                             cudaStream_t st, const std::vector<int64_t>& Ts) {
  struct DG {
    int prev = -1;
    explicit DG(int d) {
      cudaGetDevice(&prev);
      cudaSetDevice(d);
    }
    ~DG() { cudaSetDevice(prev); }
  } dg(cfg.device);
  require(layer >= 0 && layer < L_, "dep: layer out of range");
  require(T >= 0 && T <= max_tokens_, "dep: T exceeds max_tokens");
  require(int64_t(Ts.size()) == N_ && Ts[size_t(rank_)] == T, "dep mode 1: token counts out of date");
  const Nccl& n = nccl();
  const int wl = layer % WL_, per = E_ / N_, lo = rank_ * per;
  // receive layout: this rank's tokens first (the permute's shared-expert
  // rows are tokens [0, T) of its input), then the peers in rank order
  std::vector<int64_t> off(size_t(N_), 0);
  int64_t Tall = T;
  for (int r = 0; r < N_; ++r)
    if (r != rank_) {
      off[size_t(r)] = Tall;
      Tall += Ts[size_t(r)];
    }
  LayerRec rec{int64_t(layer), T, take_event(), take_event(), take_event(), nullptr, -1};
  DWDP_CUDA(cudaEventRecord(rec.gate0, st));
  DWDP_CUDA(cudaEventRecord(rec.gate1, st));
  auto mark = [&](cudaEvent_t* slot) {
    *slot = take_event();
    DWDP_CUDA(cudaEventRecord(*slot, st));
  };
  // 1. router + top-k of the rank's own tokens
  if (T > 0) route_logits(wl, x, T, st);
  mark(&rec.k[0]);
  mark(&rec.comm[0]);  // dispatch start (same point as the router end)
  // 2. dispatch: every token row once to every peer, with its k expert ids
  // and weights (the receiver keeps the pairs of its own expert block);
  // quantised experts: the rows travel quantised (codes, row scale, nvfp4
  // block scales)
  const size_t hk = size_t(k_);
  const bool q = fp8_ || fp4_;
  const size_t qrow = size_t(qrow_bytes()), sfb = size_t(h_ / 16);
  uint8_t* rx = reinterpret_cast<uint8_t*>(dep2_x_);
  if (q) dq_quantize_own(x, T, st);
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    if (T > 0) {
      if (q) {
        nccl_check(n.Send(dq_x_, size_t(T) * qrow, kUint8, p, nccl_, st), "ncclSend");
        nccl_check(n.Send(dq_xs_, size_t(T), kFloat32, p, nccl_, st), "ncclSend");
        if (fp4_) nccl_check(n.Send(dq_sfl_, size_t(T) * sfb, kUint8, p, nccl_, st), "ncclSend");
      } else {
        nccl_check(n.Send(x, size_t(T) * size_t(h_), kBf16, p, nccl_, st), "ncclSend");
      }
      nccl_check(n.Send(idx_, size_t(T) * hk, kInt32, p, nccl_, st), "ncclSend");
      nccl_check(n.Send(wts_, size_t(T) * hk, kFloat32, p, nccl_, st), "ncclSend");
    }
    const int64_t o = off[size_t(p)], tp = Ts[size_t(p)];
    if (tp > 0) {
      if (q) {
        nccl_check(n.Recv(rx + size_t(o) * qrow, size_t(tp) * qrow, kUint8, p, nccl_, st), "ncclRecv");
        nccl_check(n.Recv(dq_xsr_ + o, size_t(tp), kFloat32, p, nccl_, st), "ncclRecv");
        if (fp4_) nccl_check(n.Recv(dq_sflr_ + size_t(o) * sfb, size_t(tp) * sfb, kUint8, p, nccl_, st), "ncclRecv");
      } else {
        nccl_check(n.Recv(dep2_x_ + o * h_, size_t(tp) * size_t(h_), kBf16, p, nccl_, st), "ncclRecv");
      }
      nccl_check(n.Recv(dep2_idx_ + o * k_, size_t(tp) * hk, kInt32, p, nccl_, st), "ncclRecv");
      nccl_check(n.Recv(dep2_wts_ + o * k_, size_t(tp) * hk, kFloat32, p, nccl_, st), "ncclRecv");
    }
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  if (T > 0) {  // own rows first in the receive layout
    if (q) {
      DWDP_CUDA(cudaMemcpyAsync(rx, dq_x_, size_t(T) * qrow, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dq_xsr_, dq_xs_, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
      if (fp4_) DWDP_CUDA(cudaMemcpyAsync(dq_sflr_, dq_sfl_, size_t(T) * sfb, cudaMemcpyDeviceToDevice, st));
    } else {
      DWDP_CUDA(cudaMemcpyAsync(dep2_x_, x, size_t(T) * h_ * 2, cudaMemcpyDeviceToDevice, st));
    }
    DWDP_CUDA(cudaMemcpyAsync(dep2_idx_, idx_, size_t(T) * hk * 4, cudaMemcpyDeviceToDevice, st));
    DWDP_CUDA(cudaMemcpyAsync(dep2_wts_, wts_, size_t(T) * hk * 4, cudaMemcpyDeviceToDevice, st));
  }
  mark(&rec.comm[1]);
  // 3. receive-side permute over every rank's tokens, local experts only:
  // each expert's rows of all sources form one segment; shared expert on
  // the rank's own T tokens (its A rows read from x)
  int np = dep2_experts(layer, x, T, Tall, st, rec);
  // 5. partial combine per received token: sum over this rank's experts of
  // the token's k (row < 0: computed elsewhere); own tokens straight into
  // their slot of the final parts, the rest into the dispatch buffer
  uint16_t* parts = dep_recv_;  // [N][T] partial rows of this rank's tokens
  for (int r = 0; r < N_; ++r) {
    const int64_t o = off[size_t(r)], tr = Ts[size_t(r)];
    if (tr == 0) continue;
    uint16_t* dst = r == rank_ ? parts + int64_t(rank_) * T * h_ : dep2_x_ + o * h_;
    launch_combine_partial(dep2_xperm_, dep2_rowof_ + o * k_, dep2_wts_ + o * k_, dst, tr, k_, h_, st);
    ++np;
  }
  mark(&rec.comm[2]);
  // 6. return all-to-all: one partial row per (token, rank)
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    const int64_t tp = Ts[size_t(p)];
    if (tp > 0)
      nccl_check(n.Send(dep2_x_ + off[size_t(p)] * h_, size_t(tp) * size_t(h_), kBf16, p, nccl_, st),
                 "ncclSend");
    if (T > 0)
      nccl_check(n.Recv(parts + int64_t(p) * T * h_, size_t(T) * size_t(h_), kBf16, p, nccl_, st), "ncclRecv");
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  mark(&rec.comm[3]);
  // 7. final combine: y = sum over ranks (rank order) + shared + residual
  if (T > 0) {
    if (dep2_rowf_T_ != T) {
      launch_rank_rows(dep2_rowf_, dep2_wf_, T, N_, st);
      dep2_rowf_T_ = T;
      ++np;
    }
    combine_into(parts, dep2_rowf_, dep2_wf_, shared_ ? dep2_xperm_ : nullptr, dep2_meta_,
                 residual ? x : nullptr, y, T, N_, st);
  }
  // receive-side overflow flag (meta[4]) -> host, checked at the next stack
  // sticky per rank until raised: max over the stack's layers
  DWDP_CUDA(cudaMemcpyAsync(dep2_flag_host_ + 1, dep2_meta_ + 4, 4, cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaLaunchHostFunc(
      st, [](void* p) {
        int32_t* f = static_cast<int32_t*>(p);
        f[0] |= f[1];
      },
      dep2_flag_host_));
  launches += (T > 0 ? 3 : 0) + np + (Tall > 0 ? (fp4_ || fp8_ ? 3 : 2) : 0) + 1;
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaEventRecord(rec.moe_end, st));
  push_record(rec);
}

// ===================================================================== //
// DEP mode 2: every token row only to the ranks that own at least one of its
// experts (the own rank always), one partial row back per (token, rank).

void Ctx::dep3_alloc() {
  dep2_alloc();
  if (dep3_idx2_) return;
  const int k2 = k_ + 1;
  dep3_cap_rows_ = max_tokens_ * std::min(k2, N_) + int64_t(N_) * 128;
  dep3_idx2_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * k2 * 4, &workspace_bytes));
  dep3_rowof2_ = static_cast<int32_t*>(dalloc(size_t(max_tokens_) * k2 * 4, &workspace_bytes));
  dep3_ones_ = static_cast<float*>(dalloc(size_t(max_tokens_) * k2 * 4, &workspace_bytes));
  launch_fill_f32(dep3_ones_, max_tokens_ * k2, 1.0f, nullptr);
  dep3_xsend_ = static_cast<uint16_t*>(dalloc(size_t(dep3_cap_rows_) * h_ * 2, &workspace_bytes));
  dep3_sidx_ = static_cast<int32_t*>(dalloc(size_t(dep3_cap_rows_) * k_ * 4, &workspace_bytes));
  dep3_swts_ = static_cast<float*>(dalloc(size_t(dep3_cap_rows_) * k_ * 4, &workspace_bytes));
  dep3_counts_ = static_cast<int32_t*>(dalloc(size_t(N_ + 1) * (N_ + 2) * 4, &workspace_bytes));
  dep3_meta_ = static_cast<int32_t*>(dalloc(16 * 4, &workspace_bytes));
  dep3_scratch_ = static_cast<int32_t*>(dalloc(size_t(permute_scratch_ints(max_tokens_, N_)) * 4, &workspace_bytes));
  dep3_mblock_ = static_cast<int32_t*>(dalloc(size_t(dep3_cap_rows_ / 128 + 8) * 4, &workspace_bytes));
  dep3_mbseg_ = static_cast<int2*>(dalloc(size_t(dep3_cap_rows_ / 128 + 8) * sizeof(int2), &workspace_bytes));
  if (fp8_ || fp4_) {
    dq_xs_send_ = static_cast<float*>(dalloc(size_t(dep3_cap_rows_) * 4, &workspace_bytes));
    if (fp4_) dq_sfl_send_ = static_cast<uint8_t*>(dalloc(size_t(dep3_cap_rows_ * h_ / 16), &workspace_bytes));
  }
  DWDP_CUDA(cudaHostAlloc(&dep3_counts_host_, size_t(N_) * (N_ + 1) * 4, 0));
  DWDP_CUDA(cudaDeviceSynchronize());
}

void Ctx::dep3_layer_forward(int layer, const uint16_t* x, int64_t T, uint16_t* y, bool residual,
                             cudaStream_t st) {
  dep3_alloc();
  const Nccl& n = nccl();
  const int wl = layer % WL_, per = E_ / N_, k2 = k_ + 1;
  const bool q = fp8_ || fp4_;
  const size_t qrow = size_t(qrow_bytes()), sfb = size_t(h_ / 16);
  uint8_t* sx = reinterpret_cast<uint8_t*>(dep3_xsend_);
  uint8_t* rx = reinterpret_cast<uint8_t*>(dep2_x_);
  LayerRec rec{int64_t(layer), T, take_event(), take_event(), take_event(), nullptr, -1};
  DWDP_CUDA(cudaEventRecord(rec.gate0, st));
  DWDP_CUDA(cudaEventRecord(rec.gate1, st));
  auto mark = [&](cudaEvent_t* slot) {
    *slot = take_event();
    DWDP_CUDA(cudaEventRecord(*slot, st));
  };
  // 1. router + top-k, destination ranks, token rows permuted into one
  // segment per destination rank (128-row padded), each row's routing
  int np = 0;
  if (T > 0) route_logits(wl, x, T, st);
  mark(&rec.k[0]);
  if (T > 0) {
    launch_dest_ranks(idx_, T, k_, per, rank_, dep3_idx2_, st);
    if (q) {  // quantised experts: the rows travel quantised, with their scales
      dq_quantize_own(x, T, st);
      np += 2 + launch_permute(dep3_idx2_, reinterpret_cast<const uint16_t*>(dq_x_), T, N_, k2, qrow / 2, 0,
                               dep3_counts_, dep3_rowof2_, dep3_mblock_, dep3_mbseg_, nullptr, dep3_meta_,
                               dep3_xsend_, dep3_scratch_, st, nullptr, nullptr, 128);
      launch_qrow_meta(dep3_rowof2_, T, k2, dq_xs_, fp4_ ? dq_sfl_ : nullptr, int(sfb), dq_xs_send_, dq_sfl_send_,
                       nullptr, 0, nullptr, 0, nullptr, st);
    } else {
      np += 1 + launch_permute(dep3_idx2_, x, T, N_, k2, h_, 0, dep3_counts_, dep3_rowof2_, dep3_mblock_,
                               dep3_mbseg_, nullptr, dep3_meta_, dep3_xsend_, dep3_scratch_, st, nullptr, nullptr, 128);
    }
    DWDP_CUDA(cudaMemsetAsync(dep3_sidx_, 0xFF, size_t(dep3_cap_rows_) * k_ * 4, st));  // padding rows: idx -1
    launch_scatter_routing(idx_, wts_, dep3_rowof2_, T, k_, k2, dep3_sidx_, dep3_swts_, st);
    ++np;
  } else {
    DWDP_CUDA(cudaMemsetAsync(dep3_counts_, 0, size_t(N_) * 4, st));
  }
  mark(&rec.comm[0]);  // the send-side permute counts as dispatch
  // 2. rows per (source, destination) from every rank (one host sync, as mode 0)
  // plus this rank's sticky receive-overflow flag of earlier layers: every
  // rank raises at the same point (one rank raising alone would leave the
  // others waiting in NCCL)
  const size_t nc = size_t(N_) + 1;
  int32_t* call = dep3_counts_ + nc;
  DWDP_CUDA(cudaMemcpyAsync(dep3_counts_ + N_, dep2_flag_host_, 4, cudaMemcpyHostToDevice, st));
  nccl_check(n.AllGather(dep3_counts_, call, nc, kInt32, nccl_, st), "ncclAllGather");
  DWDP_CUDA(cudaMemcpyAsync(dep3_counts_host_, call, size_t(N_) * nc * 4, cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < N_; ++p)
    invariant(dep3_counts_host_[size_t(p) * nc + size_t(N_)] == 0,
              "dep mode 2: receive-side rows exceeded the workspace on some rank");
  auto pad = [](int64_t v) { return (v + 127) / 128 * 128; };
  const size_t nr = size_t(N_);
  std::vector<int64_t> send_off(nr), send_rows(nr), recv_off(nr), recv_rows(nr);
  int64_t acc = 0;
  for (int p = 0; p < N_; ++p) {  // the permute's segment layout, rank order
    send_off[size_t(p)] = acc;
    send_rows[size_t(p)] = pad(dep3_counts_host_[size_t(rank_) * nc + size_t(p)]);
    acc += send_rows[size_t(p)];
  }
  for (int p = 0; p < N_; ++p) recv_rows[size_t(p)] = pad(dep3_counts_host_[size_t(p) * nc + size_t(rank_)]);
  int64_t Rtot = recv_rows[size_t(rank_)];  // own rows first: tokens [0, T) in order
  recv_off[size_t(rank_)] = 0;
  for (int p = 0; p < N_; ++p)
    if (p != rank_) {
      recv_off[size_t(p)] = Rtot;
      Rtot += recv_rows[size_t(p)];
    }
  invariant(Rtot <= int64_t(N_) * (max_tokens_ + 128) && acc <= dep3_cap_rows_, "dep mode 2: row capacity");
  // 3. dispatch: rows + their routing
  const size_t hk = size_t(k_);
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    const size_t so = size_t(send_off[size_t(p)]), sr = size_t(send_rows[size_t(p)]);
    const size_t ro = size_t(recv_off[size_t(p)]), rr = size_t(recv_rows[size_t(p)]);
    if (sr) {
      if (q) {
        nccl_check(n.Send(sx + so * qrow, sr * qrow, kUint8, p, nccl_, st), "ncclSend");
        nccl_check(n.Send(dq_xs_send_ + so, sr, kFloat32, p, nccl_, st), "ncclSend");
        if (fp4_) nccl_check(n.Send(dq_sfl_send_ + so * sfb, sr * sfb, kUint8, p, nccl_, st), "ncclSend");
      } else {
        nccl_check(n.Send(dep3_xsend_ + so * h_, sr * size_t(h_), kBf16, p, nccl_, st), "ncclSend");
      }
      nccl_check(n.Send(dep3_sidx_ + so * hk, sr * hk, kInt32, p, nccl_, st), "ncclSend");
      nccl_check(n.Send(dep3_swts_ + so * hk, sr * hk, kFloat32, p, nccl_, st), "ncclSend");
    }
    if (rr) {
      if (q) {
        nccl_check(n.Recv(rx + ro * qrow, rr * qrow, kUint8, p, nccl_, st), "ncclRecv");
        nccl_check(n.Recv(dq_xsr_ + ro, rr, kFloat32, p, nccl_, st), "ncclRecv");
        if (fp4_) nccl_check(n.Recv(dq_sflr_ + ro * sfb, rr * sfb, kUint8, p, nccl_, st), "ncclRecv");
      } else {
        nccl_check(n.Recv(dep2_x_ + ro * h_, rr * size_t(h_), kBf16, p, nccl_, st), "ncclRecv");
      }
      nccl_check(n.Recv(dep2_idx_ + ro * hk, rr * hk, kInt32, p, nccl_, st), "ncclRecv");
      nccl_check(n.Recv(dep2_wts_ + ro * hk, rr * hk, kFloat32, p, nccl_, st), "ncclRecv");
    }
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  {
    const size_t so = size_t(send_off[size_t(rank_)]), sr = size_t(send_rows[size_t(rank_)]);
    if (sr && q) {
      DWDP_CUDA(cudaMemcpyAsync(rx, sx + so * qrow, sr * qrow, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dq_xsr_, dq_xs_send_ + so, sr * 4, cudaMemcpyDeviceToDevice, st));
      if (fp4_) DWDP_CUDA(cudaMemcpyAsync(dq_sflr_, dq_sfl_send_ + so * sfb, sr * sfb, cudaMemcpyDeviceToDevice, st));
    } else if (sr) {
      DWDP_CUDA(cudaMemcpyAsync(dep2_x_, dep3_xsend_ + so * h_, sr * h_ * 2, cudaMemcpyDeviceToDevice, st));
    }
    if (sr) {
      DWDP_CUDA(cudaMemcpyAsync(dep2_idx_, dep3_sidx_ + so * hk, sr * hk * 4, cudaMemcpyDeviceToDevice, st));
      DWDP_CUDA(cudaMemcpyAsync(dep2_wts_, dep3_swts_ + so * hk, sr * hk * 4, cudaMemcpyDeviceToDevice, st));
    }
  }
  mark(&rec.comm[1]);
  // 4. the rank's experts on every received row (+ shared expert on its own T)
  np += dep2_experts(layer, x, T, Rtot, st, rec);
  // 5. one partial row per received row, in the receive layout
  launch_combine_partial(dep2_xperm_, dep2_rowof_, dep2_wts_, dep2_x_, Rtot, k_, h_, st);
  ++np;
  mark(&rec.comm[2]);
  // 6. return: the partial rows back into the send layout
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int p = 0; p < N_; ++p) {
    if (p == rank_) continue;
    const size_t so = size_t(send_off[size_t(p)]), sr = size_t(send_rows[size_t(p)]);
    const size_t ro = size_t(recv_off[size_t(p)]), rr = size_t(recv_rows[size_t(p)]);
    if (rr) nccl_check(n.Send(dep2_x_ + ro * h_, rr * size_t(h_), kBf16, p, nccl_, st), "ncclSend");
    if (sr) nccl_check(n.Recv(dep3_xsend_ + so * h_, sr * size_t(h_), kBf16, p, nccl_, st), "ncclRecv");
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
  if (send_rows[size_t(rank_)])
    DWDP_CUDA(cudaMemcpyAsync(dep3_xsend_ + send_off[size_t(rank_)] * h_, dep2_x_,
                              size_t(send_rows[size_t(rank_)]) * h_ * 2, cudaMemcpyDeviceToDevice, st));
  mark(&rec.comm[3]);
  // 7. y = sum of the token's partials (own rank first, then its destination
  // ranks in first-occurrence order) + shared + residual
  if (T > 0) {
    const uint16_t* resid = residual ? x : nullptr;
    uint16_t* out = (resid != nullptr && resid == y) ? ping() : y;
    launch_combine_sparse(dep3_xsend_, dep3_rowof2_, dep3_ones_, shared_ ? dep2_xperm_ : nullptr, dep2_meta_, resid,
                          out, T, k2, h_, st);
    if (out != y) DWDP_CUDA(cudaMemcpyAsync(y, out, size_t(T) * h_ * 2, cudaMemcpyDeviceToDevice, st));
    ++np;
  }
  // receive-side overflow (meta[4]) -> the sticky host flag, exchanged with
  // the next layer's counts
  DWDP_CUDA(cudaMemcpyAsync(dep2_flag_host_ + 1, dep2_meta_ + 4, 4, cudaMemcpyDeviceToHost, st));
  DWDP_CUDA(cudaLaunchHostFunc(
      st, [](void* p) {
        int32_t* f = static_cast<int32_t*>(p);
        f[0] |= f[1];
      },
      dep2_flag_host_));
  launches += np + (T > 0 ? 2 : 0) + (Rtot > 0 ? (fp4_ || fp8_ ? 3 : 2) : 0);
  DWDP_CUDA(cudaGetLastError());
  DWDP_CUDA(cudaEventRecord(rec.moe_end, st));
  push_record(rec);
}

}  // namespace dwdp
