// MLA prefill attention block (host side): the attention step of the DWDP
// prefetch window on sm_100a kernels only -- the five projections on the
// tcgen05 GEMM (one dense group), RMSNorm / RoPE / K-V assembly glue kernels
// and the tcgen05 flash-attention core (attn_sm100.cu). Reference cost model:
// attention_entries (/root/reference/proj/src/modelspec.cpp:38-55).
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dwdp.h"
#include "attn_sm100.hpp"
#include "plan.hpp"
#include "runtime.hpp"

namespace dwdp {

namespace {
void dense_gemm(const uint16_t* A, int64_t M, int64_t K, const uint16_t* W, int64_t N, uint16_t* D,
                cudaStream_t st) {
  if (M <= 0) return;
  const CUtensorMap ta = make_tmap_bf16(A, M, K, 128);
  const CUtensorMap tb = make_tmap_bf16(W, N, K, 256);
  GemmArgs g{};
  g.K = int(K);
  g.n_out = int(N);
  g.rows_per_slot = int(N);
  g.E = -1;
  g.D = D;
  g.ldd = N;
  g.m_limit = M;
  g.dense_m = M;
  launch_grouped_gemm(GEMM_PLAIN, ta, ta, tb, tb, g, int((M + 127) / 128 * (N / 256)), st);
}
}  // namespace

class Mla {
 public:
  explicit Mla(const dwdp_mla_config& c) : cfg(c) {
    require(c.nope == 128 && c.rope == 64 && c.v_dim == 128,
            "mla: the attention kernel is built for qk_nope 128, qk_rope 64, v_head 128");
    require(c.heads >= 1 && c.heads % 4 == 0, "mla: heads must be a positive multiple of 4");
    require(c.hidden > 0 && c.hidden % 256 == 0, "mla: hidden must be a positive multiple of 256");
    require(c.q_lora > 0 && c.q_lora % 256 == 0, "mla: q_lora must be a positive multiple of 256");
    require(c.kv_lora > 0 && c.kv_lora % 64 == 0, "mla: kv_lora must be a positive multiple of 64");
    require(c.max_tokens >= 1, "mla: max_tokens must be >= 1");
    DWDP_CUDA(cudaSetDevice(c.device));
    H_ = c.heads;
    T_ = c.max_tokens;
    kva_ld_ = (c.kv_lora + c.rope + 255) / 256 * 256;
    max_tiles_ = T_ / 128 + T_ + 1;  // one partial tile per sequence at most
    // every sequence's V^T columns start 64-aligned: room for 64 sequences'
    // padding up front, grown on demand (forward) for more, shorter ones
    ldv_ = (T_ + 64 * 64 + 7) / 8 * 8;
    auto alloc = [&](size_t bytes) {
      void* p = nullptr;
      DWDP_CUDA(cudaMalloc(&p, bytes));
      bufs_.push_back(p);
      bytes_ += bytes;
      return static_cast<uint16_t*>(p);
    };
    qa_ = alloc(size_t(T_) * c.q_lora * 2);
    q_ = alloc(size_t(T_) * H_ * 192 * 2);
    kva_ = alloc(size_t(T_) * kva_ld_ * 2);
    ckv_ = alloc(size_t(T_) * c.kv_lora * 2);
    kv_ = alloc(size_t(T_) * H_ * 256 * 2);
    k_ = alloc(size_t(T_) * H_ * 192 * 2);
    DWDP_CUDA(cudaMalloc(reinterpret_cast<void**>(&vt_), size_t(H_) * 128 * ldv_ * 2));
    o_ = alloc(size_t(T_) * H_ * 128 * 2);
    pos_ = reinterpret_cast<int32_t*>(alloc(size_t(2 * T_) * 4));  // positions, then V^T columns
    tiles_ = reinterpret_cast<AttnTile*>(alloc(size_t(max_tiles_) * sizeof(AttnTile)));
    DWDP_CUDA(cudaHostAlloc(&pos_h_, size_t(2 * T_) * 4, 0));
    DWDP_CUDA(cudaHostAlloc(&tiles_h_, size_t(max_tiles_) * sizeof(AttnTile), 0));
    DWDP_CUDA(cudaEventCreateWithFlags(&staged_, cudaEventDisableTiming));
  }
  ~Mla() {
    cudaDeviceSynchronize();
    for (void* p : bufs_) cudaFree(p);
    if (vt_) cudaFree(vt_);
    if (pos_h_) cudaFreeHost(pos_h_);
    if (tiles_h_) cudaFreeHost(tiles_h_);
    if (staged_) cudaEventDestroy(staged_);
  }

  void forward(const dwdp_mla_weights& w, const uint16_t* x, int64_t T, const int64_t* seqs, int nseq,
               uint16_t* y, cudaStream_t st) {
    require(T >= 0 && T <= T_, "mla: T exceeds max_tokens");
    require(nseq >= 0, "mla: negative sequence count");
    int64_t sum = 0;
    for (int i = 0; i < nseq; ++i) {
      require(seqs[i] >= 1, "mla: empty sequence");
      sum += seqs[i];
    }
    require(sum == T, "mla: sequence lengths must sum to T");
    if (T == 0) return;
    for (const void* p : {w.wq_a, w.wq_b, w.wkv_a, w.wkv_b, w.wo})
      require(p != nullptr, "mla: missing weight");
    // positions and (heaviest-first) query tiles, staged through pinned memory
    DWDP_CUDA(cudaEventSynchronize(staged_));
    std::vector<AttnTile> tl;
    const int qstep = mla_attention_query_step();
    int64_t s0 = 0, v0 = 0;
    for (int i = 0; i < nseq; ++i) {
      const int64_t L = seqs[i];
      for (int64_t t = 0; t < L; ++t) {
        pos_h_[s0 + t] = int32_t(t);
        pos_h_[T + s0 + t] = int32_t(v0 + t);
      }
      for (int64_t q0 = 0; q0 < L; q0 += qstep) tl.push_back({int32_t(s0), int32_t(L), int32_t(q0), int32_t(v0)});
      s0 += L;
      v0 += (L + 63) / 64 * 64;
    }
    if (v0 > ldv_) {  // many short sequences: grow V^T (cudaFree synchronises)
      cudaFree(vt_);
      ldv_ = (v0 + 4096 + 7) / 8 * 8;
      DWDP_CUDA(cudaMalloc(reinterpret_cast<void**>(&vt_), size_t(H_) * 128 * ldv_ * 2));
    }
    std::stable_sort(tl.begin(), tl.end(), [qstep](const AttnTile& a, const AttnTile& b) {
      return std::min(a.q0 + qstep, a.len) > std::min(b.q0 + qstep, b.len);
    });
    require(int64_t(tl.size()) <= max_tiles_, "mla: too many query tiles");
    std::copy(tl.begin(), tl.end(), tiles_h_);
    DWDP_CUDA(cudaMemcpyAsync(pos_, pos_h_, size_t(2 * T) * 4, cudaMemcpyHostToDevice, st));
    DWDP_CUDA(cudaMemcpyAsync(tiles_, tiles_h_, tl.size() * sizeof(AttnTile), cudaMemcpyHostToDevice, st));
    DWDP_CUDA(cudaEventRecord(staged_, st));
    auto W = [](const void* p) { return static_cast<const uint16_t*>(p); };
    // DWDP_MLA_SYNC=1: synchronise and check after every step (debugging)
    static const bool dbg = std::getenv("DWDP_MLA_SYNC") != nullptr;
    auto chk = [&](const char* what) {
      if (!dbg) return;
      const cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) throw CudaError(std::string("mla ") + what + ": " + cudaGetErrorString(e));
    };
    const int64_t h = cfg.hidden, ql = cfg.q_lora, kl = cfg.kv_lora;
    // q = rms(x Wq_a^T) Wq_b^T
    dense_gemm(x, T, h, W(w.wq_a), ql, qa_, st);
    chk("q_a gemm");
    launch_rmsnorm(qa_, ql, qa_, ql, T, int(ql), 1e-6f, st);
    chk("q rmsnorm");
    dense_gemm(qa_, T, ql, W(w.wq_b), int64_t(H_) * 192, q_, st);
    chk("q_b gemm");
    // kva = x Wkv_a^T (rows padded to 256), kv = rms(ckv) Wkv_b^T
    dense_gemm(x, T, h, W(w.wkv_a), kva_ld_, kva_, st);
    chk("kv_a gemm");
    launch_rmsnorm(kva_, kva_ld_, ckv_, kl, T, int(kl), 1e-6f, st);
    chk("kv rmsnorm");
    dense_gemm(ckv_, T, kl, W(w.wkv_b), int64_t(H_) * 256, kv_, st);
    chk("kv_b gemm");
    // RoPE, K / V^T assembly, attention, output projection
    launch_q_rope(q_, pos_, T, H_, cfg.rope_theta, st);
    chk("q rope");
    launch_kv_assemble(kv_, kva_, kva_ld_, int(kl), pos_, pos_ + T, T, H_, cfg.rope_theta, k_, vt_, ldv_, st);
    chk("kv assemble");
    launch_mla_attention(q_, k_, vt_, T, ldv_, H_, tiles_, int(tl.size()), cfg.softmax_scale, o_, st);
    chk("attention");
    dense_gemm(o_, T, int64_t(H_) * 128, W(w.wo), h, y, st);
    chk("o_proj gemm");
    launches += 10;
    DWDP_CUDA(cudaGetLastError());
  }

  dwdp_mla_config cfg;
  int64_t launches = 0;
  uint64_t bytes_ = 0;

 private:
  int H_ = 0;
  int64_t T_ = 0, kva_ld_ = 0, ldv_ = 0, max_tiles_ = 0;
  std::vector<void*> bufs_;
  uint16_t *qa_ = nullptr, *q_ = nullptr, *kva_ = nullptr, *ckv_ = nullptr, *kv_ = nullptr, *k_ = nullptr,
           *vt_ = nullptr, *o_ = nullptr;
  int32_t* pos_ = nullptr;
  AttnTile* tiles_ = nullptr;
  int32_t* pos_h_ = nullptr;
  AttnTile* tiles_h_ = nullptr;
  cudaEvent_t staged_ = nullptr;
};

}  // namespace dwdp

struct dwdp_mla {
  dwdp::Mla* impl;
};

extern "C" {

int dwdp_mla_create(const dwdp_mla_config* cfg, dwdp_mla** out) {
  return dwdp::capi_guard([&] {
    dwdp::require(cfg != nullptr && out != nullptr, "mla: cfg / out is NULL");
    *out = new dwdp_mla{new dwdp::Mla(*cfg)};
  });
}

int dwdp_mla_destroy(dwdp_mla* m) {
  return dwdp::capi_guard([&] {
    if (!m) return;
    delete m->impl;
    delete m;
  });
}

int dwdp_mla_forward(dwdp_mla* m, const dwdp_mla_weights* w, const void* x, int64_t T, const int64_t* seq_lens,
                     int n_seqs, void* y, void* stream) {
  return dwdp::capi_guard([&] {
    dwdp::require(m != nullptr && w != nullptr, "mla: handle / weights is NULL");
    dwdp::require(T == 0 || (x != nullptr && y != nullptr && seq_lens != nullptr), "mla: NULL buffer");
    m->impl->forward(*w, static_cast<const uint16_t*>(x), T, seq_lens, n_seqs, static_cast<uint16_t*>(y),
                     static_cast<cudaStream_t>(stream));
  });
}

int dwdp_mla_launch_count(const dwdp_mla* m, int64_t* n) {
  return dwdp::capi_guard([&] {
    dwdp::require(m != nullptr && n != nullptr, "mla: NULL argument");
    *n = m->impl->launches;
  });
}

}  // extern "C"
