// GPU drop-in probe: a C++ host program written against the reference-named
// adapter (include/dwdp.hpp) and the C-ABI only -- no Python, no torch. Two
// DWDP ranks on device 0 own half the experts each and pull the rest through
// the prefetch engine (CopyEngineSim::issue_plan / plan_done made real); every
// layer's output must equal the all-local model's, byte for byte.
// Device buffers come from the CUDA driver API (the primary context that
// libdwdp.so's runtime also uses). Built and run by tests/test_cpp_gpu.py.
#include <cuda.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "dwdp.hpp"

#define CU(x)                                                            \
  do {                                                                   \
    CUresult r_ = (x);                                                   \
    if (r_ != CUDA_SUCCESS) {                                            \
      std::printf("CUDA driver error %d at %s:%d\n", int(r_), __FILE__, __LINE__); \
      return 1;                                                          \
    }                                                                    \
  } while (0)

static dwdp_ctx_config tiny(int rank, int group, int engine) {
  dwdp_ctx_config c;
  std::memset(&c, 0, sizeof c);
  c.num_layers = 3;
  c.num_experts = 16;
  c.hidden = 512;
  c.ffn = 1024;
  c.shared_ffn = 1024;
  c.top_k = 2;
  c.scoring = 0;  // softmax top-2 (BASELINE config 1)
  c.n_group = 1;
  c.topk_group = 1;
  c.norm_topk = 1;
  c.routed_scale = 1.0f;
  c.rank = rank;
  c.group_size = group;
  c.merge_elim = 1;
  c.tdm = 1;
  c.slice_size = 1 << 18;
  c.engine = engine;
  c.pull_ctas = 0;
  c.ce_inflight = 2;
  c.weight_dtype = DWDP_WEIGHT_BF16;
  c.weight_seed = 2604;
  c.weight_layers = 3;
  c.max_tokens = 512;
  return c;
}

int main() {
  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUcontext pctx;
  CU(cuDevicePrimaryCtxRetain(&pctx, dev));
  CU(cuCtxSetCurrent(pctx));
  int bad = 0;
  try {
    for (int engine : {DWDP_ENGINE_COPY, DWDP_ENGINE_PULL}) {
      dwdpsim::Engine r0(tiny(0, 2, engine)), r1(tiny(1, 2, engine)), full(tiny(0, 1, engine));
      r0.init_weights();
      r1.init_weights();
      full.init_weights();
      dwdp_ctx* pair[2] = {r0.get(), r1.get()};
      dwdpsim::detail::check(dwdp_ctx_link_local(pair, 2));
      const int64_t T = 300, h = 512;
      CUdeviceptr x, y, yf;
      CU(cuMemAlloc(&x, size_t(T * h * 2)));
      CU(cuMemAlloc(&y, size_t(T * h * 2)));
      CU(cuMemAlloc(&yf, size_t(T * h * 2)));
      dwdpsim::detail::check(dwdp_fill_bf16(reinterpret_cast<void*>(x), T * h, 77, 1.0f, nullptr));
      std::vector<uint16_t> a(size_t(T * h)), b(size_t(T * h));
      for (int64_t g = 0; g < 4; ++g) {  // crosses the stack boundary (L = 3)
        r0.layer_forward(g, reinterpret_cast<void*>(x), T, reinterpret_cast<void*>(y), false, nullptr);
        dwdpsim::detail::check(dwdp_moe_forward(full.get(), int(g % 3), reinterpret_cast<void*>(x), T,
                                             reinterpret_cast<void*>(yf), nullptr));
        CU(cuCtxSynchronize());
        CU(cuMemcpyDtoH(a.data(), y, a.size() * 2));
        CU(cuMemcpyDtoH(b.data(), yf, b.size() * 2));
        const bool same = std::memcmp(a.data(), b.data(), a.size() * 2) == 0;
        std::printf("L engine=%d layer=%lld %s\n", engine, static_cast<long long>(g),
                    same ? "bitwise-equal" : "MISMATCH");
        bad += same ? 0 : 1;
      }
      dwdp_layer_record rec[8];
      size_t n = 8;
      dwdpsim::detail::check(dwdp_ctx_records(r0.get(), rec, &n));
      std::printf("R engine=%d records=%zu prefetch_bytes=%.0f\n", engine, n,
                  n > 1 ? rec[1].prefetch_bytes : -1.0);
      cuMemFree(x);
      cuMemFree(y);
      cuMemFree(yf);
    }
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    return 2;
  }
  std::printf("DONE bad=%d\n", bad);
  return bad ? 1 : 0;
}
