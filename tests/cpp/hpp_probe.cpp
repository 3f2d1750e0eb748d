// Drop-in check: code written against the reference API names compiles
// against include/dwdp.hpp + libdwdp.so and reproduces the reference's
// results (compared with tests/golden/ref_*.json by tests/test_dwdp_hpp.py).
#include <cstdio>

#include "dwdp.hpp"

using namespace dwdpsim;

int main() {
  const int cases[][3] = {{256, 8, 0}, {256, 3, 0}, {16, 4, 1}, {97, 5, 2}};
  for (const auto& c : cases) {
    const PlacementPlan p = build_placement(c[0], c[1], c[2]);
    std::printf("P %d %d %d %d %d", c[0], c[1], c[2], p.local_count, p.redundancy);
    for (const auto& fl : p.fetch_lists)
      for (const auto& [e, s] : fl) std::printf(" %d:%d", e, s);
    std::printf("\n");
  }
  const CopyPlan plan = build_copy_plan({{1, 0, 5, 0}, {2, 0, 5, 0}}, 2, 0);
  std::printf("C");
  for (const auto& s : plan.slices)
    std::printf(" %d,%llu,%llu", s.src_rank, static_cast<unsigned long long>(s.dst_offset),
                static_cast<unsigned long long>(s.length));
  std::printf("\n");
  try {
    build_placement(8, 1, 0);
    std::printf("E none\n");
  } catch (const ConfigError&) {
    std::printf("E ConfigError\n");
  }
  MoeModelSpec m;
  m.hidden_dim = 512;
  m.num_experts = 16;
  m.top_k = 2;
  m.expert_ffn_dim = 1024;
  m.attn_proj_params = 1;
  const auto r = route_tokens(100, m, 1.2, 1);
  std::printf("R");
  for (auto v : r) std::printf(" %lld", static_cast<long long>(v));
  std::printf("\n");
  return 0;
}
