// Written against the reference API only (include "dwdpsim/..."): built once
// against the adapter + libdwdp.so and once against the reference library;
// tests/test_reference_unit_tests.py requires byte-identical output.
#include <cstdio>
#include <string>

#include "dwdpsim/placement.hpp"
#include "dwdpsim/simcore.hpp"
#include "dwdpsim/workload.hpp"

using namespace dwdpsim;

int main() {
  MoeModelSpec m;
  m.hidden_dim = 7168;
  m.num_experts = 256;
  m.top_k = 8;
  m.expert_ffn_dim = 2048;
  m.shared_ffn_dim = 2048;
  m.attn_proj_params = 187e6;
  m.kv_bytes_per_token_per_layer = 576;
  m.others_bytes_factor = 40;
  m.calib.grouped_gemm = 0.55;
  WorkloadSpec spec;
  spec.isl_dist = IslDist::from_cv(8192, 0.2);
  spec.max_num_tokens = 65536;
  spec.batch_per_rank = 8;
  spec.routing_skew = 0.8;
  spec.seed = 7;
  const auto batches = sample_batches(spec, m, 4, 6);
  const std::string csv = batches_to_csv(batches);
  std::fputs(csv.c_str(), stdout);
  std::printf("roundtrip %d\n", batches_to_csv(batches_from_csv(csv)) == csv ? 1 : 0);
  for (const auto& b : batches) std::printf("cv %.17g\n", imbalance_cv(b));
  const PlacementPlan plan = build_placement(256, 3, 5);
  std::fputs(describe_placement(plan).c_str(), stdout);
  GpuSpec gpu;
  for (long msl : {1024L, 8192L}) {
    const AnalyticResult r = analytic_compare(m, gpu, plan, 32768, msl);
    std::printf("analytic %.17g %.17g %.17g %.17g %d\n", r.t_compute_s, r.t_prefetch_s,
                r.t_all2all_s, r.dep_dwdp_speedup, r.prefetch_saturated ? 1 : 0);
  }
  const LayerWork w = layer_costs(m, 4096, 2048);
  for (const auto& op : w.attn) std::printf("attn %s %.17g %.17g\n", category_name(op.category), op.flops, op.bytes);
  for (const auto& op : w.moe) std::printf("moe %s %.17g %.17g\n", category_name(op.category), op.flops, op.bytes);
  std::printf("total %.17g\n", w.total_time(gpu));
  return 0;
}
