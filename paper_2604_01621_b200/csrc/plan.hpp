// Host-side planning layer of the DWDP hot path (pure, reentrant C++).
//
// B200-native counterparts of the reference's L2 planners
// (/root/reference/proj/include/dwdpsim/{placement,copyplan,workload}.hpp)
// and of the MoE cost formulas it uses as a roofline
// (include/dwdpsim/modelspec.hpp). Same semantics and error contract
// (ConfigError / InvariantViolation), independent implementation.
#pragma once

#include <cstdint>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace dwdp {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvariantViolation : std::logic_error {
  using std::logic_error::logic_error;
};
inline void require(bool ok, const char* msg) {
  if (!ok) throw ConfigError(msg);
}
inline void require(bool ok, const std::string& msg) {
  if (!ok) throw ConfigError(msg);
}
inline void invariant(bool ok, const char* msg) {
  if (!ok) throw InvariantViolation(msg);
}

// ---------------------------------------------------------------- placement
struct Placement {
  int group_size = 0, num_experts = 0, local_count = 0, redundancy = 0;
  std::vector<std::vector<int>> local_sets;                    // sorted
  std::vector<std::vector<std::pair<int, int>>> fetch_lists;   // (expert, src)
  bool holds(int rank, int expert) const;
  void validate() const;
  std::string describe() const;
};

Placement build_placement(int num_experts, int group_size, int extra);
std::vector<std::vector<std::pair<int, int>>> assign_fetch_sources(
    int num_experts, const std::vector<std::vector<int>>& local_sets);

// ---------------------------------------------------------------- copy plan
struct ShardRef {
  int peer = 0;
  uint64_t param_id = 0, size = 0, src_offset = 0;
};
struct Slice {
  uint64_t param_id = 0;
  int src_rank = 0;
  uint64_t src_offset = 0, dst_offset = 0, length = 0;
};
std::vector<Slice> build_copy_plan(const std::vector<ShardRef>& shards,
                                   uint64_t slice_size, int dst_rank);

// ---------------------------------------------------------------- workload
// Bit-reproducible generator: std::mt19937_64 (sequence fixed by the C++
// standard) with the transforms written out (rng.hpp:13-70).
class Rng {
 public:
  explicit Rng(uint64_t seed) : g_(seed) {}
  static uint64_t mix(uint64_t a, uint64_t b);
  uint64_t u64() { return g_(); }
  double u01() { return static_cast<double>(g_() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n);
  double normal(double mean, double sd);

 private:
  std::mt19937_64 g_;
};

struct WorkloadSpec {
  int isl_kind = 0;  // 0 fixed, 1 uniform_ratio, 2 normal
  double length = 8192, ratio = 1.0, stddev = 0.0;
  int64_t max_num_tokens = 32768;
  int batch_per_rank = 1;
  double routing_skew = 0.0;
  uint64_t seed = 1;
  void validate() const;
  double cv() const;
};

std::vector<int64_t> route_tokens(int64_t tokens, int num_experts, int top_k,
                                  double skew, uint64_t seed);
struct Batches {  // [iteration][rank] (+ [expert])
  std::vector<std::vector<int64_t>> tokens, requests;
  std::vector<std::vector<std::vector<int64_t>>> routed;
};
Batches sample_batches(const WorkloadSpec& spec, int num_experts, int top_k,
                       int num_ranks, int iterations, bool with_routing);
double imbalance_cv(const std::vector<int64_t>& tokens);
// Exact workload replay (workload.hpp:77-79): one row per (iteration, rank),
// expert counts ';'-separated. routed may be empty (no routing drawn).
std::string batches_to_csv(const Batches& b);
Batches batches_from_csv(const std::string& csv);

// ---------------------------------------------------------------- costs
// MoeModelSpec (modelspec.hpp:13-40) incl. the attention block terms and
// the per-category calibration scalars.
struct ModelSpec {
  int num_layers = 1, num_experts = 1, top_k = 1;
  int64_t hidden = 0, ffn = 0, shared_ffn = 0;
  double wbytes = 2.0, abytes = 2.0;
  double attn_proj_params = 0, kv_bytes = 0, others_factor = 0;
  double calib_attention = 1.0, calib_grouped = 1.0, calib_dense = 1.0;
  void validate() const;  // modelspec.cpp:6-23
};
double expert_shard_bytes(const ModelSpec& m);
struct OpCost {
  int category;  // Category order of hwmodel.hpp:14-23
  double flops, bytes;
};
std::vector<OpCost> attention_entries(const ModelSpec& m, double tokens, double msl);
std::vector<OpCost> moe_entries(const ModelSpec& m, double tokens,
                                double pairs, int touched);
// layer_costs (modelspec.cpp:88-98): validates, then attn + moe entries
// with routed_pairs = T*k over all E experts.
void layer_costs(const ModelSpec& m, int64_t tokens, int64_t msl, std::vector<OpCost>& attn,
                 std::vector<OpCost>& moe);

}  // namespace dwdp
