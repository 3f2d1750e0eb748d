// dwdp.hpp — header-only C++ adapter over the C-ABI (dwdp.h) that mirrors the
// reference operator API for the DWDP path: the names, value types, argument
// meaning and exception behaviour of /root/reference/proj/include/dwdpsim/
// {placement,copyplan,workload,modelspec}.hpp. A maintainer of the reference
// swaps `#include "dwdpsim/placement.hpp"` for this header and links
// libdwdp.so; see INTEGRATION.md.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dwdp.h"

namespace dwdpsim_b200 {

// errors.hpp:11-21
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class InvariantViolation : public std::logic_error {
 public:
  explicit InvariantViolation(const std::string& m) : std::logic_error(m) {}
};
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int st) {
  if (st == DWDP_OK) return;
  const std::string msg = dwdp_last_error();
  if (st == DWDP_ERR_CONFIG) throw ConfigError(msg);
  if (st == DWDP_ERR_INVARIANT) throw InvariantViolation(msg);
  throw CudaError(msg);
}

// placement.hpp:13-25
struct PlacementPlan {
  int group_size = 0, num_experts = 0, local_count = 0, redundancy = 0;
  std::vector<std::vector<int>> local_sets;
  std::vector<std::vector<std::pair<int, int>>> fetch_lists;
  bool holds(int rank, int expert) const {
    for (int e : local_sets.at(static_cast<size_t>(rank)))
      if (e == expert) return true;
    return false;
  }
};

// placement.hpp:30-34
inline PlacementPlan build_placement(int num_experts, int group_size, int extra_redundancy = 0) {
  dwdp_placement* p = nullptr;
  check(dwdp_placement_build(num_experts, group_size, extra_redundancy, &p));
  PlacementPlan out;
  check(dwdp_placement_info(p, &out.group_size, &out.num_experts, &out.local_count,
                            &out.redundancy));
  for (int r = 0; r < out.group_size; ++r) {
    std::vector<int> ls(static_cast<size_t>(out.local_count));
    check(dwdp_placement_local_set(p, r, ls.data()));
    const size_t m = static_cast<size_t>(out.num_experts - out.local_count);
    std::vector<int> fe(m + 1), fs(m + 1);
    check(dwdp_placement_fetch_list(p, r, fe.data(), fs.data()));
    std::vector<std::pair<int, int>> fl;
    for (size_t i = 0; i < m; ++i) fl.emplace_back(fe[i], fs[i]);
    out.local_sets.push_back(std::move(ls));
    out.fetch_lists.push_back(std::move(fl));
  }
  dwdp_placement_free(p);
  return out;
}

// placement.hpp:41-42 (shard bytes = expert_shard_bytes(model))
inline double prefetch_bytes(const PlacementPlan& plan, double expert_shard_bytes) {
  return static_cast<double>(plan.num_experts - plan.local_count) * expert_shard_bytes;
}

// copyplan.hpp:15-38
struct ShardRef {
  int peer = 0;
  std::uint64_t param_id = 0, size = 0, src_offset = 0;
};
struct Slice {
  std::uint64_t param_id = 0;
  int src_rank = 0;
  std::uint64_t src_offset = 0, dst_offset = 0, length = 0;
};
struct CopyPlan {
  int dst_rank = 0;
  std::uint64_t slice_size = 0;
  std::vector<Slice> slices;
  std::uint64_t total_bytes() const {
    std::uint64_t n = 0;
    for (const auto& s : slices) n += s.length;
    return n;
  }
};

// copyplan.hpp:44-45
inline CopyPlan build_copy_plan(const std::vector<ShardRef>& shards, std::uint64_t slice_size,
                                int dst_rank = 0) {
  std::vector<dwdp_shard_ref> in;
  for (const auto& s : shards) in.push_back({s.peer, 0, s.param_id, s.size, s.src_offset});
  size_t n = 0;
  check(dwdp_copy_plan_build(in.data(), in.size(), slice_size, dst_rank, nullptr, &n));
  std::vector<dwdp_slice> out(n + 1);
  check(dwdp_copy_plan_build(in.data(), in.size(), slice_size, dst_rank, out.data(), &n));
  CopyPlan plan;
  plan.dst_rank = dst_rank;
  plan.slice_size = slice_size;
  for (size_t i = 0; i < n; ++i)
    plan.slices.push_back({out[i].param_id, out[i].src_rank, out[i].src_offset,
                           out[i].dst_offset, out[i].length});
  return plan;
}

// workload.hpp:57-65
inline std::vector<std::int64_t> route_tokens(std::int64_t tokens, int num_experts, int top_k,
                                              double routing_skew, std::uint64_t seed) {
  std::vector<std::int64_t> counts(static_cast<size_t>(num_experts));
  check(dwdp_route_tokens(tokens, num_experts, top_k, routing_skew, seed, counts.data()));
  return counts;
}

// The real per-GPU engine behind simulate_dwdp's step loop (simcore.cpp:640-733):
// owns the split-weight arenas, the prefetch engine and the MoE kernels.
class Engine {
 public:
  explicit Engine(const dwdp_ctx_config& cfg) { check(dwdp_ctx_create(&cfg, &ctx_)); }
  ~Engine() { dwdp_ctx_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  dwdp_ctx* get() const { return ctx_; }
  void init_weights(float bias_scale = 0.0f) { check(dwdp_ctx_init_weights(ctx_, bias_scale)); }
  // CopyEngineSim::issue_plan / plan_done (simcore.hpp:93-101)
  std::int64_t issue_plan(std::int64_t global_layer) {
    dwdp_prefetch h = -1;
    check(dwdp_prefetch_issue(ctx_, global_layer, &h));
    return h;
  }
  bool plan_done(std::int64_t h) {
    int d = 0;
    check(dwdp_prefetch_query(ctx_, h, &d));
    return d != 0;
  }
  void layer_forward(std::int64_t g, const void* x, std::int64_t T, void* y, bool residual,
                     void* stream) {
    check(dwdp_layer_forward(ctx_, g, x, T, y, residual ? 1 : 0, stream));
  }
  void stack_forward(const void* x, std::int64_t T, void* y, void* stream) {
    check(dwdp_stack_forward(ctx_, x, T, y, stream));
  }

 private:
  dwdp_ctx* ctx_ = nullptr;
};

}  // namespace dwdpsim_b200
