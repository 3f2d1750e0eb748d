// dwdp.hpp — header-only C++ adapter over the C-ABI (dwdp.h) with the
// reference operator API of the DWDP path: namespace `dwdpsim`, the value
// types, names, argument meaning and exception behaviour of
// /root/reference/proj/include/dwdpsim/{errors,rng,hwmodel,modelspec,
// placement,copyplan,workload,simcore}.hpp. include/dwdpsim/<name>.hpp
// forward here, so code written against the reference (its unit tests
// included: tests/test_reference_unit_tests.py) compiles unchanged with
// `-I include` and links libdwdp.so. What the adapter does NOT carry is the
// reference's discrete-event simulator (CopyEngineSim, simulate_dwdp,
// simulate_dep): on B200 those are the real engine (dwdpsim::Engine below,
// the dwdp_ctx runtime) measured with CUDA events. See INTEGRATION.md.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dwdp.h"

namespace dwdpsim {

// ===================================================================== errors.hpp:11-28
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class InvariantViolation : public std::logic_error {
 public:
  explicit InvariantViolation(const std::string& m) : std::logic_error(m) {}
};
// Status 4 of the C-ABI (CUDA / driver failure); no reference counterpart.
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
inline void require(bool cond, const std::string& msg) {
  if (!cond) throw ConfigError(msg);
}
inline void check_invariant(bool cond, const std::string& msg) {
  if (!cond) throw InvariantViolation(msg);
}
namespace detail {
inline void check(int st) {
  if (st == DWDP_OK) return;
  const std::string msg = dwdp_last_error();
  if (st == DWDP_ERR_CONFIG) throw ConfigError(msg);
  if (st == DWDP_ERR_INVARIANT) throw InvariantViolation(msg);
  throw CudaError(msg);
}
}  // namespace detail

// ===================================================================== rng.hpp:17-123
// Value-semantics generator: std::mt19937_64 (sequence fixed by the C++
// standard) with the transforms written out; mix() is the library's.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  static Rng forked(std::uint64_t seed, std::uint64_t salt) { return Rng(mix(seed, salt)); }
  std::uint64_t next_u64() { return engine_(); }
  double uniform01() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  std::uint64_t uniform_below(std::uint64_t n) {
    check_invariant(n > 0, "uniform_below: empty range");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
      const std::uint64_t x = engine_();
      if (x < limit) return x % n;
    }
  }
  bool bernoulli(double p) { return uniform01() < p; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double normal(double mean, double stddev) {
    double u1 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    const double u2 = uniform01();
    return mean + stddev * std::sqrt(-2.0 * std::log(u1)) *
                      std::cos(2.0 * 3.14159265358979323846 * u2);
  }
  static std::uint64_t mix(std::uint64_t a, std::uint64_t b) { return dwdp_rng_mix(a, b); }

 private:
  std::mt19937_64 engine_;
};

// Walker alias table; stacks filled in index order, LIFO pops (the
// library's route_tokens uses the same construction).
class AliasTable {
 public:
  explicit AliasTable(const std::vector<double>& w) {
    const std::size_t n = w.size();
    check_invariant(n > 0, "AliasTable: empty weights");
    double total = 0.0;
    for (double v : w) {
      check_invariant(v >= 0.0, "AliasTable: negative weight");
      total += v;
    }
    check_invariant(total > 0.0, "AliasTable: zero total weight");
    prob_.assign(n, 0.0);
    alias_.assign(n, 0);
    std::vector<double> sc(n);
    std::vector<std::uint32_t> lo, hi;
    for (std::size_t i = 0; i < n; ++i) {
      sc[i] = w[i] * static_cast<double>(n) / total;
      (sc[i] < 1.0 ? lo : hi).push_back(static_cast<std::uint32_t>(i));
    }
    while (!lo.empty() && !hi.empty()) {
      const std::uint32_t s = lo.back(), l = hi.back();
      lo.pop_back();
      prob_[s] = sc[s];
      alias_[s] = l;
      sc[l] -= 1.0 - sc[s];
      if (sc[l] < 1.0) {
        hi.pop_back();
        lo.push_back(l);
      }
    }
    for (std::uint32_t i : hi) prob_[i] = 1.0;
    for (std::uint32_t i : lo) prob_[i] = 1.0;
  }
  std::size_t sample(Rng& rng) const {
    const std::size_t i = static_cast<std::size_t>(rng.uniform_below(prob_.size()));
    return rng.uniform01() < prob_[i] ? i : alias_[i];
  }
  std::size_t size() const { return prob_.size(); }

 private:
  std::vector<double> prob_;
  std::vector<std::uint32_t> alias_;
};

// ===================================================================== hwmodel.hpp:14-53
enum class Category {
  Attention = DWDP_CAT_ATTENTION,
  GroupedGemm = DWDP_CAT_GROUPED_GEMM,
  DenseGemm = DWDP_CAT_DENSE_GEMM,
  Others = DWDP_CAT_OTHERS,
  Communication = DWDP_CAT_COMMUNICATION,
  D2DCopy = DWDP_CAT_D2D_COPY,
  P2PCopy = DWDP_CAT_P2P_COPY,
  SyncWait = DWDP_CAT_SYNC_WAIT,
};
inline const char* category_name(Category c) {
  const char* n = dwdp_category_name(static_cast<int>(c));
  return n ? n : "?";
}
inline Category category_from_name(const std::string& name) {
  for (int c = 0; c < DWDP_NUM_CATEGORIES; ++c)
    if (name == dwdp_category_name(c)) return static_cast<Category>(c);
  throw ConfigError("unknown category name: " + name);
}

struct GpuSpec {
  double peak_flops = 5e15;
  double mem_bw = 8e12;
  double link_bw = 1.8e12;
  int ce_inflight = 2;
  double tdp = 1.0;
  double idle_power_frac = 0.129;
  void validate() const {
    require(peak_flops > 0, "gpu.peak_flops must be > 0");
    require(mem_bw > 0, "gpu.mem_bw must be > 0");
    require(link_bw > 0, "gpu.link_bw must be > 0");
    require(ce_inflight >= 1, "gpu.ce_inflight must be >= 1");
    require(tdp > 0, "gpu.tdp must be > 0");
    require(idle_power_frac >= 0 && idle_power_frac < 1,
            "gpu.idle_power_frac must be in [0, 1)");
  }
  dwdp_gpu_spec c() const { return {peak_flops, mem_bw, link_bw}; }
};

inline double roofline_time(double flops, double bytes, const GpuSpec& gpu) {
  const dwdp_gpu_spec g = gpu.c();
  double s = 0;
  detail::check(dwdp_roofline_time(flops, bytes, &g, &s));
  return s;
}

// ===================================================================== modelspec.hpp:13-75
struct CostCalibration {
  double attention = 1.0;
  double grouped_gemm = 1.0;
  double dense_gemm = 1.0;
};

struct MoeModelSpec {
  int num_layers = 1;
  std::int64_t hidden_dim = 0;
  int num_experts = 1;
  int top_k = 1;
  std::int64_t expert_ffn_dim = 0;
  std::int64_t shared_ffn_dim = 0;
  double attn_proj_params = 0;
  double weight_bytes_per_param = 2.0;
  double kv_bytes_per_token_per_layer = 0.0;
  double act_bytes_per_element = 2.0;
  double others_bytes_factor = 0.0;
  CostCalibration calib;

  dwdp_model_spec c() const {
    dwdp_model_spec m{};
    m.num_layers = num_layers;
    m.num_experts = num_experts;
    m.hidden_dim = hidden_dim;
    m.top_k = top_k;
    m.expert_ffn_dim = expert_ffn_dim;
    m.shared_ffn_dim = shared_ffn_dim;
    m.weight_bytes_per_param = weight_bytes_per_param;
    m.act_bytes_per_element = act_bytes_per_element;
    m.attn_proj_params = attn_proj_params;
    m.kv_bytes_per_token_per_layer = kv_bytes_per_token_per_layer;
    m.others_bytes_factor = others_bytes_factor;
    m.calib_attention = calib.attention;
    m.calib_grouped_gemm = calib.grouped_gemm;
    m.calib_dense_gemm = calib.dense_gemm;
    return m;
  }
  void validate() const {
    const dwdp_model_spec m = c();
    detail::check(dwdp_model_validate(&m));
  }
};

struct OpCost {
  Category category;
  double flops = 0;
  double bytes = 0;
};

struct LayerWork {
  std::vector<OpCost> attn;
  std::vector<OpCost> moe;
  double total_time(const GpuSpec& gpu) const {
    double t = 0;
    for (const auto& op : attn) t += roofline_time(op.flops, op.bytes, gpu);
    for (const auto& op : moe) t += roofline_time(op.flops, op.bytes, gpu);
    return t;
  }
};

namespace detail {
inline std::vector<OpCost> costs(const dwdp_op_cost* a, int n) {
  std::vector<OpCost> out;
  for (int i = 0; i < n; ++i)
    out.push_back({static_cast<Category>(a[i].category), a[i].flops, a[i].bytes});
  return out;
}
}  // namespace detail

inline double expert_shard_bytes(const MoeModelSpec& model) {
  const dwdp_model_spec m = model.c();
  double b = 0;
  detail::check(dwdp_expert_shard_bytes(&m, &b));
  return b;
}

inline std::vector<OpCost> attention_entries(const MoeModelSpec& model, double tokens,
                                             double mean_seq_len) {
  const dwdp_model_spec m = model.c();
  dwdp_op_cost out[2];
  int n = 0;
  detail::check(dwdp_attention_entries(&m, tokens, mean_seq_len, out, &n));
  return detail::costs(out, n);
}

inline std::vector<OpCost> moe_entries(const MoeModelSpec& model, double tokens,
                                       double routed_pairs, int experts_touched) {
  const dwdp_model_spec m = model.c();
  dwdp_op_cost out[3];
  int n = 0;
  detail::check(dwdp_moe_entries(&m, tokens, routed_pairs, experts_touched, out, &n));
  return detail::costs(out, n);
}

inline LayerWork layer_costs(const MoeModelSpec& model, std::int64_t tokens,
                             std::int64_t mean_seq_len) {
  const dwdp_model_spec m = model.c();
  dwdp_op_cost a[2], b[3];
  int na = 0, nb = 0;
  detail::check(dwdp_layer_costs(&m, tokens, mean_seq_len, a, &na, b, &nb));
  return {detail::costs(a, na), detail::costs(b, nb)};
}

// ===================================================================== placement.hpp:13-43
struct PlacementPlan {
  int group_size = 0;
  int num_experts = 0;
  int local_count = 0;
  int redundancy = 0;
  std::vector<std::vector<int>> local_sets;
  std::vector<std::vector<std::pair<int, int>>> fetch_lists;

  bool holds(int rank, int expert) const {
    const auto& s = local_sets.at(static_cast<std::size_t>(rank));
    for (int e : s)
      if (e == expert) return true;
    return false;
  }
  // Checks this value's tables in the library (src/placement.cpp:15-45).
  void validate() const;
};

namespace detail {
// Library handle over a plan: built from parameters, or from a value's own
// tables (validated on the way in).
struct PlacementHandle {
  dwdp_placement* p = nullptr;
  PlacementHandle(int E, int N, int extra) { check(dwdp_placement_build(E, N, extra, &p)); }
  explicit PlacementHandle(const PlacementPlan& v) {
    check_invariant(static_cast<int>(v.local_sets.size()) == v.group_size,
                    "placement: local_sets size mismatch");
    check_invariant(static_cast<int>(v.fetch_lists.size()) == v.group_size,
                    "placement: fetch_lists size mismatch");
    std::vector<int> lo{0}, lf, fo{0}, fe, fs;
    for (const auto& s : v.local_sets) {
      lf.insert(lf.end(), s.begin(), s.end());
      lo.push_back(static_cast<int>(lf.size()));
    }
    for (const auto& f : v.fetch_lists) {
      for (const auto& [e, src] : f) {
        fe.push_back(e);
        fs.push_back(src);
      }
      fo.push_back(static_cast<int>(fe.size()));
    }
    lf.push_back(0);
    fe.push_back(0);
    fs.push_back(0);
    check(dwdp_placement_from_tables(v.group_size, v.num_experts, v.local_count, v.redundancy,
                                     lo.data(), lf.data(), fo.data(), fe.data(), fs.data(), &p));
  }
  ~PlacementHandle() { dwdp_placement_free(p); }
  PlacementHandle(const PlacementHandle&) = delete;
  PlacementHandle& operator=(const PlacementHandle&) = delete;
};
}  // namespace detail

inline void PlacementPlan::validate() const { detail::PlacementHandle h(*this); }

inline PlacementPlan build_placement(int num_experts, int group_size, int extra_redundancy = 0) {
  detail::PlacementHandle h(num_experts, group_size, extra_redundancy);
  PlacementPlan out;
  detail::check(dwdp_placement_info(h.p, &out.group_size, &out.num_experts, &out.local_count,
                                    &out.redundancy));
  for (int r = 0; r < out.group_size; ++r) {
    std::vector<int> ls(static_cast<std::size_t>(out.local_count) + 1);
    detail::check(dwdp_placement_local_set(h.p, r, ls.data()));
    ls.resize(static_cast<std::size_t>(out.local_count));
    const std::size_t m = static_cast<std::size_t>(out.num_experts - out.local_count);
    std::vector<int> fe(m + 1), fs(m + 1);
    detail::check(dwdp_placement_fetch_list(h.p, r, fe.data(), fs.data()));
    std::vector<std::pair<int, int>> fl;
    for (std::size_t i = 0; i < m; ++i) fl.emplace_back(fe[i], fs[i]);
    out.local_sets.push_back(std::move(ls));
    out.fetch_lists.push_back(std::move(fl));
  }
  return out;
}

inline std::vector<std::vector<std::pair<int, int>>> assign_fetch_sources(
    int num_experts, const std::vector<std::vector<int>>& local_sets) {
  const int n = static_cast<int>(local_sets.size());
  std::vector<int> offs{0}, flat;
  for (const auto& s : local_sets) {
    flat.insert(flat.end(), s.begin(), s.end());
    offs.push_back(static_cast<int>(flat.size()));
  }
  flat.push_back(0);
  const std::size_t cap = static_cast<std::size_t>(n) * static_cast<std::size_t>(num_experts) + 1;
  std::vector<int> counts(static_cast<std::size_t>(n) + 1), fe(cap), fs(cap);
  detail::check(dwdp_assign_fetch_sources(num_experts, n, offs.data(), flat.data(), counts.data(),
                                          fe.data(), fs.data()));
  std::vector<std::vector<std::pair<int, int>>> out(static_cast<std::size_t>(n));
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < counts[static_cast<std::size_t>(r)]; ++i) {
      const std::size_t k = static_cast<std::size_t>(r) * static_cast<std::size_t>(num_experts) +
                            static_cast<std::size_t>(i);
      out[static_cast<std::size_t>(r)].emplace_back(fe[k], fs[k]);
    }
  return out;
}

inline double prefetch_bytes(const PlacementPlan& plan, const MoeModelSpec& model) {
  return static_cast<double>(plan.num_experts - plan.local_count) * expert_shard_bytes(model);
}

inline std::string describe_placement(const PlacementPlan& plan) {
  detail::PlacementHandle h(plan);
  std::size_t len = 0;
  detail::check(dwdp_placement_describe(h.p, nullptr, &len));
  std::string s(len, '\0');
  detail::check(dwdp_placement_describe(h.p, &s[0], &len));
  s.resize(len - 1);
  return s;
}

// ===================================================================== copyplan.hpp:15-51
struct ShardRef {
  int peer = 0;
  std::uint64_t param_id = 0;
  std::uint64_t size = 0;
  std::uint64_t src_offset = 0;
};

struct Slice {
  std::uint64_t param_id = 0;
  int src_rank = 0;
  std::uint64_t src_offset = 0;
  std::uint64_t dst_offset = 0;
  std::uint64_t length = 0;
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
  std::string to_csv() const {  // src/copyplan.cpp:15-23
    std::string out = "param_id,src_rank,src_offset,dst_offset,length\n";
    for (const auto& s : slices)
      out += std::to_string(s.param_id) + "," + std::to_string(s.src_rank) + "," +
             std::to_string(s.src_offset) + "," + std::to_string(s.dst_offset) + "," +
             std::to_string(s.length) + "\n";
    return out;
  }
};

namespace detail {
inline dwdp_slice to_c(const Slice& s) {
  return {s.param_id, s.src_rank, 0, s.src_offset, s.dst_offset, s.length};
}
inline Slice from_c(const dwdp_slice& s) {
  return {s.param_id, s.src_rank, s.src_offset, s.dst_offset, s.length};
}
}  // namespace detail

inline CopyPlan build_copy_plan(const std::vector<ShardRef>& shards, std::uint64_t slice_size,
                                int dst_rank = 0) {
  std::vector<dwdp_shard_ref> in;
  for (const auto& s : shards) in.push_back({s.peer, 0, s.param_id, s.size, s.src_offset});
  std::size_t n = 0;
  detail::check(dwdp_copy_plan_build(in.data(), in.size(), slice_size, dst_rank, nullptr, &n));
  std::vector<dwdp_slice> out(n + 1);
  detail::check(dwdp_copy_plan_build(in.data(), in.size(), slice_size, dst_rank, out.data(), &n));
  CopyPlan plan;
  plan.dst_rank = dst_rank;
  plan.slice_size = slice_size;
  for (std::size_t i = 0; i < n; ++i) plan.slices.push_back(detail::from_c(out[i]));
  return plan;
}

inline std::map<int, std::vector<Slice>> source_queues(const std::vector<CopyPlan>& plans,
                                                       int source) {
  std::vector<std::vector<dwdp_slice>> cs;
  std::vector<const dwdp_slice*> ptrs;
  std::vector<std::size_t> lens;
  std::vector<int> dsts;
  for (const auto& p : plans) {
    std::vector<dwdp_slice> v;
    for (const auto& s : p.slices) v.push_back(detail::to_c(s));
    v.push_back({});
    cs.push_back(std::move(v));
    dsts.push_back(p.dst_rank);
    lens.push_back(p.slices.size());
  }
  for (const auto& v : cs) ptrs.push_back(v.data());
  std::size_t nq = 0, n = 0;
  detail::check(dwdp_source_queues(plans.size(), dsts.data(), ptrs.data(), lens.data(), source,
                                   nullptr, nullptr, &nq, nullptr, &n));
  std::vector<int> qd(nq + 1);
  std::vector<std::size_t> qc(nq + 1);
  std::vector<dwdp_slice> out(n + 1);
  detail::check(dwdp_source_queues(plans.size(), dsts.data(), ptrs.data(), lens.data(), source,
                                   qd.data(), qc.data(), &nq, out.data(), &n));
  std::map<int, std::vector<Slice>> q;
  std::size_t at = 0;
  for (std::size_t k = 0; k < nq; ++k) {
    auto& v = q[qd[k]];
    for (std::size_t i = 0; i < qc[k]; ++i) v.push_back(detail::from_c(out[at++]));
  }
  return q;
}

// ===================================================================== workload.hpp:14-79
struct IslDist {
  enum class Kind { Fixed = DWDP_ISL_FIXED, UniformRatio = DWDP_ISL_UNIFORM_RATIO,
                    Normal = DWDP_ISL_NORMAL };
  Kind kind = Kind::Fixed;
  double length = 8192;
  double ratio = 1.0;
  double stddev = 0.0;

  void validate() const {  // src/workload.cpp:10-22
    require(length >= 1, "workload.isl: length/mean must be >= 1");
    if (kind == Kind::UniformRatio)
      require(ratio > 0 && ratio <= 1, "workload.isl: ratio must be in (0, 1]");
    if (kind == Kind::Normal) require(stddev >= 0, "workload.isl: stddev must be >= 0");
  }
  double cv() const {
    dwdp_workload_spec w{};
    w.isl_kind = static_cast<std::int32_t>(kind);
    w.length = length;
    w.ratio = ratio;
    w.stddev = stddev;
    double v = 0;
    detail::check(dwdp_isl_cv(&w, &v));
    return v;
  }
  static IslDist fixed(double length) {
    IslDist d;
    d.length = length;
    return d;
  }
  static IslDist uniform_ratio(double max_length, double ratio) {
    IslDist d;
    d.kind = Kind::UniformRatio;
    d.length = max_length;
    d.ratio = ratio;
    return d;
  }
  static IslDist normal(double mean, double stddev) {
    IslDist d;
    d.kind = Kind::Normal;
    d.length = mean;
    d.stddev = stddev;
    return d;
  }
  static IslDist from_cv(double mean, double cv) {
    require(cv >= 0, "workload.isl: cv must be >= 0");
    return cv == 0.0 ? fixed(mean) : normal(mean, cv * mean);
  }
};

struct WorkloadSpec {
  IslDist isl_dist;
  std::int64_t max_num_tokens = 32768;
  int batch_per_rank = 1;
  double routing_skew = 0.0;
  std::uint64_t seed = 1;

  dwdp_workload_spec c() const {
    dwdp_workload_spec w{};
    w.isl_kind = static_cast<std::int32_t>(isl_dist.kind);
    w.batch_per_rank = batch_per_rank;
    w.length = isl_dist.length;
    w.ratio = isl_dist.ratio;
    w.stddev = isl_dist.stddev;
    w.max_num_tokens = max_num_tokens;
    w.routing_skew = routing_skew;
    w.seed = seed;
    return w;
  }
  void validate() const {
    const dwdp_workload_spec w = c();
    detail::check(dwdp_workload_validate(&w));
  }
};

struct RankBatch {
  std::vector<std::int64_t> tokens;
  std::vector<std::int64_t> requests;
  std::vector<std::vector<std::int64_t>> routed;
  std::int64_t mean_seq_len(int rank) const {
    const auto r = static_cast<std::size_t>(rank);
    if (requests[r] <= 0) return tokens[r];
    return std::max<std::int64_t>(1, tokens[r] / requests[r]);
  }
};

inline std::vector<std::int64_t> route_tokens(std::int64_t tokens, const MoeModelSpec& model,
                                              double routing_skew, std::uint64_t seed) {
  model.validate();
  std::vector<std::int64_t> counts(static_cast<std::size_t>(model.num_experts));
  detail::check(dwdp_route_tokens(tokens, model.num_experts, model.top_k, routing_skew, seed,
                                  counts.data()));
  return counts;
}

inline std::vector<RankBatch> sample_batches(const WorkloadSpec& spec, const MoeModelSpec& model,
                                             int num_ranks, int iterations) {
  spec.validate();
  model.validate();
  require(num_ranks >= 1, "sample_batches: num_ranks must be >= 1");
  require(iterations >= 1, "sample_batches: iterations must be >= 1");
  const dwdp_workload_spec w = spec.c();
  const std::size_t n = static_cast<std::size_t>(num_ranks) * static_cast<std::size_t>(iterations);
  const std::size_t E = static_cast<std::size_t>(model.num_experts);
  std::vector<std::int64_t> t(n), q(n), r(n * E);
  detail::check(dwdp_sample_batches(&w, model.num_experts, model.top_k, num_ranks, iterations,
                                    t.data(), q.data(), r.data()));
  std::vector<RankBatch> out(static_cast<std::size_t>(iterations));
  for (std::size_t it = 0; it < out.size(); ++it)
    for (std::size_t k = 0; k < static_cast<std::size_t>(num_ranks); ++k) {
      const std::size_t i = it * static_cast<std::size_t>(num_ranks) + k;
      out[it].tokens.push_back(t[i]);
      out[it].requests.push_back(q[i]);
      out[it].routed.emplace_back(r.begin() + static_cast<std::ptrdiff_t>(i * E),
                                  r.begin() + static_cast<std::ptrdiff_t>((i + 1) * E));
    }
  return out;
}

inline double imbalance_cv(const RankBatch& batch) {
  double v = 0;
  detail::check(dwdp_imbalance_cv(batch.tokens.data(), static_cast<int>(batch.tokens.size()), &v));
  return v;
}

inline std::string batches_to_csv(const std::vector<RankBatch>& batches) {
  const int iters = static_cast<int>(batches.size());
  const int N = iters ? static_cast<int>(batches[0].tokens.size()) : 0;
  int E = 0;
  bool uniform = true;
  for (const auto& b : batches) {
    require(static_cast<int>(b.tokens.size()) == N && static_cast<int>(b.requests.size()) == N,
            "batches csv: ragged rank count");
    for (const auto& c : b.routed) {
      if (E == 0) E = static_cast<int>(c.size());
      uniform = uniform && static_cast<int>(c.size()) == E;
    }
    uniform = uniform && (b.routed.empty() || static_cast<int>(b.routed.size()) == N);
  }
  require(uniform, "batches csv: ragged expert counts");
  std::vector<std::int64_t> t, q, r;
  for (const auto& b : batches) {
    t.insert(t.end(), b.tokens.begin(), b.tokens.end());
    q.insert(q.end(), b.requests.begin(), b.requests.end());
    for (const auto& c : b.routed) r.insert(r.end(), c.begin(), c.end());
  }
  t.push_back(0);
  q.push_back(0);
  const std::int64_t* rp = E > 0 ? r.data() : nullptr;
  std::size_t len = 0;
  detail::check(dwdp_batches_to_csv(t.data(), q.data(), rp, iters, N, E, nullptr, &len));
  std::string s(len, '\0');
  detail::check(dwdp_batches_to_csv(t.data(), q.data(), rp, iters, N, E, &s[0], &len));
  s.resize(len - 1);
  return s;
}

inline std::vector<RankBatch> batches_from_csv(const std::string& csv) {
  int iters = 0, N = 0, E = 0;
  detail::check(dwdp_batches_from_csv(csv.c_str(), &iters, &N, &E, nullptr, nullptr, nullptr,
                                      nullptr));
  const std::size_t n = static_cast<std::size_t>(iters) * static_cast<std::size_t>(N);
  std::vector<std::int64_t> t(n + 1), q(n + 1), r(n * static_cast<std::size_t>(E) + 1);
  std::vector<std::int32_t> len(n + 1);
  detail::check(dwdp_batches_from_csv(csv.c_str(), &iters, &N, &E, t.data(), q.data(), r.data(),
                                      len.data()));
  std::vector<RankBatch> out(static_cast<std::size_t>(iters));
  for (std::size_t it = 0; it < out.size(); ++it)
    for (std::size_t k = 0; k < static_cast<std::size_t>(N); ++k) {
      const std::size_t i = it * static_cast<std::size_t>(N) + k;
      out[it].tokens.push_back(t[i]);
      out[it].requests.push_back(q[i]);
      const auto b = r.begin() + static_cast<std::ptrdiff_t>(i * static_cast<std::size_t>(E));
      out[it].routed.emplace_back(b, b + len[i]);
    }
  return out;
}

// ===================================================================== simcore.hpp:19-229
using TimeNs = std::int64_t;
inline TimeNs to_ns(double seconds) { return static_cast<TimeNs>(std::llround(seconds * 1e9)); }

enum class Stream { Compute, CopyEngine };

struct SimEvent {
  int rank = 0;
  Stream stream = Stream::Compute;
  Category category = Category::Others;
  TimeNs start = 0;
  TimeNs end = 0;
  int layer = 0;
  int iteration = 0;
  double bytes = 0;
  std::string detail;
};

// A run's event list: the reference fills it from its simulator; here from
// the CUDA events of the real engine (dwdp_report_from_records / Engine).
struct RunReport {
  std::string strategy;
  int num_ranks = 0;
  int num_layers = 0;
  int iterations = 0;
  int warmup_iterations = 0;
  std::vector<SimEvent> events;
  std::vector<std::vector<TimeNs>> iter_start;
  std::vector<std::vector<TimeNs>> iter_end;
  std::vector<std::vector<std::int64_t>> iter_tokens;

  int steady_iterations() const { return iterations - warmup_iterations; }
  double mean_latency_us(int rank) const {
    double total = 0;
    int n = 0;
    for (int it = warmup_iterations; it < iterations; ++it, ++n)
      total += static_cast<double>(iter_end[static_cast<std::size_t>(rank)][static_cast<std::size_t>(it)] -
                                   iter_start[static_cast<std::size_t>(rank)][static_cast<std::size_t>(it)]);
    check_invariant(n > 0, "report: no steady iterations");
    return total / n / 1e3;
  }
  double mean_latency_us() const {
    double t = 0;
    for (int r = 0; r < num_ranks; ++r) t += mean_latency_us(r);
    return t / num_ranks;
  }
  double throughput_tokens_per_s() const;
  void validate_streams() const;
};

struct DwdpOptions {
  bool merge_elim = true;
  bool tdm = true;
  std::uint64_t slice_size = 1 << 20;
  bool model_contention = true;  // simulator-only knob; real links share themselves
  void validate() const {
    if (tdm) require(slice_size > 0, "dwdp.slice_size must be > 0 with tdm");
  }
};

struct BreakdownTable {
  std::map<Category, double> compute_us;
  std::map<Category, double> copy_us;
  double iteration_latency_us = 0;
  bool p2p_fully_overlapped = false;
  double tokens_per_s = 0;  // RunReport::throughput_tokens_per_s of the source run

  double category_us(Category c) const {
    const auto a = compute_us.find(c);
    if (a != compute_us.end()) return a->second;
    const auto b = copy_us.find(c);
    return b != copy_us.end() ? b->second : 0.0;
  }
  dwdp_breakdown c() const {
    dwdp_breakdown b{};
    for (const auto& [k, v] : compute_us) {
      b.compute_us[static_cast<int>(k)] = v;
      b.compute_present[static_cast<int>(k)] = 1;
    }
    for (const auto& [k, v] : copy_us) {
      b.copy_us[static_cast<int>(k)] = v;
      b.copy_present[static_cast<int>(k)] = 1;
    }
    b.iteration_latency_us = iteration_latency_us;
    b.p2p_fully_overlapped = p2p_fully_overlapped ? 1 : 0;
    b.tokens_per_s = tokens_per_s;
    return b;
  }
  static BreakdownTable from_c(const dwdp_breakdown& b) {
    BreakdownTable t;
    for (int k = 0; k < DWDP_NUM_CATEGORIES; ++k) {
      if (b.compute_present[k]) t.compute_us[static_cast<Category>(k)] = b.compute_us[k];
      if (b.copy_present[k]) t.copy_us[static_cast<Category>(k)] = b.copy_us[k];
    }
    t.iteration_latency_us = b.iteration_latency_us;
    t.p2p_fully_overlapped = b.p2p_fully_overlapped != 0;
    t.tokens_per_s = b.tokens_per_s;
    return t;
  }
  std::string to_csv() const {
    const dwdp_breakdown b = c();
    std::size_t len = 0;
    detail::check(dwdp_breakdown_csv(&b, nullptr, &len));
    std::string s(len, '\0');
    detail::check(dwdp_breakdown_csv(&b, &s[0], &len));
    s.resize(len - 1);
    return s;
  }
};

namespace detail {
inline int detail_code(const std::string& d) {
  if (d == "weight_wait") return DWDP_DETAIL_WEIGHT_WAIT;
  if (d == "dispatch") return DWDP_DETAIL_DISPATCH;
  if (d == "combine") return DWDP_DETAIL_COMBINE;
  if (d == "barrier") return DWDP_DETAIL_BARRIER;
  return DWDP_DETAIL_NONE;
}
inline dwdp_breakdown breakdown_c(const RunReport& rep) {
  std::vector<dwdp_sim_event> ev;
  for (const auto& e : rep.events)
    ev.push_back({e.rank, static_cast<std::int32_t>(e.stream), static_cast<std::int32_t>(e.category),
                  e.layer, e.iteration, detail_code(e.detail), e.start, e.end, e.bytes});
  std::vector<std::int64_t> is, ie, tk;
  for (int r = 0; r < rep.num_ranks; ++r)
    for (int it = 0; it < rep.iterations; ++it) {
      is.push_back(rep.iter_start.at(static_cast<std::size_t>(r)).at(static_cast<std::size_t>(it)));
      ie.push_back(rep.iter_end.at(static_cast<std::size_t>(r)).at(static_cast<std::size_t>(it)));
      tk.push_back(rep.iter_tokens.at(static_cast<std::size_t>(r)).at(static_cast<std::size_t>(it)));
    }
  ev.push_back({});
  is.push_back(0);
  ie.push_back(0);
  tk.push_back(0);
  dwdp_breakdown b{};
  check(dwdp_report_breakdown(ev.data(), ev.size() - 1, rep.num_ranks, rep.iterations,
                              rep.warmup_iterations, is.data(), ie.data(), tk.data(), &b));
  return b;
}
}  // namespace detail

inline double RunReport::throughput_tokens_per_s() const {
  return detail::breakdown_c(*this).tokens_per_s;
}
// dwdp_report_breakdown checks per-(rank, stream) overlap before accounting.
inline void RunReport::validate_streams() const { (void)detail::breakdown_c(*this); }

inline BreakdownTable breakdown(const RunReport& report) {
  return BreakdownTable::from_c(detail::breakdown_c(report));
}

struct ComparisonRow {
  Category category = Category::Others;
  double a_us = 0;
  double b_us = 0;
  std::optional<double> delta_frac;
};

struct ComparisonTable {
  std::vector<ComparisonRow> rows;
  double a_latency_us = 0;
  double b_latency_us = 0;
  double overall_frac = 0;
  double gross_sync_comm_pct = 0;
  dwdp_comparison raw{};

  std::string to_csv() const {
    std::size_t len = 0;
    detail::check(dwdp_comparison_csv(&raw, nullptr, &len));
    std::string s(len, '\0');
    detail::check(dwdp_comparison_csv(&raw, &s[0], &len));
    s.resize(len - 1);
    return s;
  }
};

inline ComparisonTable compare_reports(const BreakdownTable& a, const BreakdownTable& b) {
  const dwdp_breakdown ca = a.c(), cb = b.c();
  ComparisonTable t;
  detail::check(dwdp_compare_reports(&ca, &cb, &t.raw));
  for (int k = 0; k < DWDP_NUM_CATEGORIES; ++k) {
    ComparisonRow row;
    row.category = static_cast<Category>(k);
    row.a_us = t.raw.a_us[k];
    row.b_us = t.raw.b_us[k];
    if (t.raw.has_delta[k]) row.delta_frac = t.raw.delta_frac[k];
    t.rows.push_back(row);
  }
  t.a_latency_us = t.raw.a_latency_us;
  t.b_latency_us = t.raw.b_latency_us;
  t.overall_frac = t.raw.overall_frac;
  t.gross_sync_comm_pct = t.raw.gross_sync_comm_pct;
  return t;
}
inline ComparisonTable compare_reports(const RunReport& a, const RunReport& b) {
  return compare_reports(breakdown(a), breakdown(b));
}

struct AnalyticResult {
  double t_compute_s = 0;
  double t_prefetch_s = 0;
  double t_all2all_s = 0;
  double compute_prefetch_ratio = 0;
  double dep_dwdp_speedup = 0;
  bool prefetch_saturated = false;
};

// simcore.cpp:882-905; mean_seq_len == 0 selects the MoE block alone.
inline AnalyticResult analytic_compare(const MoeModelSpec& model, const GpuSpec& gpu,
                                       const PlacementPlan& placement, std::int64_t tokens,
                                       std::int64_t mean_seq_len) {
  if (mean_seq_len > 0) gpu.validate();
  const dwdp_model_spec m = model.c();
  const dwdp_gpu_spec g = gpu.c();
  detail::PlacementHandle h(placement);
  dwdp_analytic_result r{};
  detail::check(dwdp_analytic_compare(&m, &g, h.p, tokens, mean_seq_len, &r));
  return {r.t_compute_s, r.t_prefetch_s, r.t_all2all_s, r.compute_prefetch_ratio,
          r.dep_dwdp_speedup, r.prefetch_saturated != 0};
}

// ===================================================================== the real engine
// One GPU's DWDP runtime (dwdp_ctx): split-weight arenas, the prefetch engine
// behind the CopyEngineSim handle API (simcore.hpp:87-106), and the sm_100a
// MoE layer that simulate_dwdp's step loop (simcore.cpp:640-733) costs.
class Engine {
 public:
  explicit Engine(const dwdp_ctx_config& cfg) { detail::check(dwdp_ctx_create(&cfg, &ctx_)); }
  ~Engine() { dwdp_ctx_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  dwdp_ctx* get() const { return ctx_; }
  void init_weights(float bias_scale = 0.0f) {
    detail::check(dwdp_ctx_init_weights(ctx_, bias_scale));
  }
  static void link_local(const std::vector<Engine*>& group) {
    std::vector<dwdp_ctx*> c;
    for (auto* e : group) c.push_back(e->ctx_);
    detail::check(dwdp_ctx_link_local(c.data(), static_cast<int>(c.size())));
  }
  // CopyEngineSim::issue_plan / plan_done / plan_start_time /
  // plan_complete_time / plan_bytes; times in ns on the engine's clock.
  std::int64_t issue_plan(std::int64_t global_layer) {
    dwdp_prefetch h = -1;
    detail::check(dwdp_prefetch_issue(ctx_, global_layer, &h));
    return h;
  }
  bool plan_done(std::int64_t h) {
    int d = 0;
    detail::check(dwdp_prefetch_query(ctx_, h, &d));
    return d != 0;
  }
  void plan_wait(std::int64_t h, void* stream) { detail::check(dwdp_prefetch_wait(ctx_, h, stream)); }
  TimeNs plan_start_time(std::int64_t h) { return times(h).first; }
  TimeNs plan_complete_time(std::int64_t h) { return times(h).second; }
  double plan_bytes(std::int64_t h) {
    std::int64_t s = 0, e = 0;
    double b = 0;
    detail::check(dwdp_prefetch_times(ctx_, h, &s, &e, &b));
    return b;
  }
  void moe_forward(int layer, const void* x, std::int64_t T, void* y, void* stream) {
    detail::check(dwdp_moe_forward(ctx_, layer, x, T, y, stream));
  }
  void layer_forward(std::int64_t g, const void* x, std::int64_t T, void* y, bool residual,
                     void* stream) {
    detail::check(dwdp_layer_forward(ctx_, g, x, T, y, residual ? 1 : 0, stream));
  }
  void stack_forward(const void* x, std::int64_t T, void* y, void* stream) {
    detail::check(dwdp_stack_forward(ctx_, x, T, y, stream));
  }

 private:
  std::pair<TimeNs, TimeNs> times(std::int64_t h) {
    std::int64_t s = 0, e = 0;
    double b = 0;
    detail::check(dwdp_prefetch_times(ctx_, h, &s, &e, &b));
    return {s, e};
  }
  dwdp_ctx* ctx_ = nullptr;
};

}  // namespace dwdpsim

// Round-1 name of this adapter's namespace.
namespace dwdpsim_b200 = dwdpsim;
