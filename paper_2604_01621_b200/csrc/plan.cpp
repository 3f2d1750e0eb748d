// Host planners of the DWDP hot path. See plan.hpp; reference semantics
// cited per function (paths under /root/reference/proj).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <numeric>
#include <set>
#include <sstream>
#include <tuple>

namespace dwdp {

// ===================================================================== //
// Placement — src/placement.cpp:10-150.
//
// A rank's block is the arc [r*stride, r*stride + c) of the expert ring;
// membership is kept as a bitmap so holder lookups are O(1).

bool Placement::holds(int rank, int expert) const {
  const auto& s = local_sets.at(static_cast<size_t>(rank));
  return std::binary_search(s.begin(), s.end(), expert);
}

void Placement::validate() const {
  invariant(static_cast<int>(local_sets.size()) == group_size &&
                static_cast<int>(fetch_lists.size()) == group_size,
            "placement: table shape mismatch");
  std::vector<int> copies(static_cast<size_t>(num_experts), 0);
  for (int r = 0; r < group_size; ++r) {
    const auto& loc = local_sets[static_cast<size_t>(r)];
    invariant(static_cast<int>(loc.size()) == local_count,
              "placement: unequal local counts");
    std::vector<char> covered(static_cast<size_t>(num_experts), 0);
    for (int e : loc) {
      invariant(e >= 0 && e < num_experts, "placement: expert out of range");
      ++copies[static_cast<size_t>(e)];
      covered[static_cast<size_t>(e)] = 1;
    }
    for (const auto& [e, src] : fetch_lists[static_cast<size_t>(r)]) {
      invariant(e >= 0 && e < num_experts, "placement: expert out of range");
      invariant(!covered[static_cast<size_t>(e)], "placement: fetched expert is local");
      invariant(src != r, "placement: self-fetch");
      invariant(src >= 0 && src < group_size, "placement: source does not hold expert");
      invariant(holds(src, e), "placement: source does not hold expert");
      covered[static_cast<size_t>(e)] = 1;
    }
    invariant(std::all_of(covered.begin(), covered.end(), [](char c) { return c != 0; }),
              "placement: rank does not cover all experts");
  }
  int surplus = 0;
  for (int n : copies) {
    invariant(n >= 1, "placement: expert not stored anywhere");
    surplus += n - 1;
  }
  invariant(surplus == redundancy, "placement: redundancy miscount");
}

std::vector<std::vector<std::pair<int, int>>> assign_fetch_sources(
    int num_experts, const std::vector<std::vector<int>>& local_sets) {
  const int n = static_cast<int>(local_sets.size());
  // holder bitmap [expert][rank]
  std::vector<char> holder(static_cast<size_t>(num_experts) * static_cast<size_t>(n), 0);
  for (int r = 0; r < n; ++r)
    for (int e : local_sets[static_cast<size_t>(r)])
      holder[static_cast<size_t>(e) * static_cast<size_t>(n) + static_cast<size_t>(r)] = 1;
  std::vector<std::vector<std::pair<int, int>>> out(static_cast<size_t>(n));
  for (int dst = 0; dst < n; ++dst) {
    std::vector<int> pulled(static_cast<size_t>(n), 0);
    const char* mine = nullptr;
    for (int e = 0; e < num_experts; ++e) {
      const char* row = &holder[static_cast<size_t>(e) * static_cast<size_t>(n)];
      mine = row + dst;
      if (*mine) continue;
      // least-loaded holder, first (lowest rank) on ties
      int pick = -1;
      for (int h = 0; h < n; ++h)
        if (row[h] && h != dst && (pick < 0 || pulled[static_cast<size_t>(h)] <
                                                   pulled[static_cast<size_t>(pick)]))
          pick = h;
      invariant(pick >= 0, "assign_fetch_sources: uncovered expert");
      ++pulled[static_cast<size_t>(pick)];
      out[static_cast<size_t>(dst)].emplace_back(e, pick);
    }
  }
  return out;
}

Placement build_placement(int num_experts, int group_size, int extra) {
  require(group_size >= 2, "placement: group_size must be >= 2");
  require(num_experts >= group_size, "placement: num_experts must be >= group_size");
  require(extra >= 0, "placement: extra_redundancy must be >= 0");
  Placement p;
  p.group_size = group_size;
  p.num_experts = num_experts;
  p.local_count = std::min((num_experts + group_size - 1) / group_size + extra, num_experts);
  p.redundancy = group_size * p.local_count - num_experts;
  // Ring arcs start every floor(E/N) experts; if that leaves a gap before
  // the ring closes, arcs start every c experts instead (placement.cpp:89-94).
  const int floor_stride = num_experts / group_size;
  const int stride =
      (group_size - 1) * floor_stride + p.local_count < num_experts ? p.local_count : floor_stride;
  p.local_sets.resize(static_cast<size_t>(group_size));
  for (int r = 0; r < group_size; ++r) {
    std::vector<char> in(static_cast<size_t>(num_experts), 0);
    for (int i = 0; i < p.local_count; ++i)
      in[static_cast<size_t>((r * stride + i) % num_experts)] = 1;
    for (int e = 0; e < num_experts; ++e)
      if (in[static_cast<size_t>(e)]) p.local_sets[static_cast<size_t>(r)].push_back(e);
  }
  p.fetch_lists = assign_fetch_sources(num_experts, p.local_sets);
  p.validate();
  return p;
}

std::string Placement::describe() const {
  std::ostringstream os;
  os << "placement: " << num_experts << " experts over " << group_size << " ranks, "
     << local_count << " local each, redundancy " << redundancy << "\n";
  for (int r = 0; r < group_size; ++r) {
    os << "  rank " << r << ": experts ";
    const auto& s = local_sets[static_cast<size_t>(r)];
    bool first = true;
    for (size_t i = 0; i < s.size();) {
      size_t j = i;
      while (j + 1 < s.size() && s[j + 1] == s[j] + 1) ++j;
      os << (first ? "" : ",") << s[i];
      if (j > i) os << "-" << s[j];
      first = false;
      i = j + 1;
    }
    std::map<int, int> per_src;
    for (const auto& f : fetch_lists[static_cast<size_t>(r)]) ++per_src[f.second];
    os << "; fetches";
    if (per_src.empty()) os << " nothing";
    bool any = false;
    for (const auto& [src, n] : per_src) {
      os << (any ? ", " : " ") << n << " from rank " << src;
      any = true;
    }
    os << "\n";
  }
  return os.str();
}

// ===================================================================== //
// TDM copy plan — src/copyplan.cpp:25-80 (paper Listing 1).
//
// Every shard is cut into ceil(size/s) slices; the schedule is the sort of
// all slices by (param first-appearance rank, offset, rotated peer rank),
// which is the order the reference's params -> offsets -> peers loop nest
// visits them in.

std::vector<Slice> build_copy_plan(const std::vector<ShardRef>& shards,
                                   uint64_t slice_size, int dst_rank) {
  require(slice_size > 0, "copy plan: slice_size must be > 0");
  std::set<std::pair<int, uint64_t>> seen;
  for (const auto& sh : shards) {
    require(sh.size > 0, "copy plan: shard size must be > 0");
    require(sh.peer != dst_rank, "copy plan: shard hosted on destination");
    require(seen.insert({sh.peer, sh.param_id}).second,
            "copy plan: duplicate (peer, param) shard");
  }
  std::vector<uint64_t> param_order;
  std::vector<int> peers;
  for (const auto& sh : shards) {
    if (std::find(param_order.begin(), param_order.end(), sh.param_id) == param_order.end())
      param_order.push_back(sh.param_id);
    peers.push_back(sh.peer);
  }
  std::sort(peers.begin(), peers.end());
  peers.erase(std::unique(peers.begin(), peers.end()), peers.end());
  if (peers.empty()) return {};
  const size_t phase = static_cast<size_t>(dst_rank) % peers.size();
  auto peer_rank = [&](int peer) {  // position after rotating left by phase
    const size_t pos = static_cast<size_t>(
        std::lower_bound(peers.begin(), peers.end(), peer) - peers.begin());
    return (pos + peers.size() - phase) % peers.size();
  };
  auto param_rank = [&](uint64_t p) {
    return static_cast<size_t>(std::find(param_order.begin(), param_order.end(), p) -
                               param_order.begin());
  };
  using Key = std::tuple<size_t, uint64_t, size_t>;
  std::vector<std::pair<Key, Slice>> all;
  for (const auto& sh : shards) {
    const size_t pr = param_rank(sh.param_id), qr = peer_rank(sh.peer);
    for (uint64_t off = 0; off < sh.size; off += slice_size)
      all.push_back({Key{pr, off, qr},
                     Slice{sh.param_id, sh.peer, sh.src_offset + off, off,
                           std::min(slice_size, sh.size - off)}});
  }
  std::sort(all.begin(), all.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<Slice> plan;
  plan.reserve(all.size());
  for (auto& kv : all) plan.push_back(kv.second);
  return plan;
}

// ===================================================================== //
// RNG + workload — include/dwdpsim/rng.hpp:17-123, src/workload.cpp.

uint64_t Rng::mix(uint64_t a, uint64_t b) {  // splitmix64 finalizer
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t Rng::below(uint64_t n) {
  invariant(n > 0, "uniform_below: empty range");
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  for (;;) {
    const uint64_t x = g_();
    if (x < limit) return x % n;
  }
}

double Rng::normal(double mean, double sd) {
  double u1;
  do {
    u1 = u01();
  } while (u1 <= 0.0);
  const double u2 = u01();
  const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  return mean + sd * z;
}

void WorkloadSpec::validate() const {
  require(length >= 1, "workload.isl: length/mean must be >= 1");
  if (isl_kind == 1) require(ratio > 0 && ratio <= 1, "workload.isl: ratio must be in (0, 1]");
  if (isl_kind == 2) require(stddev >= 0, "workload.isl: stddev must be >= 0");
  require(isl_kind >= 0 && isl_kind <= 2, "workload.isl: unknown kind");
  require(batch_per_rank >= 1, "workload.batch_per_rank must be >= 1");
  require(routing_skew >= 0, "workload.routing_skew must be >= 0");
  require(max_num_tokens >= static_cast<int64_t>(length),
          "workload.max_num_tokens smaller than the smallest request");
}

double WorkloadSpec::cv() const {
  if (isl_kind == 1) return (1.0 - ratio) / ((1.0 + ratio) * std::sqrt(3.0));
  if (isl_kind == 2) return stddev / length;
  return 0.0;
}

namespace {
// Walker alias sampler; table built with the reference's LIFO stacks so the
// sampled sequence matches bit-for-bit (rng.hpp:77-123).
struct Alias {
  std::vector<double> prob;
  std::vector<uint32_t> alt;
  explicit Alias(const std::vector<double>& w) : prob(w.size(), 0.0), alt(w.size(), 0) {
    const double total = std::accumulate(w.begin(), w.end(), 0.0);
    const double n = static_cast<double>(w.size());
    std::vector<double> sc(w.size());
    std::vector<uint32_t> lo, hi;
    for (size_t i = 0; i < w.size(); ++i) {
      sc[i] = w[i] * n / total;
      (sc[i] < 1.0 ? lo : hi).push_back(static_cast<uint32_t>(i));
    }
    while (!lo.empty() && !hi.empty()) {
      const uint32_t s = lo.back();
      lo.pop_back();
      const uint32_t l = hi.back();
      prob[s] = sc[s];
      alt[s] = l;
      sc[l] -= 1.0 - sc[s];
      if (sc[l] < 1.0) {
        hi.pop_back();
        lo.push_back(l);
      }
    }
    for (uint32_t i : hi) prob[i] = 1.0;
    for (uint32_t i : lo) prob[i] = 1.0;
  }
  size_t draw(Rng& r) const {
    const size_t i = static_cast<size_t>(r.below(prob.size()));
    return r.u01() < prob[i] ? i : alt[i];
  }
};
}  // namespace

std::vector<int64_t> route_tokens(int64_t tokens, int num_experts, int top_k,
                                  double skew, uint64_t seed) {
  require(num_experts >= 1 && top_k >= 1 && top_k <= num_experts,
          "model.top_k must be in [1, num_experts]");
  require(tokens >= 0, "route_tokens: negative tokens");
  std::vector<int64_t> counts(static_cast<size_t>(num_experts), 0);
  const int64_t pairs = tokens * top_k;
  if (pairs == 0) return counts;
  if (skew == 0.0) {
    for (int e = 0; e < num_experts; ++e)
      counts[static_cast<size_t>(e)] = pairs / num_experts + (e < pairs % num_experts ? 1 : 0);
    return counts;
  }
  std::vector<double> w(static_cast<size_t>(num_experts));
  for (int e = 0; e < num_experts; ++e) w[static_cast<size_t>(e)] = std::pow(e + 1.0, -skew);
  const Alias table(w);
  Rng rng(seed);
  for (int64_t a = 0; a < pairs; ++a) ++counts[table.draw(rng)];
  return counts;
}

Batches sample_batches(const WorkloadSpec& spec, int num_experts, int top_k,
                       int num_ranks, int iterations, bool with_routing) {
  spec.validate();
  require(num_ranks >= 1, "sample_batches: num_ranks must be >= 1");
  require(iterations >= 1, "sample_batches: iterations must be >= 1");
  Batches b;
  b.tokens.assign(static_cast<size_t>(iterations), std::vector<int64_t>(static_cast<size_t>(num_ranks)));
  b.requests = b.tokens;
  if (with_routing)
    b.routed.assign(static_cast<size_t>(iterations),
                    std::vector<std::vector<int64_t>>(static_cast<size_t>(num_ranks)));
  const double mnt = static_cast<double>(spec.max_num_tokens);
  for (int r = 0; r < num_ranks; ++r) {
    Rng rng(Rng::mix(spec.seed, 0x10000ULL + static_cast<uint64_t>(r)));
    std::deque<int64_t> backlog;
    for (int it = 0; it < iterations; ++it) {
      for (int q = 0; q < spec.batch_per_rank; ++q) {
        double len = spec.length;
        if (spec.isl_kind == 1)
          len = spec.ratio * spec.length + (spec.length - spec.ratio * spec.length) * rng.u01();
        else if (spec.isl_kind == 2)
          len = rng.normal(spec.length, spec.stddev);
        backlog.push_back(static_cast<int64_t>(std::llround(std::clamp(len, 1.0, mnt))));
      }
      int64_t used = 0, reqs = 0;
      for (; !backlog.empty() && used + backlog.front() <= spec.max_num_tokens; ++reqs) {
        used += backlog.front();
        backlog.pop_front();
      }
      b.tokens[static_cast<size_t>(it)][static_cast<size_t>(r)] = used;
      b.requests[static_cast<size_t>(it)][static_cast<size_t>(r)] = reqs;
      if (with_routing)
        b.routed[static_cast<size_t>(it)][static_cast<size_t>(r)] = route_tokens(
            used, num_experts, top_k, spec.routing_skew,
            Rng::mix(Rng::mix(spec.seed, 0x20000ULL + static_cast<uint64_t>(r)),
                     static_cast<uint64_t>(it)));
    }
  }
  return b;
}

double imbalance_cv(const std::vector<int64_t>& tokens) {
  require(tokens.size() >= 2, "imbalance_cv: need at least 2 ranks");
  const double n = static_cast<double>(tokens.size());
  double mean = 0;
  for (auto t : tokens) mean += static_cast<double>(t);
  mean /= n;
  require(mean != 0, "imbalance_cv: zero mean token count");
  double var = 0;
  for (auto t : tokens) var += (static_cast<double>(t) - mean) * (static_cast<double>(t) - mean);
  return std::sqrt(var / n) / mean;
}

// ===================================================================== //
// Batch CSV — src/workload.cpp:191-247 (same text format, so replay files
// interoperate with the reference's own batches_to_csv/batches_from_csv).

std::string batches_to_csv(const Batches& b) {
  std::ostringstream os;
  os << "iteration,rank,tokens,requests,expert_counts\n";
  for (size_t it = 0; it < b.tokens.size(); ++it)
    for (size_t r = 0; r < b.tokens[it].size(); ++r) {
      os << it << ',' << r << ',' << b.tokens[it][r] << ',' << b.requests[it][r] << ',';
      if (it < b.routed.size() && r < b.routed[it].size()) {
        const auto& c = b.routed[it][r];
        for (size_t e = 0; e < c.size(); ++e) os << (e ? ";" : "") << c[e];
      }
      os << '\n';
    }
  return os.str();
}

namespace {
int64_t parse_i64(const std::string& s, const char* what) {
  size_t used = 0;
  int64_t v = 0;
  try {
    v = std::stoll(s, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  require(used > 0 && used == s.size(), (std::string("batches csv: bad ") + what).c_str());
  return v;
}
}  // namespace

Batches batches_from_csv(const std::string& csv) {
  std::istringstream in(csv);
  std::string line;
  require(static_cast<bool>(std::getline(in, line)), "batches csv: empty file");
  require(line == "iteration,rank,tokens,requests,expert_counts", "batches csv: unexpected header");
  Batches b;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::vector<std::string> f;
    size_t pos = 0;
    for (int i = 0; i < 4; ++i) {
      const size_t c = line.find(',', pos);
      require(c != std::string::npos, "batches csv: missing field");
      f.push_back(line.substr(pos, c - pos));
      pos = c + 1;
    }
    const int64_t it = parse_i64(f[0], "iteration"), r = parse_i64(f[1], "rank");
    require(it >= 0 && r >= 0, "batches csv: negative index");
    std::vector<int64_t> counts;
    const std::string rest = line.substr(pos);
    for (size_t a = 0; a < rest.size();) {
      size_t e = rest.find(';', a);
      if (e == std::string::npos) e = rest.size();
      counts.push_back(parse_i64(rest.substr(a, e - a), "expert count"));
      a = e + 1;
    }
    const size_t I = size_t(it), R = size_t(r);
    if (b.tokens.size() <= I) {
      b.tokens.resize(I + 1);
      b.requests.resize(I + 1);
      b.routed.resize(I + 1);
    }
    if (b.tokens[I].size() <= R) {
      b.tokens[I].resize(R + 1, 0);
      b.requests[I].resize(R + 1, 0);
      b.routed[I].resize(R + 1);
    }
    b.tokens[I][R] = parse_i64(f[2], "tokens");
    b.requests[I][R] = parse_i64(f[3], "requests");
    b.routed[I][R] = std::move(counts);
  }
  require(!b.tokens.empty(), "batches csv: no rows");
  return b;
}

// ===================================================================== //
// Cost formulas — src/modelspec.cpp:6-98.

void ModelSpec::validate() const {
  require(num_layers >= 1, "model.num_layers must be >= 1");
  require(hidden > 0, "model.hidden_dim must be > 0");
  require(num_experts >= 1, "model.num_experts must be >= 1");
  require(top_k >= 1 && top_k <= num_experts, "model.top_k must be in [1, num_experts]");
  require(ffn > 0, "model.expert_ffn_dim must be > 0");
  require(shared_ffn >= 0, "model.shared_ffn_dim must be >= 0");
  require(attn_proj_params > 0, "model.attn_proj_params must be > 0");
  require(wbytes > 0, "model.weight_bytes_per_param must be > 0");
  require(kv_bytes >= 0, "model.kv_bytes_per_token_per_layer must be >= 0");
  require(abytes > 0, "model.act_bytes_per_element must be > 0");
  require(others_factor >= 0, "model.others_bytes_factor must be >= 0");
  require(calib_attention > 0 && calib_grouped > 0 && calib_dense > 0,
          "model.calib scalars must be > 0");
}

double expert_shard_bytes(const ModelSpec& m) {
  return 3.0 * static_cast<double>(m.hidden) * static_cast<double>(m.ffn) * m.wbytes;
}

// Category ids (hwmodel.hpp:14-23): 0 Attention, 1 GroupedGemm, 2 DenseGemm, 3 Others.
std::vector<OpCost> attention_entries(const ModelSpec& m, double tokens, double msl) {
  const double h = static_cast<double>(m.hidden), act = tokens * h * m.abytes;
  const double k = m.calib_attention;
  std::vector<OpCost> out;
  out.push_back({0, k * (2.0 * tokens * m.attn_proj_params + 2.0 * tokens * msl * h),
                 k * (m.attn_proj_params * m.wbytes + act + tokens * m.kv_bytes)});
  if (m.others_factor > 0) out.push_back({3, 0.0, 0.5 * m.others_factor * act});
  return out;
}

std::vector<OpCost> moe_entries(const ModelSpec& m, double tokens, double pairs, int touched) {
  const double h = static_cast<double>(m.hidden), f = static_cast<double>(m.ffn);
  std::vector<OpCost> out;
  const double g = m.calib_grouped;
  out.push_back({1, g * 2.0 * pairs * 3.0 * h * f,
                 g * (static_cast<double>(touched) * expert_shard_bytes(m) +
                      2.0 * pairs * h * m.abytes)});
  if (m.shared_ffn > 0) {
    const double fs = static_cast<double>(m.shared_ffn), d = m.calib_dense;
    out.push_back({2, d * 2.0 * tokens * 3.0 * h * fs,
                   d * (3.0 * h * fs * m.wbytes + tokens * h * m.abytes)});
  }
  if (m.others_factor > 0) out.push_back({3, 0.0, 0.5 * m.others_factor * tokens * h * m.abytes});
  return out;
}

void layer_costs(const ModelSpec& m, int64_t tokens, int64_t msl, std::vector<OpCost>& attn,
                 std::vector<OpCost>& moe) {
  m.validate();
  require(tokens >= 1, "layer_costs: tokens must be >= 1");
  require(msl >= 1, "layer_costs: mean_seq_len must be >= 1");
  const double t = static_cast<double>(tokens);
  attn = attention_entries(m, t, static_cast<double>(msl));
  moe = moe_entries(m, t, t * m.top_k, m.num_experts);
}

}  // namespace dwdp
