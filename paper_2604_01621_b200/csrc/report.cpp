// Measured-run accounting (see report.hpp).
#include "report.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "plan.hpp"

namespace dwdp {

const char* category_name(Category c) {
  static const char* names[kNumCategories] = {"Attention",     "GroupedGEMM", "DenseGEMM",
                                              "Others",        "Communication", "D2DCopy",
                                              "P2PCopy",       "SyncWait"};
  const int i = static_cast<int>(c);
  return i >= 0 && i < kNumCategories ? names[i] : "?";
}

// ---------------------------------------------------------------- RunReport
// simcore.cpp:18-58: per-rank steady window [iter_start[warmup], iter_end[last]].

double RunReport::mean_latency_us(int rank) const {
  require(rank >= 0 && rank < num_ranks, "report: rank out of range");
  const int steady = steady_iterations();
  invariant(steady > 0, "report: no steady iterations");
  double sum = 0;
  for (int it = warmup_iterations; it < iterations; ++it)
    sum += double(iter_end[size_t(rank)][size_t(it)] - iter_start[size_t(rank)][size_t(it)]);
  return sum / steady / 1e3;
}

double RunReport::mean_latency_us() const {
  double sum = 0;
  for (int r = 0; r < num_ranks; ++r) sum += mean_latency_us(r);
  return sum / num_ranks;
}

double RunReport::throughput_tokens_per_s() const {
  double total = 0;
  for (int r = 0; r < num_ranks; ++r) {
    double tok = 0;
    for (int it = warmup_iterations; it < iterations; ++it) tok += double(iter_tokens[size_t(r)][size_t(it)]);
    const double span = double(iter_end[size_t(r)][size_t(iterations - 1)] -
                               iter_start[size_t(r)][size_t(warmup_iterations)]);
    invariant(span > 0, "report: empty steady window");
    total += tok / (span / 1e9);
  }
  return total;
}

void RunReport::validate_streams() const {
  std::map<std::pair<int, int>, std::vector<std::pair<int64_t, int64_t>>> lanes;
  for (const SimEvent& e : events) {
    invariant(e.end >= e.start, "event ends before it starts");
    lanes[{e.rank, static_cast<int>(e.stream)}].emplace_back(e.start, e.end);
  }
  for (auto& kv : lanes) {
    auto& v = kv.second;
    std::sort(v.begin(), v.end());
    for (size_t i = 1; i < v.size(); ++i)
      invariant(v[i].first >= v[i - 1].second, "overlapping events on one (rank, stream)");
  }
}

// ---------------------------------------------------------------- breakdown

double BreakdownTable::category_us(Category c) const {
  auto it = compute_us.find(c);
  if (it != compute_us.end()) return it->second;
  it = copy_us.find(c);
  return it == copy_us.end() ? 0.0 : it->second;
}

std::string BreakdownTable::to_csv() const {
  std::ostringstream os;
  char num[64];
  os << "category,stream,mean_us_per_iteration\n";
  for (const auto& kv : compute_us) {
    std::snprintf(num, sizeof num, "%.4f", kv.second);
    os << category_name(kv.first) << ",compute," << num << "\n";
  }
  for (const auto& kv : copy_us) {
    std::snprintf(num, sizeof num, "%.4f", kv.second);
    os << category_name(kv.first) << ",copy_engine," << num << "\n";
  }
  std::snprintf(num, sizeof num, "%.4f", iteration_latency_us);
  os << "IterationLatency,," << num << "\n";
  return os.str();
}

BreakdownTable breakdown(const RunReport& rep) {
  const int steady = rep.steady_iterations();
  invariant(steady > 0, "breakdown: no steady iterations");
  const double per = double(rep.num_ranks) * steady;  // mean per rank and steady iteration
  BreakdownTable t;
  bool exposed = false;
  for (const SimEvent& e : rep.events) {
    if (e.iteration < rep.warmup_iterations) continue;
    const double us = double(e.end - e.start) / 1e3;
    if (e.stream == Stream::CopyEngine) {
      t.copy_us[e.category] += us / per;
      continue;
    }
    t.compute_us[e.category] += us / per;
    if (e.category == Category::SyncWait && e.detail == DWDP_DETAIL_WEIGHT_WAIT && e.end > e.start)
      exposed = true;
  }
  t.iteration_latency_us = rep.mean_latency_us();
  t.p2p_fully_overlapped = t.copy_us.count(Category::P2PCopy) > 0 && !exposed;
  return t;
}

// ---------------------------------------------------------------- compare

ComparisonTable compare_reports(const BreakdownTable& a, const BreakdownTable& b) {
  require(a.iteration_latency_us > 0, "compare_reports: zero baseline iteration latency");
  ComparisonTable out;
  out.a_latency_us = a.iteration_latency_us;
  out.b_latency_us = b.iteration_latency_us;
  out.overall_frac = (a.iteration_latency_us - b.iteration_latency_us) / a.iteration_latency_us;
  auto pct2 = [](double frac) { return std::round(frac * 100.0 * 100.0) / 100.0; };
  double comm = 0, sync = 0;
  for (int i = 0; i < kNumCategories; ++i) {
    const Category c = static_cast<Category>(i);
    ComparisonRow row{c, a.category_us(c), b.category_us(c), std::nullopt};
    if (c != Category::P2PCopy) {  // the pull is off the critical path
      row.delta_frac = (row.a_us - row.b_us) / a.iteration_latency_us;
      if (c == Category::Communication) comm = pct2(*row.delta_frac);
      if (c == Category::SyncWait) sync = pct2(*row.delta_frac);
    }
    out.rows.push_back(row);
  }
  out.gross_sync_comm_pct = comm + sync;
  return out;
}

std::string ComparisonTable::to_csv() const {
  std::ostringstream os;
  char line[128];
  os << "category,a_us,b_us,delta_pct_of_a\n";
  for (const ComparisonRow& r : rows) {
    if (r.delta_frac)
      std::snprintf(line, sizeof line, "%s,%.2f,%.2f,%.2f\n", category_name(r.category), r.a_us, r.b_us,
                    *r.delta_frac * 100.0);
    else
      std::snprintf(line, sizeof line, "%s,%.2f,%.2f,--\n", category_name(r.category), r.a_us, r.b_us);
    os << line;
  }
  std::snprintf(line, sizeof line, "IterationLatency,%.2f,%.2f,%.2f\n", a_latency_us, b_latency_us,
                overall_frac * 100.0);
  os << line;
  std::snprintf(line, sizeof line, "GrossSyncComm,,,%.2f\n", gross_sync_comm_pct);
  os << line;
  return os.str();
}

// ---------------------------------------------------------------- records -> events

void append_rank_events(RunReport& rep, int rank, const dwdp_layer_record* recs, size_t n) {
  const int L = rep.num_layers;
  require(L >= 1, "report: num_layers must be >= 1");
  require(n % size_t(L) == 0, "report: records must be whole iterations of num_layers layers");
  const int iters = int(n / size_t(L));
  if (rep.iterations == 0) rep.iterations = iters;
  require(rep.iterations == iters, "report: every rank needs the same iteration count");
  require(rank >= 0 && rank < rep.num_ranks, "report: rank out of range");
  rep.iter_start.resize(size_t(rep.num_ranks));
  rep.iter_end.resize(size_t(rep.num_ranks));
  rep.iter_tokens.resize(size_t(rep.num_ranks));
  auto& is = rep.iter_start[size_t(rank)];
  auto& ie = rep.iter_end[size_t(rank)];
  auto& tk = rep.iter_tokens[size_t(rank)];
  is.assign(size_t(iters), 0);
  ie.assign(size_t(iters), 0);
  tk.assign(size_t(iters), 0);
  auto ns = [](double v) { return int64_t(std::llround(v)); };
  for (size_t i = 0; i < n; ++i) {
    const dwdp_layer_record& r = recs[i];
    const int it = int(i / size_t(L)), layer = int(i % size_t(L));
    if (layer == 0) {
      is[size_t(it)] = ns(r.start_ns);
      tk[size_t(it)] = r.tokens;
    }
    if (layer == L - 1) ie[size_t(it)] = ns(r.end_ns);
    int64_t t = ns(r.start_ns);
    auto emit = [&](Category c, double dur, int detail = DWDP_DETAIL_NONE, double bytes = 0) {
      const int64_t e = t + ns(dur);
      rep.events.push_back({rank, Stream::Compute, c, t, e, layer, it, bytes, detail});
      t = e;
    };
    const bool dep = r.comm_ns > 0 || r.dispatch_ns > 0;
    if (!dep) emit(Category::SyncWait, r.gate_wait_ns, DWDP_DETAIL_WEIGHT_WAIT);
    if (r.merge_ns > 0) emit(Category::D2DCopy, r.merge_ns, DWDP_DETAIL_NONE, r.prefetch_bytes);
    emit(Category::Others, r.router_ns);
    emit(Category::Others, r.permute_ns);
    if (dep) emit(Category::Communication, r.dispatch_ns, DWDP_DETAIL_DISPATCH);
    emit(Category::GroupedGemm, r.gemm1_ns);
    emit(Category::GroupedGemm, r.gemm2_ns);
    if (dep) emit(Category::Communication, r.comm_ns - r.dispatch_ns, DWDP_DETAIL_COMBINE);
    emit(Category::Others, r.combine_ns);
    if (r.prefetch_start_ns >= 0 && r.prefetch_end_ns >= r.prefetch_start_ns)
      rep.events.push_back({rank, Stream::CopyEngine, Category::P2PCopy, ns(r.prefetch_start_ns),
                            ns(r.prefetch_end_ns), layer, it, r.prefetch_bytes, DWDP_DETAIL_NONE});
  }
}

BreakdownTable breakdown_from_c(const dwdp_breakdown& b) {
  BreakdownTable t;
  for (int i = 0; i < kNumCategories; ++i) {
    if (b.compute_present[i]) t.compute_us[static_cast<Category>(i)] = b.compute_us[i];
    if (b.copy_present[i]) t.copy_us[static_cast<Category>(i)] = b.copy_us[i];
  }
  t.iteration_latency_us = b.iteration_latency_us;
  t.p2p_fully_overlapped = b.p2p_fully_overlapped != 0;
  return t;
}

void breakdown_to_c(const BreakdownTable& t, double tokens_per_s, dwdp_breakdown* out) {
  *out = dwdp_breakdown{};
  for (const auto& kv : t.compute_us) {
    out->compute_us[static_cast<int>(kv.first)] = kv.second;
    out->compute_present[static_cast<int>(kv.first)] = 1;
  }
  for (const auto& kv : t.copy_us) {
    out->copy_us[static_cast<int>(kv.first)] = kv.second;
    out->copy_present[static_cast<int>(kv.first)] = 1;
  }
  out->iteration_latency_us = t.iteration_latency_us;
  out->p2p_fully_overlapped = t.p2p_fully_overlapped ? 1 : 0;
  out->tokens_per_s = tokens_per_s;
}

}  // namespace dwdp
