// Accounting: SimEvent / RunReport / breakdown / compare_reports
// (reference include/dwdpsim/simcore.hpp:29-61, 177-213; src/simcore.cpp:18-63,
// 766-876), filled from measured CUDA-event timestamps instead of a simulated
// clock. The arithmetic (order of the per-event accumulation, the steady
// window, the two-decimal gross figure) follows the reference so the same
// event list gives bit-identical tables (tests/test_report.py).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "../../include/dwdp.h"

namespace dwdp {

enum class Category : int {  // hwmodel.hpp:14-23, same order
  Attention = DWDP_CAT_ATTENTION,
  GroupedGemm = DWDP_CAT_GROUPED_GEMM,
  DenseGemm = DWDP_CAT_DENSE_GEMM,
  Others = DWDP_CAT_OTHERS,
  Communication = DWDP_CAT_COMMUNICATION,
  D2DCopy = DWDP_CAT_D2D_COPY,
  P2PCopy = DWDP_CAT_P2P_COPY,
  SyncWait = DWDP_CAT_SYNC_WAIT,
};
constexpr int kNumCategories = 8;
const char* category_name(Category c);

enum class Stream : int { Compute = 0, CopyEngine = 1 };

struct SimEvent {
  int rank = 0;
  Stream stream = Stream::Compute;
  Category category = Category::Others;
  int64_t start = 0, end = 0;  // ns
  int layer = 0, iteration = 0;
  double bytes = 0;
  int detail = DWDP_DETAIL_NONE;
};

struct RunReport {
  std::string strategy;
  int num_ranks = 0, num_layers = 0, iterations = 0, warmup_iterations = 0;
  std::vector<SimEvent> events;
  std::vector<std::vector<int64_t>> iter_start, iter_end, iter_tokens;  // [rank][iteration]

  int steady_iterations() const { return iterations - warmup_iterations; }
  double mean_latency_us(int rank) const;
  double mean_latency_us() const;
  double throughput_tokens_per_s() const;
  void validate_streams() const;
};

struct BreakdownTable {
  std::map<Category, double> compute_us, copy_us;
  double iteration_latency_us = 0;
  bool p2p_fully_overlapped = false;
  double category_us(Category c) const;
  std::string to_csv() const;
};

BreakdownTable breakdown(const RunReport& report);

struct ComparisonRow {
  Category category = Category::Others;
  double a_us = 0, b_us = 0;
  std::optional<double> delta_frac;
};

struct ComparisonTable {
  std::vector<ComparisonRow> rows;
  double a_latency_us = 0, b_latency_us = 0, overall_frac = 0, gross_sync_comm_pct = 0;
  std::string to_csv() const;
};

ComparisonTable compare_reports(const BreakdownTable& a, const BreakdownTable& b);

// One rank's measured layer records -> that rank's events and iteration
// spans. Records are whole stack iterations of `num_layers` layers, in order.
// DWDP layer: SyncWait(weight_wait) [+ D2DCopy merge] then router / permute
// (Others), GEMM1 / GEMM2 (GroupedGemm; the shared expert rides in the same
// grouped GEMM), combine (Others); its plan is a P2PCopy on the copy stream.
// DEP layer: router, permute, dispatch (Communication), GEMM1, GEMM2,
// combine all-to-all (Communication), combine.
void append_rank_events(RunReport& rep, int rank, const dwdp_layer_record* recs, size_t n);

// C-ABI struct conversions
BreakdownTable breakdown_from_c(const dwdp_breakdown& b);
void breakdown_to_c(const BreakdownTable& t, double tokens_per_s, dwdp_breakdown* out);

}  // namespace dwdp
