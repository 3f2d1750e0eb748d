// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// Flat C entry points over the UNMODIFIED reference library `dwdpsim`
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdwdpref.so). Used by tests/ to pin the C restatement in
// oracle/dwdp_oracle.c and the product host code against the reference's own
// behaviour, by oracle/gen_golden.py to emit tests/golden/*.json, and by
// bench.py's cpu_baseline leg (simulator timing).
//
// Error convention mirrors include/dwdp.h: 0 ok, 2 ConfigError, 3
// InvariantViolation (reference: include/dwdpsim/errors.hpp:11-28).
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "dwdpsim/copyplan.hpp"
#include "dwdpsim/placement.hpp"
#include "dwdpsim/rng.hpp"
#include "dwdpsim/simcore.hpp"
#include "dwdpsim/workload.hpp"

using namespace dwdpsim;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const InvariantViolation& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

MoeModelSpec make_model(int layers, int64_t hidden, int experts, int top_k,
                        int64_t ffn, int64_t shared_ffn, double wbytes,
                        double abytes) {
  MoeModelSpec m;
  m.num_layers = layers;
  m.hidden_dim = hidden;
  m.num_experts = experts;
  m.top_k = top_k;
  m.expert_ffn_dim = ffn;
  m.shared_ffn_dim = shared_ffn;
  m.attn_proj_params = 1;  // MoE-only stack: attention is out of scope,
  m.calib.attention = 1e-12;  // so its cost entries are scaled to ~0 ns
  m.weight_bytes_per_param = wbytes;
  m.act_bytes_per_element = abytes;
  return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix(uint64_t a, uint64_t b) { return Rng::mix(a, b); }

void ref_rng_u64(uint64_t seed, int n, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}

void ref_rng_normal(uint64_t seed, int n, double mean, double sd, double* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.normal(mean, sd);
}

// local_sets: [N * c]; fetch_expert/fetch_src: [N * (E - c)] (row-major per rank).
int ref_build_placement(int E, int N, int extra, int* local_count,
                        int* redundancy, int* local_sets, int* fetch_expert,
                        int* fetch_src, int capacity) {
  return guarded([&] {
    const PlacementPlan p = build_placement(E, N, extra);
    *local_count = p.local_count;
    *redundancy = p.redundancy;
    const int c = p.local_count;
    if (capacity < N * E) return;
    for (int r = 0; r < N; ++r) {
      for (int i = 0; i < c; ++i) local_sets[r * c + i] = p.local_sets[r][i];
      for (int i = 0; i < E - c; ++i) {
        fetch_expert[r * (E - c) + i] = p.fetch_lists[r][i].first;
        fetch_src[r * (E - c) + i] = p.fetch_lists[r][i].second;
      }
    }
  });
}

// shards: n x {peer, param, size, src_offset}; out: up to *n_out x
// {param, src_rank, src_offset, dst_offset, length}.
int ref_build_copy_plan(const int64_t* shards, int n, uint64_t slice, int dst,
                        int64_t* out, int64_t* n_out) {
  return guarded([&] {
    std::vector<ShardRef> v;
    for (int i = 0; i < n; ++i)
      v.push_back({static_cast<int>(shards[4 * i]),
                   static_cast<uint64_t>(shards[4 * i + 1]),
                   static_cast<uint64_t>(shards[4 * i + 2]),
                   static_cast<uint64_t>(shards[4 * i + 3])});
    const CopyPlan p = build_copy_plan(v, slice, dst);
    const int64_t cap = *n_out;
    *n_out = static_cast<int64_t>(p.slices.size());
    if (out == nullptr || cap < *n_out) return;
    for (size_t i = 0; i < p.slices.size(); ++i) {
      const Slice& s = p.slices[i];
      out[5 * i] = static_cast<int64_t>(s.param_id);
      out[5 * i + 1] = s.src_rank;
      out[5 * i + 2] = static_cast<int64_t>(s.src_offset);
      out[5 * i + 3] = static_cast<int64_t>(s.dst_offset);
      out[5 * i + 4] = static_cast<int64_t>(s.length);
    }
  });
}

int ref_route_tokens(int64_t tokens, int E, int top_k, double skew,
                     uint64_t seed, int64_t* counts) {
  return guarded([&] {
    MoeModelSpec m = make_model(1, 8, E, top_k, 8, 0, 2.0, 2.0);
    const auto c = route_tokens(tokens, m, skew, seed);
    for (int e = 0; e < E; ++e) counts[e] = c[e];
  });
}

// isl_kind: 0 fixed, 1 uniform_ratio, 2 normal. Outputs [iters*N] and
// routed [iters*N*E].
int ref_sample_batches(int isl_kind, double length, double ratio, double sd,
                       int64_t mnt, int batch_per_rank, double skew,
                       uint64_t seed, int E, int top_k, int N, int iters,
                       int64_t* tokens, int64_t* requests, int64_t* routed) {
  return guarded([&] {
    WorkloadSpec w;
    w.isl_dist.kind = static_cast<IslDist::Kind>(isl_kind);
    w.isl_dist.length = length;
    w.isl_dist.ratio = ratio;
    w.isl_dist.stddev = sd;
    w.max_num_tokens = mnt;
    w.batch_per_rank = batch_per_rank;
    w.routing_skew = skew;
    w.seed = seed;
    MoeModelSpec m = make_model(1, 8, E, top_k, 8, 0, 2.0, 2.0);
    const auto b = sample_batches(w, m, N, iters);
    for (int it = 0; it < iters; ++it)
      for (int r = 0; r < N; ++r) {
        tokens[it * N + r] = b[it].tokens[r];
        requests[it * N + r] = b[it].requests[r];
        if (routed)
          for (int e = 0; e < E; ++e)
            routed[(static_cast<int64_t>(it) * N + r) * E + e] =
                b[it].routed[r][e];
      }
  });
}

double ref_expert_shard_bytes(int64_t hidden, int64_t ffn, double wbytes) {
  MoeModelSpec m = make_model(1, hidden, 1, 1, ffn, 0, wbytes, 2.0);
  return expert_shard_bytes(m);
}

// GroupedGEMM and DenseGEMM entries of moe_entries (flops, bytes).
int ref_moe_entries(int64_t hidden, int E, int top_k, int64_t ffn,
                    int64_t shared_ffn, double wbytes, double abytes,
                    double tokens, double pairs, int touched, double* out4) {
  return guarded([&] {
    MoeModelSpec m =
        make_model(1, hidden, E, top_k, ffn, shared_ffn, wbytes, abytes);
    out4[0] = out4[1] = out4[2] = out4[3] = 0;
    for (const auto& op : moe_entries(m, tokens, pairs, touched)) {
      if (op.category == Category::GroupedGemm) {
        out4[0] = op.flops;
        out4[1] = op.bytes;
      } else if (op.category == Category::DenseGemm) {
        out4[2] = op.flops;
        out4[3] = op.bytes;
      }
    }
  });
}

}  // extern "C"

namespace {
RunReport g_reports[4];  // slots for the report-accounting pins

// Calibration inputs of the measured-trace loop (scripts/calibrate.py):
// GpuSpec peak/mem/link/ce_inflight and CostCalibration + Others factor
// (include/dwdpsim/modelspec.hpp:15-19, hwmodel.hpp:29-38).
struct SimCal {
  double peak_flops, mem_bw, link_bw;
  int ce_inflight;
  double grouped_gemm, dense_gemm, others_bytes_factor;
  int mem_interference;
};

RunReport run_sim_cal(int dwdp, int layers, int64_t hidden, int E, int top_k, int64_t ffn,
                      int64_t shared_ffn, double wbytes, const SimCal& c, int N, int iters,
                      int warmup, int isl_kind, double length, double ratio, double sd,
                      int64_t mnt, int batch_per_rank, uint64_t seed, int tdm, uint64_t slice,
                      int merge_elim);

RunReport run_sim(int dwdp, int layers, int64_t hidden, int E, int top_k, int64_t ffn,
                  int64_t shared_ffn, double wbytes, double peak_flops, double mem_bw,
                  double link_bw, int N, int iters, int warmup, int isl_kind, double length,
                  double ratio, double sd, int64_t mnt, int batch_per_rank, uint64_t seed,
                  int tdm, uint64_t slice, int merge_elim) {
  const SimCal c{peak_flops, mem_bw, link_bw, 2, 1.0, 1.0, 0.0, 0};
  return run_sim_cal(dwdp, layers, hidden, E, top_k, ffn, shared_ffn, wbytes, c, N, iters, warmup,
                     isl_kind, length, ratio, sd, mnt, batch_per_rank, seed, tdm, slice, merge_elim);
}

RunReport run_sim_cal(int dwdp, int layers, int64_t hidden, int E, int top_k, int64_t ffn,
                      int64_t shared_ffn, double wbytes, const SimCal& c, int N, int iters,
                      int warmup, int isl_kind, double length, double ratio, double sd,
                      int64_t mnt, int batch_per_rank, uint64_t seed, int tdm, uint64_t slice,
                      int merge_elim) {
    MoeModelSpec m =
        make_model(layers, hidden, E, top_k, ffn, shared_ffn, wbytes, 2.0);
    m.calib.grouped_gemm = c.grouped_gemm;
    m.calib.dense_gemm = c.dense_gemm;
    m.others_bytes_factor = c.others_bytes_factor;
    GpuSpec g;
    g.peak_flops = c.peak_flops;
    g.mem_bw = c.mem_bw;
    g.link_bw = c.link_bw;
    g.ce_inflight = c.ce_inflight;
    InterferenceParams ip;
    ip.mem_interference_on = c.mem_interference != 0;
    ip.power_interference_on = false;
    WorkloadSpec w;
    w.isl_dist.kind = static_cast<IslDist::Kind>(isl_kind);
    w.isl_dist.length = length;
    w.isl_dist.ratio = ratio;
    w.isl_dist.stddev = sd;
    w.max_num_tokens = mnt;
    w.batch_per_rank = batch_per_rank;
    w.seed = seed;
    const auto batches = sample_batches(w, m, N, iters);
    if (dwdp) {
      DwdpOptions o;
      o.tdm = tdm != 0;
      o.slice_size = slice;
      o.merge_elim = merge_elim != 0;
      return simulate_dwdp(m, g, ip, batches, build_placement(E, N, 0), o, warmup);
    }
    return simulate_dep(m, g, ip, batches, N, warmup);
}

int detail_code(const std::string& d) {
  if (d == "weight_wait") return 1;
  if (d == "dispatch") return 2;
  if (d == "combine") return 3;
  if (d == "barrier") return 4;
  return 0;
}

// BreakdownTable <-> 35 doubles: compute[8], copy[8], compute_present[8],
// copy_present[8], latency, overlapped, tokens/s
void pack_breakdown(const BreakdownTable& t, double tps, double* o) {
  for (int i = 0; i < 35; ++i) o[i] = 0;
  for (const auto& [c, us] : t.compute_us) {
    o[static_cast<int>(c)] = us;
    o[16 + static_cast<int>(c)] = 1;
  }
  for (const auto& [c, us] : t.copy_us) {
    o[8 + static_cast<int>(c)] = us;
    o[24 + static_cast<int>(c)] = 1;
  }
  o[32] = t.iteration_latency_us;
  o[33] = t.p2p_fully_overlapped ? 1 : 0;
  o[34] = tps;
}

BreakdownTable unpack_breakdown(const double* o) {
  BreakdownTable t;
  for (int i = 0; i < 8; ++i) {
    if (o[16 + i] != 0) t.compute_us[static_cast<Category>(i)] = o[i];
    if (o[24 + i] != 0) t.copy_us[static_cast<Category>(i)] = o[8 + i];
  }
  t.iteration_latency_us = o[32];
  t.p2p_fully_overlapped = o[33] != 0;
  return t;
}

void put_str(const std::string& s, char* buf, int cap) {
  if (cap <= 0) return;
  const size_t n = std::min(s.size(), size_t(cap - 1));
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}
}  // namespace

extern "C" {

// Simulate into report slot `slot` (0..3) for the accounting pins.
int ref_simulate_store(int slot, int dwdp, int layers, int64_t hidden, int E, int top_k,
                       int64_t ffn, int64_t shared_ffn, double wbytes, double peak_flops,
                       double mem_bw, double link_bw, int N, int iters, int warmup,
                       int isl_kind, double length, double ratio, double sd, int64_t mnt,
                       int batch_per_rank, uint64_t seed, int tdm, uint64_t slice,
                       int merge_elim, int* n_events) {
  return guarded([&] {
    require(slot >= 0 && slot < 4, "slot out of range");
    g_reports[slot] = run_sim(dwdp, layers, hidden, E, top_k, ffn, shared_ffn, wbytes,
                              peak_flops, mem_bw, link_bw, N, iters, warmup, isl_kind, length,
                              ratio, sd, mnt, batch_per_rank, seed, tdm, slice, merge_elim);
    *n_events = static_cast<int>(g_reports[slot].events.size());
  });
}

// Same with the calibration loop's inputs: cal = {peak_flops, mem_bw,
// link_bw, ce_inflight, calib.grouped_gemm, calib.dense_gemm,
// others_bytes_factor, mem_interference_on}.
int ref_simulate_store_cal(int slot, int dwdp, int layers, int64_t hidden, int E, int top_k,
                           int64_t ffn, int64_t shared_ffn, double wbytes, const double* cal,
                           int N, int iters, int warmup, int isl_kind, double length,
                           double ratio, double sd, int64_t mnt, int batch_per_rank,
                           uint64_t seed, int tdm, uint64_t slice, int merge_elim,
                           int* n_events) {
  return guarded([&] {
    require(slot >= 0 && slot < 4, "slot out of range");
    const SimCal c{cal[0], cal[1], cal[2], static_cast<int>(cal[3]), cal[4], cal[5], cal[6],
                   static_cast<int>(cal[7])};
    g_reports[slot] = run_sim_cal(dwdp, layers, hidden, E, top_k, ffn, shared_ffn, wbytes, c, N,
                                  iters, warmup, isl_kind, length, ratio, sd, mnt, batch_per_rank,
                                  seed, tdm, slice, merge_elim);
    *n_events = static_cast<int>(g_reports[slot].events.size());
  });
}

// Events of a stored report: i32[n][6] {rank, stream, category, layer,
// iteration, detail}, i64[n][2] {start, end}, bytes[n]; iteration spans
// [ranks][iters]; dims = {ranks, iterations, warmup}.
int ref_report_events(int slot, int32_t* i32, int64_t* i64, double* bytes, int64_t* is,
                      int64_t* ie, int64_t* tk, int* dims) {
  return guarded([&] {
    const RunReport& r = g_reports[slot];
    for (size_t i = 0; i < r.events.size(); ++i) {
      const SimEvent& e = r.events[i];
      int32_t* p = i32 + 6 * i;
      p[0] = e.rank;
      p[1] = static_cast<int32_t>(e.stream);
      p[2] = static_cast<int32_t>(e.category);
      p[3] = e.layer;
      p[4] = e.iteration;
      p[5] = detail_code(e.detail);
      i64[2 * i] = e.start;
      i64[2 * i + 1] = e.end;
      bytes[i] = e.bytes;
    }
    for (int k = 0; k < r.num_ranks; ++k)
      for (int it = 0; it < r.iterations; ++it) {
        is[k * r.iterations + it] = r.iter_start[k][it];
        ie[k * r.iterations + it] = r.iter_end[k][it];
        tk[k * r.iterations + it] = r.iter_tokens[k][it];
      }
    dims[0] = r.num_ranks;
    dims[1] = r.iterations;
    dims[2] = r.warmup_iterations;
  });
}

int ref_report_breakdown(int slot, double* out35, char* csv, int cap) {
  return guarded([&] {
    const BreakdownTable t = breakdown(g_reports[slot]);
    pack_breakdown(t, g_reports[slot].throughput_tokens_per_s(), out35);
    put_str(t.to_csv(), csv, cap);
  });
}

// compare_reports over two packed breakdowns: out[8 a, 8 b, 8 delta,
// 8 has_delta, a_lat, b_lat, overall, gross].
int ref_compare(const double* a35, const double* b35, double* out36, char* csv, int cap) {
  return guarded([&] {
    const ComparisonTable t = compare_reports(unpack_breakdown(a35), unpack_breakdown(b35));
    for (int i = 0; i < 36; ++i) out36[i] = 0;
    for (const auto& row : t.rows) {
      const int c = static_cast<int>(row.category);
      out36[c] = row.a_us;
      out36[8 + c] = row.b_us;
      out36[16 + c] = row.delta_frac ? *row.delta_frac : 0.0;
      out36[24 + c] = row.delta_frac ? 1 : 0;
    }
    out36[32] = t.a_latency_us;
    out36[33] = t.b_latency_us;
    out36[34] = t.overall_frac;
    out36[35] = t.gross_sync_comm_pct;
    put_str(t.to_csv(), csv, cap);
  });
}

// Runs the reference simulator (DWDP when dwdp!=0, else DEP) over batches
// drawn from the workload spec; returns tokens/s, mean latency (us) and
// exposed weight-wait us per layer per rank.
int ref_simulate(int dwdp, int layers, int64_t hidden, int E, int top_k,
                 int64_t ffn, int64_t shared_ffn, double wbytes,
                 double peak_flops, double mem_bw, double link_bw, int N,
                 int iters, int warmup, int isl_kind, double length,
                 double ratio, double sd, int64_t mnt, int batch_per_rank,
                 uint64_t seed, int tdm, uint64_t slice, int merge_elim,
                 double* out3) {
  return guarded([&] {
    RunReport rep = run_sim(dwdp, layers, hidden, E, top_k, ffn, shared_ffn, wbytes, peak_flops,
                            mem_bw, link_bw, N, iters, warmup, isl_kind, length, ratio, sd, mnt,
                            batch_per_rank, seed, tdm, slice, merge_elim);
    double wait_ns = 0;
    for (const auto& e : rep.events)
      if (e.category == Category::SyncWait && e.detail == "weight_wait" &&
          e.iteration >= warmup)
        wait_ns += static_cast<double>(e.end - e.start);
    out3[0] = rep.throughput_tokens_per_s();
    out3[1] = rep.mean_latency_us();
    out3[2] = wait_ns / 1e3 / (rep.steady_iterations() * layers * N);
  });
}

// analytic_compare for an all-MoE layer (reference src/simcore.cpp:882-905).
int ref_analytic(int64_t hidden, int E, int top_k, int64_t ffn,
                 int64_t shared_ffn, double wbytes, double peak_flops,
                 double mem_bw, double link_bw, int N, int64_t tokens,
                 double* out4) {
  return guarded([&] {
    MoeModelSpec m =
        make_model(1, hidden, E, top_k, ffn, shared_ffn, wbytes, 2.0);
    GpuSpec g;
    g.peak_flops = peak_flops;
    g.mem_bw = mem_bw;
    g.link_bw = link_bw;
    const auto r =
        analytic_compare(m, g, build_placement(E, N, 0), tokens, 1);
    out4[0] = r.t_compute_s;
    out4[1] = r.t_prefetch_s;
    out4[2] = r.t_all2all_s;
    out4[3] = r.dep_dwdp_speedup;
  });
}

}  // extern "C"
