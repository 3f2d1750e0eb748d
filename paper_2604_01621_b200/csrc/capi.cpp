// extern "C" boundary: include/dwdp.h. No exception crosses it; every entry
// maps ConfigError -> 2, InvariantViolation -> 3, CUDA failures -> 4
// (reference error contract: include/dwdpsim/errors.hpp:11-28).
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dwdp.h"
#include "kernels.hpp"
#include "plan.hpp"
#include "report.hpp"
#include "runtime.hpp"

struct dwdp_placement {
  dwdp::Placement p;
};
struct dwdp_ctx {
  dwdp::Ctx* impl;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return DWDP_OK;
  } catch (const dwdp::ConfigError& e) {
    g_err = e.what();
    return DWDP_ERR_CONFIG;
  } catch (const dwdp::InvariantViolation& e) {
    g_err = e.what();
    return DWDP_ERR_INVARIANT;
  } catch (const dwdp::CudaError& e) {
    g_err = e.what();
    return DWDP_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DWDP_ERR_CUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw dwdp::ConfigError(std::string(what) + " is NULL");
}

// The MoeModelSpec fields every cost entry reads (no attention terms).
dwdp::ModelSpec to_model(const dwdp_model_spec* m) {
  need(m, "model");
  dwdp::require(m->hidden_dim > 0, "model.hidden_dim must be > 0");
  dwdp::require(m->num_experts >= 1, "model.num_experts must be >= 1");
  dwdp::require(m->top_k >= 1 && m->top_k <= m->num_experts,
                "model.top_k must be in [1, num_experts]");
  dwdp::require(m->expert_ffn_dim > 0, "model.expert_ffn_dim must be > 0");
  dwdp::require(m->shared_ffn_dim >= 0, "model.shared_ffn_dim must be >= 0");
  dwdp::require(m->weight_bytes_per_param > 0, "model.weight_bytes_per_param must be > 0");
  dwdp::require(m->act_bytes_per_element > 0, "model.act_bytes_per_element must be > 0");
  dwdp::ModelSpec s;
  s.num_layers = m->num_layers;
  s.num_experts = m->num_experts;
  s.top_k = m->top_k;
  s.hidden = m->hidden_dim;
  s.ffn = m->expert_ffn_dim;
  s.shared_ffn = m->shared_ffn_dim;
  s.wbytes = m->weight_bytes_per_param;
  s.abytes = m->act_bytes_per_element;
  s.attn_proj_params = m->attn_proj_params;
  s.kv_bytes = m->kv_bytes_per_token_per_layer;
  s.others_factor = m->others_bytes_factor;
  s.calib_attention = m->calib_attention;
  s.calib_grouped = m->calib_grouped_gemm;
  s.calib_dense = m->calib_dense_gemm;
  dwdp::require(s.others_factor >= 0, "model.others_bytes_factor must be >= 0");
  dwdp::require(s.calib_attention > 0 && s.calib_grouped > 0 && s.calib_dense > 0,
                "model.calib scalars must be > 0");
  return s;
}

// Full MoeModelSpec (modelspec.cpp:6-23), no subset pre-checks.
dwdp::ModelSpec to_model_full(const dwdp_model_spec* m) {
  need(m, "model");
  dwdp::ModelSpec s;
  s.num_layers = m->num_layers;
  s.num_experts = m->num_experts;
  s.top_k = m->top_k;
  s.hidden = m->hidden_dim;
  s.ffn = m->expert_ffn_dim;
  s.shared_ffn = m->shared_ffn_dim;
  s.wbytes = m->weight_bytes_per_param;
  s.abytes = m->act_bytes_per_element;
  s.attn_proj_params = m->attn_proj_params;
  s.kv_bytes = m->kv_bytes_per_token_per_layer;
  s.others_factor = m->others_bytes_factor;
  s.calib_attention = m->calib_attention;
  s.calib_grouped = m->calib_grouped_gemm;
  s.calib_dense = m->calib_dense_gemm;
  s.validate();
  return s;
}

void put_costs(const std::vector<dwdp::OpCost>& e, dwdp_op_cost* out, int* n_out) {
  need(out, "out");
  need(n_out, "n_out");
  for (size_t i = 0; i < e.size(); ++i) out[i] = {e[i].category, 0, e[i].flops, e[i].bytes, 0.0};
  *n_out = int(e.size());
}

dwdp::WorkloadSpec to_spec(const dwdp_workload_spec* w) {
  need(w, "spec");
  dwdp::WorkloadSpec s;
  s.isl_kind = w->isl_kind;
  s.length = w->length;
  s.ratio = w->ratio;
  s.stddev = w->stddev;
  s.max_num_tokens = w->max_num_tokens;
  s.batch_per_rank = w->batch_per_rank;
  s.routing_skew = w->routing_skew;
  s.seed = w->seed;
  return s;
}

}  // namespace

int dwdp::capi_guard(const std::function<void()>& f) { return guard(f); }

namespace {

dwdp::Ctx& C(dwdp_ctx* c) {
  need(c, "ctx");
  return *c->impl;
}
}  // namespace

extern "C" {

const char* dwdp_last_error(void) { return g_err.c_str(); }

const char* dwdp_version(void) {
  static const std::string v = "dwdp-b200 sm_100a cuda " + std::to_string(CUDART_VERSION);
  return v.c_str();
}

// ---------------------------------------------------------------- placement
int dwdp_placement_build(int E, int N, int extra, dwdp_placement** out) {
  return guard([&] {
    need(out, "out");
    *out = new dwdp_placement{dwdp::build_placement(E, N, extra)};
  });
}

void dwdp_placement_free(dwdp_placement* p) { delete p; }

int dwdp_placement_info(const dwdp_placement* p, int* n, int* e, int* c, int* r) {
  return guard([&] {
    need(p, "placement");
    if (n) *n = p->p.group_size;
    if (e) *e = p->p.num_experts;
    if (c) *c = p->p.local_count;
    if (r) *r = p->p.redundancy;
  });
}

int dwdp_placement_local_set(const dwdp_placement* p, int rank, int* experts) {
  return guard([&] {
    need(p, "placement");
    need(experts, "experts");
    dwdp::require(rank >= 0 && rank < p->p.group_size, "placement: rank out of range");
    const auto& s = p->p.local_sets[size_t(rank)];
    std::copy(s.begin(), s.end(), experts);
  });
}

int dwdp_placement_fetch_list(const dwdp_placement* p, int rank, int* experts, int* sources) {
  return guard([&] {
    need(p, "placement");
    dwdp::require(rank >= 0 && rank < p->p.group_size, "placement: rank out of range");
    const auto& f = p->p.fetch_lists[size_t(rank)];
    for (size_t i = 0; i < f.size(); ++i) {
      if (experts) experts[i] = f[i].first;
      if (sources) sources[i] = f[i].second;
    }
  });
}

int dwdp_placement_holds(const dwdp_placement* p, int rank, int expert, int* holds) {
  return guard([&] {
    need(p, "placement");
    need(holds, "holds");
    dwdp::require(rank >= 0 && rank < p->p.group_size, "placement: rank out of range");
    *holds = p->p.holds(rank, expert) ? 1 : 0;
  });
}

int dwdp_placement_validate(const dwdp_placement* p) {
  return guard([&] {
    need(p, "placement");
    p->p.validate();
  });
}

int dwdp_placement_from_tables(int N, int E, int c, int red, const int* loffs,
                               const int* lflat, const int* foffs, const int* fe, const int* fs,
                               dwdp_placement** out) {
  return guard([&] {
    need(out, "out");
    dwdp::invariant(N >= 0 && E >= 0, "placement: table shape mismatch");
    if (N > 0) {
      need(loffs, "local_offsets");
      need(foffs, "fetch_offsets");
    }
    dwdp::Placement p;
    p.group_size = N;
    p.num_experts = E;
    p.local_count = c;
    p.redundancy = red;
    p.local_sets.resize(size_t(N));
    p.fetch_lists.resize(size_t(N));
    for (int r = 0; r < N; ++r) {
      for (int i = loffs[r]; i < loffs[r + 1]; ++i) p.local_sets[size_t(r)].push_back(lflat[i]);
      for (int i = foffs[r]; i < foffs[r + 1]; ++i)
        p.fetch_lists[size_t(r)].emplace_back(fe[i], fs[i]);
    }
    p.validate();
    *out = new dwdp_placement{std::move(p)};
  });
}

int dwdp_prefetch_bytes(const dwdp_placement* p, double shard, double* bytes) {
  return guard([&] {
    need(p, "placement");
    need(bytes, "bytes");
    *bytes = double(p->p.num_experts - p->p.local_count) * shard;
  });
}

int dwdp_placement_describe(const dwdp_placement* p, char* buf, size_t* len) {
  return guard([&] {
    need(p, "placement");
    need(len, "len");
    const std::string s = p->p.describe();
    const size_t cap = *len;
    *len = s.size() + 1;
    if (buf && cap >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int dwdp_assign_fetch_sources(int E, int N, const int* offs, const int* flat, int* counts,
                              int* fe, int* fs) {
  return guard([&] {
    need(offs, "local_offsets");
    need(flat, "local_flat");
    dwdp::require(N >= 1 && E >= 1, "assign_fetch_sources: bad sizes");
    std::vector<std::vector<int>> sets(static_cast<size_t>(N));
    for (int r = 0; r < N; ++r)
      for (int i = offs[r]; i < offs[r + 1]; ++i) {
        dwdp::require(flat[i] >= 0 && flat[i] < E, "assign_fetch_sources: expert out of range");
        sets[size_t(r)].push_back(flat[i]);
      }
    const auto fl = dwdp::assign_fetch_sources(E, sets);
    for (int r = 0; r < N; ++r) {
      if (counts) counts[r] = int(fl[size_t(r)].size());
      for (size_t i = 0; i < fl[size_t(r)].size(); ++i) {
        if (fe) fe[size_t(r) * size_t(E) + i] = fl[size_t(r)][i].first;
        if (fs) fs[size_t(r) * size_t(E) + i] = fl[size_t(r)][i].second;
      }
    }
  });
}

// ---------------------------------------------------------------- copy plan
int dwdp_copy_plan_build(const dwdp_shard_ref* shards, size_t n, uint64_t slice, int dst,
                         dwdp_slice* out, size_t* n_inout) {
  return guard([&] {
    need(n_inout, "n_inout");
    if (n) need(shards, "shards");
    std::vector<dwdp::ShardRef> v(n);
    for (size_t i = 0; i < n; ++i)
      v[i] = {shards[i].peer, shards[i].param_id, shards[i].size, shards[i].src_offset};
    const auto plan = dwdp::build_copy_plan(v, slice, dst);
    const size_t cap = *n_inout;
    *n_inout = plan.size();
    if (!out) return;
    dwdp::require(cap >= plan.size(), "copy plan: output capacity too small");
    for (size_t i = 0; i < plan.size(); ++i)
      out[i] = {plan[i].param_id, plan[i].src_rank, 0, plan[i].src_offset, plan[i].dst_offset,
                plan[i].length};
  });
}

int dwdp_source_queues(size_t n_plans, const int* dsts, const dwdp_slice* const* plans,
                       const size_t* lens, int source, int* out_dsts, size_t* out_counts,
                       size_t* n_queues, dwdp_slice* out, size_t* n_inout) {
  return guard([&] {
    need(n_queues, "n_queues");
    need(n_inout, "n_inout");
    std::map<int, std::vector<dwdp_slice>> q;
    for (size_t i = 0; i < n_plans; ++i) {
      auto& v = q[dsts[i]];  // present even if empty
      for (size_t j = 0; j < lens[i]; ++j)
        if (plans[i][j].src_rank == source) v.push_back(plans[i][j]);
    }
    size_t total = 0;
    for (auto& kv : q) total += kv.second.size();
    const size_t cap = *n_inout;
    *n_inout = total;
    *n_queues = q.size();
    if (!out) return;
    dwdp::require(cap >= total, "source_queues: output capacity too small");
    size_t i = 0, k = 0;
    for (auto& kv : q) {
      if (out_dsts) out_dsts[k] = kv.first;
      if (out_counts) out_counts[k] = kv.second.size();
      ++k;
      for (auto& s : kv.second) out[i++] = s;
    }
  });
}

// ---------------------------------------------------------------- workload
uint64_t dwdp_rng_mix(uint64_t a, uint64_t b) { return dwdp::Rng::mix(a, b); }

int dwdp_route_tokens(int64_t tokens, int E, int k, double skew, uint64_t seed, int64_t* counts) {
  return guard([&] {
    need(counts, "counts");
    const auto c = dwdp::route_tokens(tokens, E, k, skew, seed);
    std::copy(c.begin(), c.end(), counts);
  });
}

int dwdp_sample_batches(const dwdp_workload_spec* w, int E, int k, int N, int iters,
                        int64_t* tokens, int64_t* requests, int64_t* routed) {
  return guard([&] {
    need(tokens, "tokens");
    dwdp::require(k >= 1 && k <= E, "model.top_k must be in [1, num_experts]");
    const auto b = dwdp::sample_batches(to_spec(w), E, k, N, iters, routed != nullptr);
    for (int it = 0; it < iters; ++it)
      for (int r = 0; r < N; ++r) {
        const size_t i = size_t(it) * size_t(N) + size_t(r);
        tokens[i] = b.tokens[size_t(it)][size_t(r)];
        if (requests) requests[i] = b.requests[size_t(it)][size_t(r)];
        if (routed)
          std::copy(b.routed[size_t(it)][size_t(r)].begin(), b.routed[size_t(it)][size_t(r)].end(),
                    routed + i * size_t(E));
      }
  });
}

int dwdp_imbalance_cv(const int64_t* tokens, int n, double* cv) {
  return guard([&] {
    need(cv, "cv");
    dwdp::require(n >= 2, "imbalance_cv: need at least 2 ranks");
    need(tokens, "tokens");
    *cv = dwdp::imbalance_cv(std::vector<int64_t>(tokens, tokens + n));
  });
}

int dwdp_workload_validate(const dwdp_workload_spec* w) {
  return guard([&] { to_spec(w).validate(); });
}

int dwdp_batches_to_csv(const int64_t* tokens, const int64_t* requests, const int64_t* routed,
                        int iters, int N, int E, char* buf, size_t* len) {
  return guard([&] {
    need(len, "len_inout");
    dwdp::require(iters >= 0 && N >= 0 && E >= 0, "batches csv: negative shape");
    if (iters * N > 0) {
      need(tokens, "tokens");
      need(requests, "requests");
    }
    dwdp::Batches b;
    b.tokens.assign(size_t(iters), std::vector<int64_t>(size_t(N)));
    b.requests = b.tokens;
    b.routed.assign(size_t(iters), std::vector<std::vector<int64_t>>(size_t(N)));
    for (int it = 0; it < iters; ++it)
      for (int r = 0; r < N; ++r) {
        const size_t i = size_t(it) * size_t(N) + size_t(r);
        b.tokens[size_t(it)][size_t(r)] = tokens[i];
        b.requests[size_t(it)][size_t(r)] = requests[i];
        if (routed) b.routed[size_t(it)][size_t(r)].assign(routed + i * size_t(E),
                                                             routed + (i + 1) * size_t(E));
      }
    const std::string s = dwdp::batches_to_csv(b);
    const size_t cap = *len;
    *len = s.size() + 1;
    if (buf && cap >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int dwdp_batches_from_csv(const char* csv, int* iters, int* N, int* E, int64_t* tokens,
                          int64_t* requests, int64_t* routed, int32_t* routed_len) {
  return guard([&] {
    need(csv, "csv");
    need(iters, "iterations");
    need(N, "num_ranks");
    need(E, "num_experts");
    const auto b = dwdp::batches_from_csv(csv);
    size_t nr = 0, ne = 0;
    for (size_t it = 0; it < b.tokens.size(); ++it) {
      nr = std::max(nr, b.tokens[it].size());
      for (const auto& c : b.routed[it]) ne = std::max(ne, c.size());
    }
    *iters = int(b.tokens.size());
    *N = int(nr);
    *E = int(ne);
    for (size_t it = 0; it < b.tokens.size(); ++it)
      for (size_t r = 0; r < nr; ++r) {
        const size_t i = it * nr + r;
        const bool have = r < b.tokens[it].size();
        if (tokens) tokens[i] = have ? b.tokens[it][r] : 0;
        if (requests) requests[i] = have ? b.requests[it][r] : 0;
        const std::vector<int64_t> none;
        const auto& c = have ? b.routed[it][r] : none;
        if (routed_len) routed_len[i] = int32_t(c.size());
        if (routed)
          for (size_t e = 0; e < ne; ++e) routed[i * ne + e] = e < c.size() ? c[e] : 0;
      }
  });
}

int dwdp_isl_cv(const dwdp_workload_spec* w, double* cv) {
  return guard([&] {
    need(cv, "cv");
    *cv = to_spec(w).cv();
  });
}

// ---------------------------------------------------------------- costs
int dwdp_expert_shard_bytes(const dwdp_model_spec* m, double* bytes) {
  return guard([&] {
    need(bytes, "bytes");
    *bytes = dwdp::expert_shard_bytes(to_model(m));
  });
}

const char* dwdp_category_name(int c) {
  static const char* const names[DWDP_NUM_CATEGORIES] = {
      "Attention", "GroupedGEMM", "DenseGEMM", "Others",
      "Communication", "D2DCopy", "P2PCopy", "SyncWait"};
  return c >= 0 && c < DWDP_NUM_CATEGORIES ? names[c] : nullptr;
}

int dwdp_model_validate(const dwdp_model_spec* m) {
  return guard([&] { to_model_full(m); });
}

int dwdp_attention_entries(const dwdp_model_spec* m, double tokens, double msl,
                           dwdp_op_cost* out, int* n_out) {
  return guard([&] { put_costs(dwdp::attention_entries(to_model(m), tokens, msl), out, n_out); });
}

int dwdp_moe_entries(const dwdp_model_spec* m, double tokens, double pairs, int touched,
                     dwdp_op_cost* out, int* n_out) {
  return guard([&] { put_costs(dwdp::moe_entries(to_model(m), tokens, pairs, touched), out, n_out); });
}

int dwdp_layer_costs(const dwdp_model_spec* m, int64_t tokens, int64_t msl, dwdp_op_cost* attn,
                     int* n_attn, dwdp_op_cost* moe, int* n_moe) {
  return guard([&] {
    std::vector<dwdp::OpCost> a, b;
    dwdp::layer_costs(to_model_full(m), tokens, msl, a, b);
    put_costs(a, attn, n_attn);
    put_costs(b, moe, n_moe);
  });
}

int dwdp_roofline_time(double flops, double bytes, const dwdp_gpu_spec* g, double* s) {
  return guard([&] {
    need(g, "gpu");
    need(s, "seconds");
    dwdp::require(flops >= 0, "roofline_time: negative flops");
    dwdp::require(bytes >= 0, "roofline_time: negative bytes");
    dwdp::require(flops > 0 || bytes > 0, "roofline_time: operator has no work");
    *s = std::max(flops / g->peak_flops, bytes / g->mem_bw);
  });
}

int dwdp_analytic_compare(const dwdp_model_spec* m, const dwdp_gpu_spec* g,
                          const dwdp_placement* p, int64_t tokens, int64_t msl,
                          dwdp_analytic_result* out) {
  return guard([&] {
    need(g, "gpu");
    need(p, "placement");
    need(out, "out");
    const auto spec = msl > 0 ? to_model_full(m) : to_model(m);
    dwdp::require(g->peak_flops > 0, "gpu.peak_flops must be > 0");
    dwdp::require(g->mem_bw > 0, "gpu.mem_bw must be > 0");
    dwdp::require(g->link_bw > 0, "gpu.link_bw must be > 0");
    dwdp::require(p->p.num_experts == spec.num_experts,
                  "analytic_compare: placement does not match the model");
    dwdp::require(tokens >= 1, "layer_costs: tokens must be >= 1");
    const double t = double(tokens);
    std::vector<dwdp::OpCost> ops, moe;
    if (msl > 0)
      dwdp::layer_costs(spec, tokens, msl, ops, moe);
    else
      moe = dwdp::moe_entries(spec, t, t * spec.top_k, spec.num_experts);
    ops.insert(ops.end(), moe.begin(), moe.end());
    double tc = 0;
    for (const auto& op : ops) tc += std::max(op.flops / g->peak_flops, op.bytes / g->mem_bw);
    const double pf = double(p->p.num_experts - p->p.local_count) * dwdp::expert_shard_bytes(spec);
    *out = {};
    out->t_compute_s = tc;
    out->t_prefetch_s = pf / g->link_bw;
    out->t_all2all_s = 2.0 * t * spec.top_k * double(spec.hidden) * spec.abytes / g->link_bw;
    const double t_dep = tc + out->t_all2all_s;
    if (out->t_prefetch_s <= 0) {
      out->prefetch_saturated = 1;
      out->compute_prefetch_ratio = 1.0 / 0.0;
      out->dep_dwdp_speedup = t_dep / tc;
    } else {
      out->compute_prefetch_ratio = tc / out->t_prefetch_s;
      out->dep_dwdp_speedup = t_dep / std::max(tc, out->t_prefetch_s);
    }
  });
}

// ---------------------------------------------------------------- runtime
int dwdp_ctx_create(const dwdp_ctx_config* cfg, dwdp_ctx** out) {
  return guard([&] {
    need(cfg, "cfg");
    need(out, "out");
    *out = new dwdp_ctx{new dwdp::Ctx(*cfg)};
  });
}

int dwdp_ctx_destroy(dwdp_ctx* c) {
  return guard([&] {
    if (!c) return;
    delete c->impl;
    delete c;
  });
}

int dwdp_ctx_memory(const dwdp_ctx* c, uint64_t* w, uint64_t* r, uint64_t* ws) {
  return guard([&] {
    need(c, "ctx");
    if (w) *w = c->impl->weight_bytes;
    if (r) *r = c->impl->recv_bytes;
    if (ws) *ws = c->impl->workspace_bytes;
  });
}

int dwdp_ctx_export_ipc(dwdp_ctx* c, void* blob) {
  return guard([&] {
    need(blob, "blob");
    C(c).export_ipc(blob);
  });
}

int dwdp_ctx_open_peers(dwdp_ctx* c, const void* blobs) {
  return guard([&] {
    need(blobs, "blobs");
    C(c).open_peers(blobs);
  });
}

int dwdp_ctx_link_local(dwdp_ctx* const* ctxs, int n) {
  return guard([&] {
    need(ctxs, "ctxs");
    std::vector<dwdp::Ctx*> all;
    for (int i = 0; i < n; ++i) all.push_back(&C(ctxs[i]));
    for (auto* c : all) c->link_local(all);
  });
}

int dwdp_ctx_init_weights(dwdp_ctx* c, float bias_scale) {
  return guard([&] { C(c).init_weights(bias_scale); });
}

int dwdp_ctx_set_bias(dwdp_ctx* c, const float* bias) {
  return guard([&] {
    need(bias, "bias");
    C(c).set_bias(bias);
  });
}

int dwdp_ctx_read_expert(dwdp_ctx* c, int layer, int expert, int t, void* host) {
  return guard([&] {
    need(host, "host");
    C(c).read_expert(layer, expert, t, host);
  });
}

int dwdp_prefetch_issue(dwdp_ctx* c, int64_t g, dwdp_prefetch* h) {
  return guard([&] {
    need(h, "handle");
    *h = C(c).prefetch_issue(g);
  });
}

int dwdp_prefetch_query(dwdp_ctx* c, dwdp_prefetch h, int* done) {
  return guard([&] {
    need(done, "done");
    *done = C(c).prefetch_done(h) ? 1 : 0;
  });
}

int dwdp_prefetch_wait(dwdp_ctx* c, dwdp_prefetch h, void* stream) {
  return guard([&] { C(c).prefetch_wait(h, static_cast<cudaStream_t>(stream)); });
}

int dwdp_prefetch_times(dwdp_ctx* c, dwdp_prefetch h, int64_t* s, int64_t* e, double* b) {
  return guard([&] {
    int64_t s0, e0;
    double b0;
    C(c).prefetch_times(h, &s0, &e0, &b0);
    if (s) *s = s0;
    if (e) *e = e0;
    if (b) *b = b0;
  });
}

int dwdp_ctx_set_engine(dwdp_ctx* c, int engine) {
  return guard([&] {
    dwdp::require(engine == DWDP_ENGINE_COPY || engine == DWDP_ENGINE_PULL || engine == DWDP_ENGINE_HYBRID,
                  "ctx: unknown engine");
    auto& ctx = C(c);
    ctx.cfg.engine = engine;
    cudaSetDevice(ctx.cfg.device);
    dwdp::configure_max_shared_carveout_kernels(ctx.cfg.group_size > 1 && engine != DWDP_ENGINE_COPY);
  });
}

int dwdp_ctx_copy_plan(dwdp_ctx* c, dwdp_slice* out, size_t* n_inout) {
  return guard([&] {
    need(n_inout, "n_inout");
    const auto plan = C(c).copy_plan();
    const size_t cap = *n_inout;
    *n_inout = plan.size();
    if (!out) return;
    dwdp::require(cap >= plan.size(), "copy plan: output capacity too small");
    for (size_t i = 0; i < plan.size(); ++i)
      out[i] = {plan[i].param_id, plan[i].src_rank, 0, plan[i].src_offset, plan[i].dst_offset,
                plan[i].length};
  });
}

int dwdp_moe_forward(dwdp_ctx* c, int layer, const void* x, int64_t T, void* y, void* stream) {
  return guard([&] {
    if (T > 0) {
      need(x, "x");
      need(y, "y");
    }
    C(c).moe_forward_resident(layer, static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(y),
                              static_cast<cudaStream_t>(stream));
  });
}

int dwdp_layer_forward(dwdp_ctx* c, int64_t g, const void* x, int64_t T, void* y, int residual,
                       void* stream) {
  return guard([&] {
    if (T > 0) {
      need(x, "x");
      need(y, "y");
    }
    C(c).layer_forward(g, static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(y),
                       residual != 0, static_cast<cudaStream_t>(stream));
  });
}

int dwdp_stack_forward(dwdp_ctx* c, const void* x, int64_t T, void* y, void* stream) {
  return guard([&] {
    if (T > 0) {
      need(x, "x");
      need(y, "y");
    }
    C(c).stack_forward(static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(y),
                       static_cast<cudaStream_t>(stream));
  });
}

int dwdp_route(dwdp_ctx* c, int layer, const void* x, int64_t T, void* idx, void* wts,
               void* counts, void* row_of, int64_t* rows, void* stream) {
  return guard([&] {
    need(x, "x");
    C(c).route(layer, static_cast<const uint16_t*>(x), T, static_cast<int32_t*>(idx),
               static_cast<float*>(wts), static_cast<int32_t*>(counts),
               static_cast<int32_t*>(row_of), rows, static_cast<cudaStream_t>(stream));
  });
}

int dwdp_ctx_records(dwdp_ctx* c, dwdp_layer_record* out, size_t* n_inout) {
  return guard([&] {
    need(n_inout, "n_inout");
    *n_inout = C(c).drain_records(out, out ? *n_inout : 0);
  });
}

int dwdp_ctx_launch_count(const dwdp_ctx* c, int64_t* n) {
  return guard([&] {
    need(c, "ctx");
    need(n, "n");
    *n = c->impl->launches;
  });
}

int dwdp_nccl_unique_id(void* id) {
  return guard([&] {
    need(id, "id");
    dwdp::nccl_unique_id(id);
  });
}

int dwdp_dep_init(dwdp_ctx* c, const void* id) {
  return guard([&] {
    need(id, "nccl_id");
    C(c).dep_init(id);
  });
}

int dwdp_dep_set_mode(dwdp_ctx* c, int mode) {
  return guard([&] {
    dwdp::require(mode >= 0 && mode <= 2,
                  "dep: mode must be 0 (per-pair), 1 (token rows to every peer) or 2 (to the owning ranks)");
    C(c).dep_mode = mode;
  });
}

int dwdp_dep_layer_forward(dwdp_ctx* c, int layer, const void* x, int64_t T, void* y,
                           int residual, void* stream) {
  return guard([&] {
    if (T > 0) {
      need(x, "x");
      need(y, "y");
    }
    C(c).dep_layer_forward(layer, static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(y),
                           residual != 0, static_cast<cudaStream_t>(stream));
  });
}

int dwdp_dep_stack_forward(dwdp_ctx* c, const void* x, int64_t T, void* y, void* stream) {
  return guard([&] {
    if (T > 0) {
      need(x, "x");
      need(y, "y");
    }
    C(c).dep_stack_forward(static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(y),
                           static_cast<cudaStream_t>(stream));
  });
}

namespace {
// A throwaway context for the kernel-level entry points: the GEMM only needs
// TMA maps and tables (one per device).
dwdp::Ctx* tiny_ctx() {
  static dwdp::Ctx* tiny[64] = {nullptr};
  static std::mutex mu;  // several host threads (one per GPU) may call in
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!tiny[dev]) {
    dwdp_ctx_config cfg{};
    cfg.num_layers = 1;
    cfg.num_experts = 1;
    cfg.hidden = 256;
    cfg.ffn = 128;
    cfg.top_k = 1;
    cfg.scoring = 0;
    cfg.n_group = 1;
    cfg.topk_group = 1;
    cfg.routed_scale = 1.0f;
    cfg.group_size = 1;
    cfg.merge_elim = 1;
    cfg.max_tokens = 1;
    cfg.weight_layers = 1;
    cfg.device = dev;
    tiny[dev] = new dwdp::Ctx(cfg);
  }
  return tiny[dev];
}
}  // namespace

int dwdp_gemm_bf16(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K,
                   void* stream) {
  return guard([&] {
    need(A, "A");
    need(B, "B");
    need(D, "D");
    tiny_ctx()->gemm_bf16(static_cast<const uint16_t*>(A), static_cast<const uint16_t*>(B),
                          static_cast<uint16_t*>(D), M, N, K, static_cast<cudaStream_t>(stream));
  });
}

int dwdp_quant_nvfp4(const void* src, int64_t rows, int64_t K, void* codes, void* sf,
                     float* row_scale, void* stream) {
  return guard([&] {
    need(src, "src");
    need(codes, "codes");
    need(sf, "sf");
    need(row_scale, "row_scale");
    dwdp::require(rows >= 1 && K > 0 && K % 256 == 0, "quant_nvfp4: need rows >= 1, K % 256 == 0");
    void* lin = nullptr;
    if (cudaMalloc(&lin, size_t(rows) * size_t(K / 16)) != cudaSuccess)
      throw dwdp::CudaError("quant_nvfp4: scratch allocation failed");
    dwdp::launch_quant_rows_nvfp4(static_cast<const uint16_t*>(src), rows, K, nullptr,
                                  static_cast<uint8_t*>(codes), static_cast<uint8_t*>(lin),
                                  static_cast<uint8_t*>(sf), row_scale, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaFree(lin);
    if (e != cudaSuccess) throw dwdp::CudaError(cudaGetErrorString(e));
  });
}

int dwdp_gemm_nvfp4(const void* A, const void* A_sf, const float* A_scale, const void* B,
                    const void* B_sf, const float* B_scale, void* D, int64_t M, int64_t N, int64_t K,
                    void* stream) {
  return guard([&] {
    for (const void* p : {A, A_sf, static_cast<const void*>(A_scale), B, B_sf,
                          static_cast<const void*>(B_scale), static_cast<const void*>(D)})
      need(p, "operand");
    tiny_ctx()->gemm_nvfp4(static_cast<const uint8_t*>(A), static_cast<const uint8_t*>(A_sf), A_scale,
                           static_cast<const uint8_t*>(B), static_cast<const uint8_t*>(B_sf), B_scale,
                           static_cast<uint16_t*>(D), M, N, K, static_cast<cudaStream_t>(stream));
  });
}

int dwdp_fill_bf16(void* dst, int64_t n, uint64_t seed, float scale, void* stream) {
  return guard([&] {
    need(dst, "dst");
    dwdp::launch_fill(static_cast<uint16_t*>(dst), n, seed, scale,
                      static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw dwdp::CudaError(cudaGetErrorString(e));
  });
}

// ---- accounting ------------------------------------------------------------

namespace {

void copy_str(const std::string& s, char* buf, size_t* len) {
  const size_t cap = *len;
  *len = s.size() + 1;
  if (buf && cap >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
}

void finish_report(const dwdp::RunReport& rep, dwdp_breakdown* out) {
  rep.validate_streams();
  dwdp::breakdown_to_c(dwdp::breakdown(rep), rep.throughput_tokens_per_s(), out);
}

}  // namespace

int dwdp_report_breakdown(const dwdp_sim_event* ev, size_t n, int num_ranks, int iterations,
                          int warmup, const int64_t* is, const int64_t* ie, const int64_t* tk,
                          dwdp_breakdown* out) {
  return guard([&] {
    need(out, "out");
    need(is, "iter_start");
    need(ie, "iter_end");
    need(tk, "iter_tokens");
    dwdp::require(ev != nullptr || n == 0, "events: null");
    dwdp::require(num_ranks >= 1 && iterations >= 1 && warmup >= 0 && warmup < iterations,
                  "report: bad rank / iteration counts");
    dwdp::RunReport rep;
    rep.num_ranks = num_ranks;
    rep.iterations = iterations;
    rep.warmup_iterations = warmup;
    for (size_t i = 0; i < n; ++i) {
      const dwdp_sim_event& e = ev[i];
      dwdp::require(e.category >= 0 && e.category < DWDP_NUM_CATEGORIES, "report: bad category");
      dwdp::require(e.rank >= 0 && e.rank < num_ranks, "report: event rank out of range");
      rep.events.push_back({e.rank, static_cast<dwdp::Stream>(e.stream != 0),
                            static_cast<dwdp::Category>(e.category), e.start_ns, e.end_ns, e.layer,
                            e.iteration, e.bytes, e.detail});
    }
    const size_t nr = static_cast<size_t>(num_ranks), ni = static_cast<size_t>(iterations);
    rep.iter_start.assign(nr, std::vector<int64_t>(ni));
    rep.iter_end.assign(nr, std::vector<int64_t>(ni));
    rep.iter_tokens.assign(nr, std::vector<int64_t>(ni));
    for (size_t r = 0; r < nr; ++r)
      for (size_t i = 0; i < ni; ++i) {
        rep.iter_start[r][i] = is[r * ni + i];
        rep.iter_end[r][i] = ie[r * ni + i];
        rep.iter_tokens[r][i] = tk[r * ni + i];
      }
    finish_report(rep, out);
  });
}

int dwdp_report_from_records(const dwdp_layer_record* recs, const size_t* counts, int num_ranks,
                             int num_layers, int warmup, dwdp_breakdown* out,
                             dwdp_sim_event* events, size_t* n_events) {
  return guard([&] {
    need(recs, "records");
    need(counts, "counts");
    need(out, "out");
    dwdp::require(num_ranks >= 1 && num_layers >= 1 && warmup >= 0, "report: bad sizes");
    dwdp::RunReport rep;
    rep.num_ranks = num_ranks;
    rep.num_layers = num_layers;
    rep.warmup_iterations = warmup;
    size_t off = 0;
    for (int r = 0; r < num_ranks; ++r) {
      dwdp::append_rank_events(rep, r, recs + off, counts[r]);
      off += counts[r];
    }
    dwdp::require(warmup < rep.iterations, "report: warmup must leave a steady iteration");
    finish_report(rep, out);
    if (n_events) {
      const size_t cap = events ? *n_events : 0;
      for (size_t i = 0; i < rep.events.size() && i < cap; ++i) {
        const dwdp::SimEvent& e = rep.events[i];
        events[i] = {e.rank, static_cast<int32_t>(e.stream), static_cast<int32_t>(e.category), e.layer,
                     e.iteration, e.detail, e.start, e.end, e.bytes};
      }
      *n_events = rep.events.size();
    }
  });
}

int dwdp_compare_reports(const dwdp_breakdown* a, const dwdp_breakdown* b, dwdp_comparison* out) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    const dwdp::ComparisonTable t =
        dwdp::compare_reports(dwdp::breakdown_from_c(*a), dwdp::breakdown_from_c(*b));
    *out = dwdp_comparison{};
    for (const auto& row : t.rows) {
      const int i = static_cast<int>(row.category);
      out->a_us[i] = row.a_us;
      out->b_us[i] = row.b_us;
      out->has_delta[i] = row.delta_frac ? 1 : 0;
      out->delta_frac[i] = row.delta_frac ? *row.delta_frac : 0.0;
    }
    out->a_latency_us = t.a_latency_us;
    out->b_latency_us = t.b_latency_us;
    out->overall_frac = t.overall_frac;
    out->gross_sync_comm_pct = t.gross_sync_comm_pct;
  });
}

int dwdp_breakdown_csv(const dwdp_breakdown* b, char* buf, size_t* len) {
  return guard([&] {
    need(b, "breakdown");
    need(len, "len");
    copy_str(dwdp::breakdown_from_c(*b).to_csv(), buf, len);
  });
}

int dwdp_comparison_csv(const dwdp_comparison* c, char* buf, size_t* len) {
  return guard([&] {
    need(c, "comparison");
    need(len, "len");
    dwdp::ComparisonTable t;
    for (int i = 0; i < DWDP_NUM_CATEGORIES; ++i) {
      dwdp::ComparisonRow row{static_cast<dwdp::Category>(i), c->a_us[i], c->b_us[i], std::nullopt};
      if (c->has_delta[i]) row.delta_frac = c->delta_frac[i];
      t.rows.push_back(row);
    }
    t.a_latency_us = c->a_latency_us;
    t.b_latency_us = c->b_latency_us;
    t.overall_frac = c->overall_frac;
    t.gross_sync_comm_pct = c->gross_sync_comm_pct;
    copy_str(t.to_csv(), buf, len);
  });
}

}  // extern "C"
