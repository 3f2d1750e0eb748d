"""ctypes binding of libdwdp.so (include/dwdp.h). Fails loudly when the
library is missing: there is no Python or CPU fallback for the hot path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdwdp.so")

i32, i64, u64, f32, f64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_size_t
P = C.c_void_p

DWDP_OK, DWDP_ERR_CONFIG, DWDP_ERR_INVARIANT, DWDP_ERR_CUDA = 0, 2, 3, 4
IPC_BLOB_BYTES = 1024
ENGINE_COPY, ENGINE_PULL, ENGINE_HYBRID = 0, 1, 2
WEIGHT_BF16, WEIGHT_FP8, WEIGHT_NVFP4 = 0, 1, 2


class ConfigError(ValueError):
    """Invalid user input (reference include/dwdpsim/errors.hpp:11-15, exit 2)."""


class InvariantViolation(AssertionError):
    """Internal invariant broken (errors.hpp:17-21, exit 3)."""


class CudaError(RuntimeError):
    """CUDA / device failure (status 4)."""


class ShardRefC(C.Structure):
    _fields_ = [("peer", i32), ("reserved", i32), ("param_id", u64), ("size", u64),
                ("src_offset", u64)]


class SliceC(C.Structure):
    _fields_ = [("param_id", u64), ("src_rank", i32), ("reserved", i32), ("src_offset", u64),
                ("dst_offset", u64), ("length", u64)]


class WorkloadSpecC(C.Structure):
    _fields_ = [("isl_kind", i32), ("batch_per_rank", i32), ("length", f64), ("ratio", f64),
                ("stddev", f64), ("max_num_tokens", i64), ("routing_skew", f64), ("seed", u64)]


class ModelSpecC(C.Structure):
    _fields_ = [("num_layers", i32), ("num_experts", i32), ("hidden_dim", i64), ("top_k", i32),
                ("reserved", i32), ("expert_ffn_dim", i64), ("shared_ffn_dim", i64),
                ("weight_bytes_per_param", f64), ("act_bytes_per_element", f64),
                ("attn_proj_params", f64), ("kv_bytes_per_token_per_layer", f64),
                ("others_bytes_factor", f64), ("calib_attention", f64),
                ("calib_grouped_gemm", f64), ("calib_dense_gemm", f64)]


class GpuSpecC(C.Structure):
    _fields_ = [("peak_flops", f64), ("mem_bw", f64), ("link_bw", f64)]


class OpCostC(C.Structure):
    _fields_ = [("category", i32), ("layer", i32), ("flops", f64), ("bytes", f64), ("ns", f64)]


class AnalyticC(C.Structure):
    _fields_ = [("t_compute_s", f64), ("t_prefetch_s", f64), ("t_all2all_s", f64),
                ("compute_prefetch_ratio", f64), ("dep_dwdp_speedup", f64),
                ("prefetch_saturated", i32), ("reserved", i32)]


class CtxConfigC(C.Structure):
    _fields_ = [("num_layers", i32), ("num_experts", i32), ("hidden", i64), ("ffn", i64),
                ("shared_ffn", i64), ("top_k", i32), ("scoring", i32), ("n_group", i32),
                ("topk_group", i32), ("norm_topk", i32), ("routed_scale", f32), ("rank", i32),
                ("group_size", i32), ("extra_redundancy", i32), ("device", i32),
                ("merge_elim", i32), ("tdm", i32), ("slice_size", u64), ("engine", i32),
                ("pull_ctas", i32), ("ce_inflight", i32), ("weight_dtype", i32),
                ("weight_seed", u64), ("weight_layers", i32),
                ("kernel_timing", i32), ("max_tokens", i64)]


class LayerRecordC(C.Structure):
    _fields_ = [("global_layer", i64), ("tokens", i64), ("gate_wait_ns", f64), ("moe_ns", f64),
                ("prefetch_ns", f64), ("prefetch_bytes", f64), ("merge_ns", f64),
                ("router_ns", f64), ("permute_ns", f64), ("gemm1_ns", f64), ("gemm2_ns", f64),
                ("combine_ns", f64), ("routed_rows", i64), ("comm_ns", f64),
                ("dispatch_ns", f64), ("start_ns", f64), ("end_ns", f64),
                ("prefetch_start_ns", f64), ("prefetch_end_ns", f64)]


class MlaConfigC(C.Structure):
    _fields_ = [("hidden", i32), ("heads", i32), ("q_lora", i32), ("kv_lora", i32), ("nope", i32),
                ("rope", i32), ("v_dim", i32), ("device", i32), ("max_tokens", i64),
                ("rope_theta", f32), ("softmax_scale", f32)]


class MlaWeightsC(C.Structure):
    _fields_ = [("wq_a", P), ("wq_b", P), ("wkv_a", P), ("wkv_b", P), ("wo", P)]


NC = 8  # DWDP_NUM_CATEGORIES


class SimEventC(C.Structure):
    _fields_ = [("rank", i32), ("stream", i32), ("category", i32), ("layer", i32),
                ("iteration", i32), ("detail", i32), ("start_ns", i64), ("end_ns", i64),
                ("bytes", f64)]


class BreakdownC(C.Structure):
    _fields_ = [("compute_us", f64 * NC), ("copy_us", f64 * NC), ("compute_present", i32 * NC),
                ("copy_present", i32 * NC), ("iteration_latency_us", f64),
                ("p2p_fully_overlapped", i32), ("reserved", i32), ("tokens_per_s", f64)]


class ComparisonC(C.Structure):
    _fields_ = [("a_us", f64 * NC), ("b_us", f64 * NC), ("delta_frac", f64 * NC),
                ("has_delta", i32 * NC), ("a_latency_us", f64), ("b_latency_us", f64),
                ("overall_frac", f64), ("gross_sync_comm_pct", f64)]


# name -> (restype, argtypes); every int-returning entry is a status code.
SIGNATURES = {
    "dwdp_last_error": (C.c_char_p, []),
    "dwdp_version": (C.c_char_p, []),
    "dwdp_placement_build": (i32, [i32, i32, i32, C.POINTER(P)]),
    "dwdp_placement_free": (None, [P]),
    "dwdp_placement_info": (i32, [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                  C.POINTER(i32)]),
    "dwdp_placement_local_set": (i32, [P, i32, P]),
    "dwdp_placement_fetch_list": (i32, [P, i32, P, P]),
    "dwdp_placement_holds": (i32, [P, i32, i32, C.POINTER(i32)]),
    "dwdp_placement_validate": (i32, [P]),
    "dwdp_prefetch_bytes": (i32, [P, f64, C.POINTER(f64)]),
    "dwdp_placement_describe": (i32, [P, C.c_char_p, C.POINTER(sz)]),
    "dwdp_assign_fetch_sources": (i32, [i32, i32, P, P, P, P, P]),
    "dwdp_copy_plan_build": (i32, [P, sz, u64, i32, P, C.POINTER(sz)]),
    "dwdp_source_queues": (i32, [sz, P, P, P, i32, P, P, C.POINTER(sz), P, C.POINTER(sz)]),
    "dwdp_rng_mix": (u64, [u64, u64]),
    "dwdp_route_tokens": (i32, [i64, i32, i32, f64, u64, P]),
    "dwdp_sample_batches": (i32, [C.POINTER(WorkloadSpecC), i32, i32, i32, i32, P, P, P]),
    "dwdp_imbalance_cv": (i32, [P, i32, C.POINTER(f64)]),
    "dwdp_isl_cv": (i32, [C.POINTER(WorkloadSpecC), C.POINTER(f64)]),
    "dwdp_workload_validate": (i32, [C.POINTER(WorkloadSpecC)]),
    "dwdp_batches_to_csv": (i32, [P, P, P, i32, i32, i32, C.c_char_p, C.POINTER(sz)]),
    "dwdp_batches_from_csv": (i32, [C.c_char_p, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                    P, P, P, P]),
    "dwdp_placement_from_tables": (i32, [i32, i32, i32, i32, P, P, P, P, P, C.POINTER(P)]),
    "dwdp_category_name": (C.c_char_p, [i32]),
    "dwdp_model_validate": (i32, [C.POINTER(ModelSpecC)]),
    "dwdp_expert_shard_bytes": (i32, [C.POINTER(ModelSpecC), C.POINTER(f64)]),
    "dwdp_attention_entries": (i32, [C.POINTER(ModelSpecC), f64, f64, P, C.POINTER(i32)]),
    "dwdp_moe_entries": (i32, [C.POINTER(ModelSpecC), f64, f64, i32, P, C.POINTER(i32)]),
    "dwdp_layer_costs": (i32, [C.POINTER(ModelSpecC), i64, i64, P, C.POINTER(i32), P,
                               C.POINTER(i32)]),
    "dwdp_roofline_time": (i32, [f64, f64, C.POINTER(GpuSpecC), C.POINTER(f64)]),
    "dwdp_analytic_compare": (i32, [C.POINTER(ModelSpecC), C.POINTER(GpuSpecC), P, i64, i64,
                                    C.POINTER(AnalyticC)]),
    "dwdp_ctx_create": (i32, [C.POINTER(CtxConfigC), C.POINTER(P)]),
    "dwdp_ctx_destroy": (i32, [P]),
    "dwdp_ctx_memory": (i32, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "dwdp_ctx_export_ipc": (i32, [P, P]),
    "dwdp_ctx_open_peers": (i32, [P, P]),
    "dwdp_ctx_link_local": (i32, [P, i32]),
    "dwdp_ctx_init_weights": (i32, [P, f32]),
    "dwdp_ctx_set_bias": (i32, [P, P]),
    "dwdp_ctx_read_expert": (i32, [P, i32, i32, i32, P]),
    "dwdp_prefetch_issue": (i32, [P, i64, C.POINTER(i64)]),
    "dwdp_prefetch_query": (i32, [P, i64, C.POINTER(i32)]),
    "dwdp_prefetch_wait": (i32, [P, i64, P]),
    "dwdp_prefetch_times": (i32, [P, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(f64)]),
    "dwdp_ctx_set_engine": (i32, [P, i32]),
    "dwdp_ctx_copy_plan": (i32, [P, P, C.POINTER(sz)]),
    "dwdp_moe_forward": (i32, [P, i32, P, i64, P, P]),
    "dwdp_layer_forward": (i32, [P, i64, P, i64, P, i32, P]),
    "dwdp_stack_forward": (i32, [P, P, i64, P, P]),
    "dwdp_route": (i32, [P, i32, P, i64, P, P, P, P, C.POINTER(i64), P]),
    "dwdp_ctx_records": (i32, [P, P, C.POINTER(sz)]),
    "dwdp_ctx_launch_count": (i32, [P, C.POINTER(i64)]),
    "dwdp_nccl_unique_id": (i32, [P]),
    "dwdp_dep_init": (i32, [P, P]),
    "dwdp_dep_set_mode": (i32, [P, i32]),
    "dwdp_dep_layer_forward": (i32, [P, i32, P, i64, P, i32, P]),
    "dwdp_dep_stack_forward": (i32, [P, P, i64, P, P]),
    "dwdp_mla_create": (i32, [C.POINTER(MlaConfigC), C.POINTER(P)]),
    "dwdp_mla_destroy": (i32, [P]),
    "dwdp_mla_forward": (i32, [P, C.POINTER(MlaWeightsC), P, i64, P, i32, P, P]),
    "dwdp_mla_launch_count": (i32, [P, C.POINTER(i64)]),
    "dwdp_gemm_bf16": (i32, [P, P, P, i64, i64, i64, P]),
    "dwdp_quant_nvfp4": (i32, [P, i64, i64, P, P, P, P]),
    "dwdp_gemm_nvfp4": (i32, [P, P, P, P, P, P, P, i64, i64, i64, P]),
    "dwdp_fill_bf16": (i32, [P, i64, u64, f32, P]),

    "dwdp_report_breakdown": (i32, [P, sz, i32, i32, i32, P, P,
                                    P, C.POINTER(BreakdownC)]),
    "dwdp_report_from_records": (i32, [P, P, i32, i32, i32,
                                       C.POINTER(BreakdownC), P,
                                       C.POINTER(sz)]),
    "dwdp_compare_reports": (i32, [C.POINTER(BreakdownC), C.POINTER(BreakdownC),
                                   C.POINTER(ComparisonC)]),
    "dwdp_breakdown_csv": (i32, [C.POINTER(BreakdownC), C.c_char_p, C.POINTER(sz)]),
    "dwdp_comparison_csv": (i32, [C.POINTER(ComparisonC), C.c_char_p, C.POINTER(sz)]),
}

_lib = None


def lib():
    """Load libdwdp.so (building it first in a source checkout)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _b
        _b.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdwdp.so not found at {LIB_PATH}; run python -m paper_2604_01621_b200.build")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status == DWDP_OK:
        return
    msg = lib().dwdp_last_error().decode(errors="replace")
    if status == DWDP_ERR_CONFIG:
        raise ConfigError(msg)
    if status == DWDP_ERR_INVARIANT:
        raise InvariantViolation(msg)
    raise CudaError(msg)
