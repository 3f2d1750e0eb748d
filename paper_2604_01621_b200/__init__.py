"""B200-native DWDP (Distributed Weight Data Parallelism) MoE hot path.

The drop-in boundary is the C-ABI in include/dwdp.h (libdwdp.so, sm_100a).
This package mirrors the reference operator API (dwdpsim names) on top of it.
"""
from ._lib import (ENGINE_COPY, ENGINE_HYBRID, ENGINE_PULL, WEIGHT_BF16, WEIGHT_FP8, WEIGHT_NVFP4, ConfigError, CudaError, InvariantViolation,  # noqa: F401
                   lib)
from .planning import (CopyPlan, CostCalibration, GpuSpec, LayerWork, attention_entries, batches_from_csv,
                       batches_to_csv, layer_costs, IslDist, MoeModelSpec, OpCost, PlacementPlan,  # noqa: F401
                       RankBatch, ShardRef, Slice, WorkloadSpec, analytic_compare,
                       assign_fetch_sources, build_copy_plan, build_placement,
                       describe_placement, expert_shard_bytes, imbalance_cv, moe_entries,
                       prefetch_bytes, r1_model, roofline_time, route_tokens, sample_batches,
                       source_queues)
from .runtime import DwdpConfig, DwdpContext, fill_bf16, gemm_bf16, gemm_nvfp4, nccl_unique_id, quant_nvfp4  # noqa: F401
