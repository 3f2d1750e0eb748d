"""Python mirror of the reference's planning API (dwdpsim names, argument
meaning and error behaviour), each call going through libdwdp.so's C-ABI.

Reference: /root/reference/proj/include/dwdpsim/{placement,copyplan,workload,
modelspec,hwmodel,simcore}.hpp.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (AnalyticC, ConfigError, GpuSpecC, InvariantViolation, ModelSpecC, OpCostC, ShardRefC, SliceC,
                   WorkloadSpecC, check, lib)

# --------------------------------------------------------------------------- placement


@dataclass
class PlacementPlan:
    """include/dwdpsim/placement.hpp:13-25."""
    group_size: int = 0
    num_experts: int = 0
    local_count: int = 0
    redundancy: int = 0
    local_sets: list[list[int]] = field(default_factory=list)
    fetch_lists: list[list[tuple[int, int]]] = field(default_factory=list)

    def holds(self, rank: int, expert: int) -> bool:
        return expert in self.local_sets[rank]

    def validate(self) -> None:
        """Checks this plan's tables through the library (placement.cpp:15-45);
        InvariantViolation on any broken invariant."""
        with _Placement.from_plan(self):
            pass


class _Placement:
    def __init__(self, h):
        self.h = h

    @classmethod
    def build(cls, E: int, N: int, extra: int) -> "_Placement":
        h = C.c_void_p()
        check(lib().dwdp_placement_build(E, N, extra, C.byref(h)))
        return cls(h)

    @classmethod
    def from_plan(cls, plan: PlacementPlan) -> "_Placement":
        """Handle over this plan's own tables (validated)."""
        if len(plan.local_sets) != plan.group_size or len(plan.fetch_lists) != plan.group_size:
            raise InvariantViolation("placement: local_sets size mismatch")
        loffs = np.cumsum([0] + [len(s) for s in plan.local_sets]).astype(np.int32)
        foffs = np.cumsum([0] + [len(f) for f in plan.fetch_lists]).astype(np.int32)
        lflat = np.array([e for s in plan.local_sets for e in s] + [0], np.int32)
        fe = np.array([e for f in plan.fetch_lists for e, _ in f] + [0], np.int32)
        fs = np.array([s for f in plan.fetch_lists for _, s in f] + [0], np.int32)
        h = C.c_void_p()
        check(lib().dwdp_placement_from_tables(
            plan.group_size, plan.num_experts, plan.local_count, plan.redundancy,
            loffs.ctypes.data, lflat.ctypes.data, foffs.ctypes.data, fe.ctypes.data,
            fs.ctypes.data, C.byref(h)))
        return cls(h)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        lib().dwdp_placement_free(self.h)

    def to_plan(self) -> PlacementPlan:
        L = lib()
        n, e, c, r = (C.c_int32() for _ in range(4))
        check(L.dwdp_placement_info(self.h, C.byref(n), C.byref(e), C.byref(c), C.byref(r)))
        plan = PlacementPlan(n.value, e.value, c.value, r.value)
        for rank in range(n.value):
            ls = np.zeros(max(c.value, 1), np.int32)
            check(L.dwdp_placement_local_set(self.h, rank, ls.ctypes.data))
            plan.local_sets.append(ls[: c.value].tolist())
            m = e.value - c.value
            fe = np.zeros(max(m, 1), np.int32)
            fs = np.zeros(max(m, 1), np.int32)
            check(L.dwdp_placement_fetch_list(self.h, rank, fe.ctypes.data, fs.ctypes.data))
            plan.fetch_lists.append(list(zip(fe[:m].tolist(), fs[:m].tolist())))
        return plan


def build_placement(num_experts: int, group_size: int, extra_redundancy: int = 0) -> PlacementPlan:
    """placement.hpp:30-34 / src/placement.cpp:75-111."""
    with _Placement.build(num_experts, group_size, extra_redundancy) as p:
        return p.to_plan()


def assign_fetch_sources(num_experts: int, local_sets: list[list[int]]):
    """placement.hpp:36-39 / src/placement.cpp:47-73."""
    N = len(local_sets)
    offs = np.zeros(N + 1, np.int32)
    for r, s in enumerate(local_sets):
        offs[r + 1] = offs[r] + len(s)
    flat = np.array([e for s in local_sets for e in s] or [0], np.int32)
    counts = np.zeros(N, np.int32)
    fe = np.zeros(N * num_experts, np.int32)
    fs = np.zeros(N * num_experts, np.int32)
    check(lib().dwdp_assign_fetch_sources(num_experts, N, offs.ctypes.data, flat.ctypes.data,
                                          counts.ctypes.data, fe.ctypes.data, fs.ctypes.data))
    return [list(zip(fe[r * num_experts:r * num_experts + counts[r]].tolist(),
                     fs[r * num_experts:r * num_experts + counts[r]].tolist())) for r in range(N)]


def prefetch_bytes(plan: PlacementPlan, model: "MoeModelSpec") -> float:
    """src/placement.cpp:113-116."""
    return float(plan.num_experts - plan.local_count) * expert_shard_bytes(model)


def describe_placement(plan: PlacementPlan) -> str:
    with _Placement.from_plan(plan) as p:
        n = C.c_size_t(0)
        check(lib().dwdp_placement_describe(p.h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().dwdp_placement_describe(p.h, buf, C.byref(n)))
        return buf.value.decode()


# --------------------------------------------------------------------------- copy plan


@dataclass
class ShardRef:
    """copyplan.hpp:17-22."""
    peer: int = 0
    param_id: int = 0
    size: int = 0
    src_offset: int = 0


@dataclass
class Slice:
    """copyplan.hpp:24-30."""
    param_id: int = 0
    src_rank: int = 0
    src_offset: int = 0
    dst_offset: int = 0
    length: int = 0


@dataclass
class CopyPlan:
    """copyplan.hpp:33-38."""
    dst_rank: int = 0
    slice_size: int = 0
    slices: list[Slice] = field(default_factory=list)

    def total_bytes(self) -> int:
        return sum(s.length for s in self.slices)

    def to_csv(self) -> str:
        rows = ["param_id,src_rank,src_offset,dst_offset,length"]
        rows += [f"{s.param_id},{s.src_rank},{s.src_offset},{s.dst_offset},{s.length}"
                 for s in self.slices]
        return "\n".join(rows) + "\n"


def _slices_from_c(arr, n) -> list[Slice]:
    return [Slice(arr[i].param_id, arr[i].src_rank, arr[i].src_offset, arr[i].dst_offset,
                  arr[i].length) for i in range(n)]


def build_copy_plan(shards: list[ShardRef], slice_size: int, dst_rank: int = 0) -> CopyPlan:
    """copyplan.hpp:44-45 / src/copyplan.cpp:25-80."""
    if slice_size < 0 or any(s.size < 0 for s in shards):
        raise ConfigError("copy plan: negative sizes")
    arr = (ShardRefC * max(len(shards), 1))()
    for i, s in enumerate(shards):
        arr[i] = ShardRefC(s.peer, 0, s.param_id, s.size, s.src_offset)
    n = C.c_size_t(0)
    check(lib().dwdp_copy_plan_build(arr, len(shards), slice_size, dst_rank, None, C.byref(n)))
    out = (SliceC * max(n.value, 1))()
    check(lib().dwdp_copy_plan_build(arr, len(shards), slice_size, dst_rank, out, C.byref(n)))
    return CopyPlan(dst_rank, slice_size, _slices_from_c(out, n.value))


def source_queues(plans: list[CopyPlan], source: int) -> dict[int, list[Slice]]:
    """copyplan.hpp:47-51 / src/copyplan.cpp:82-92."""
    k = len(plans)
    arrs = [(SliceC * max(len(p.slices), 1))(*[SliceC(s.param_id, s.src_rank, 0, s.src_offset,
                                                      s.dst_offset, s.length) for s in p.slices])
            for p in plans]
    ptrs = (C.c_void_p * max(k, 1))(*[C.cast(a, C.c_void_p) for a in arrs])
    lens = (C.c_size_t * max(k, 1))(*[len(p.slices) for p in plans])
    dsts = (C.c_int32 * max(k, 1))(*[p.dst_rank for p in plans])
    nq, n = C.c_size_t(0), C.c_size_t(0)
    check(lib().dwdp_source_queues(k, dsts, ptrs, lens, source, None, None, C.byref(nq), None,
                                   C.byref(n)))
    out = (SliceC * max(n.value, 1))()
    odst = (C.c_int32 * max(nq.value, 1))()
    ocnt = (C.c_size_t * max(nq.value, 1))()
    check(lib().dwdp_source_queues(k, dsts, ptrs, lens, source, odst, ocnt, C.byref(nq), out,
                                   C.byref(n)))
    res, i = {}, 0
    flat = _slices_from_c(out, n.value)
    for q in range(nq.value):
        res[int(odst[q])] = flat[i:i + ocnt[q]]
        i += ocnt[q]
    return res


# --------------------------------------------------------------------------- workload


@dataclass
class IslDist:
    """workload.hpp:14-31."""
    kind: int = 0  # 0 Fixed, 1 UniformRatio, 2 Normal
    length: float = 8192
    ratio: float = 1.0
    stddev: float = 0.0

    @staticmethod
    def fixed(length):
        return IslDist(0, length)

    @staticmethod
    def uniform_ratio(max_length, ratio):
        return IslDist(1, max_length, ratio)

    @staticmethod
    def normal(mean, stddev):
        return IslDist(2, mean, 1.0, stddev)

    @staticmethod
    def from_cv(mean, cv):
        if cv < 0:
            raise ConfigError("workload.isl: cv must be >= 0")
        return IslDist.fixed(mean) if cv == 0 else IslDist.normal(mean, cv * mean)

    def cv(self) -> float:
        v = C.c_double()
        check(lib().dwdp_isl_cv(C.byref(_spec_c(WorkloadSpec(isl_dist=self))), C.byref(v)))
        return v.value


@dataclass
class WorkloadSpec:
    """workload.hpp:33-43."""
    isl_dist: IslDist = field(default_factory=IslDist)
    max_num_tokens: int = 32768
    batch_per_rank: int = 1
    routing_skew: float = 0.0
    seed: int = 1

    def validate(self) -> None:
        """src/workload.cpp:66-77 (+ IslDist::validate)."""
        check(lib().dwdp_workload_validate(C.byref(_spec_c(self))))


def _spec_c(w: WorkloadSpec) -> WorkloadSpecC:
    d = w.isl_dist
    return WorkloadSpecC(d.kind, w.batch_per_rank, d.length, d.ratio, d.stddev, w.max_num_tokens,
                         w.routing_skew, w.seed)


@dataclass
class CostCalibration:
    """modelspec.hpp:13-19: one scalar per category (1.0 = neutral)."""
    attention: float = 1.0
    grouped_gemm: float = 1.0
    dense_gemm: float = 1.0


@dataclass
class MoeModelSpec:
    """modelspec.hpp:22-40."""
    num_layers: int = 1
    hidden_dim: int = 0
    num_experts: int = 1
    top_k: int = 1
    expert_ffn_dim: int = 0
    shared_ffn_dim: int = 0
    weight_bytes_per_param: float = 2.0
    act_bytes_per_element: float = 2.0
    attn_proj_params: float = 0.0
    kv_bytes_per_token_per_layer: float = 0.0
    others_bytes_factor: float = 0.0
    calib: CostCalibration = field(default_factory=CostCalibration)

    def c(self) -> ModelSpecC:
        return ModelSpecC(self.num_layers, self.num_experts, self.hidden_dim, self.top_k, 0,
                          self.expert_ffn_dim, self.shared_ffn_dim, self.weight_bytes_per_param,
                          self.act_bytes_per_element, self.attn_proj_params,
                          self.kv_bytes_per_token_per_layer, self.others_bytes_factor,
                          self.calib.attention, self.calib.grouped_gemm, self.calib.dense_gemm)

    def validate(self) -> None:
        """src/modelspec.cpp:6-23."""
        check(lib().dwdp_model_validate(C.byref(self.c())))


def r1_model(layers: int = 8, weight_bytes: float = 2.0) -> MoeModelSpec:
    """DeepSeek-R1 MoE shapes (reference src/config.cpp:24-42: attention
    projection params 187e6, KV 576 B/token/layer); neutral calibration and
    no Others traffic, i.e. the uncalibrated roofline of the measured path."""
    return MoeModelSpec(layers, 7168, 256, 8, 2048, 2048, weight_bytes, 2.0,
                        attn_proj_params=187e6, kv_bytes_per_token_per_layer=576.0)


@dataclass
class RankBatch:
    """workload.hpp:45-55."""
    tokens: list[int]
    requests: list[int]
    routed: list[list[int]]

    def mean_seq_len(self, rank: int) -> int:
        if self.requests[rank] <= 0:
            return self.tokens[rank]
        return max(1, self.tokens[rank] // self.requests[rank])


def route_tokens(tokens: int, model: MoeModelSpec, routing_skew: float, seed: int) -> list[int]:
    """workload.hpp:57-65 / src/workload.cpp:85-111."""
    out = np.zeros(model.num_experts, np.int64)
    check(lib().dwdp_route_tokens(tokens, model.num_experts, model.top_k, routing_skew, seed,
                                  out.ctypes.data))
    return out.tolist()


def sample_batches(spec: WorkloadSpec, model: MoeModelSpec, num_ranks: int, iterations: int,
                   with_routing: bool = True) -> list[RankBatch]:
    """workload.hpp:67-73 / src/workload.cpp:137-173."""
    if num_ranks < 1 or iterations < 1:
        raise ConfigError("sample_batches: num_ranks and iterations must be >= 1")
    t = np.zeros(iterations * num_ranks, np.int64)
    q = np.zeros(iterations * num_ranks, np.int64)
    r = np.zeros(iterations * num_ranks * model.num_experts, np.int64) if with_routing else None
    check(lib().dwdp_sample_batches(C.byref(_spec_c(spec)), model.num_experts, model.top_k,
                                    num_ranks, iterations, t.ctypes.data, q.ctypes.data,
                                    None if r is None else r.ctypes.data))
    out = []
    for it in range(iterations):
        sl = slice(it * num_ranks, (it + 1) * num_ranks)
        routed = ([] if r is None else r.reshape(iterations, num_ranks, -1)[it].tolist())
        out.append(RankBatch(t[sl].tolist(), q[sl].tolist(), routed))
    return out


def batches_to_csv(batches: list[RankBatch]) -> str:
    """workload.hpp:77-78 / src/workload.cpp:191-208 (the reference's replay format)."""
    iters = len(batches)
    N = len(batches[0].tokens) if iters else 0
    E = len(batches[0].routed[0]) if iters and batches[0].routed and batches[0].routed[0] else 0
    t = np.array([b.tokens for b in batches] or [[0]], np.int64)
    q = np.array([b.requests for b in batches] or [[0]], np.int64)
    r = np.array([b.routed for b in batches], np.int64) if E else None
    n = C.c_size_t(0)
    L = lib()
    args = (t.ctypes.data, q.ctypes.data, None if r is None else r.ctypes.data, iters, N, E)
    check(L.dwdp_batches_to_csv(*args, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    check(L.dwdp_batches_to_csv(*args, buf, C.byref(n)))
    return buf.value.decode()


def batches_from_csv(csv: str) -> list[RankBatch]:
    """workload.hpp:79 / src/workload.cpp:210-247."""
    L = lib()
    raw = csv.encode()
    it, N, E = C.c_int32(), C.c_int32(), C.c_int32()
    check(L.dwdp_batches_from_csv(raw, C.byref(it), C.byref(N), C.byref(E), None, None, None, None))
    n = it.value * N.value
    t = np.zeros(max(n, 1), np.int64)
    q = np.zeros(max(n, 1), np.int64)
    r = np.zeros(max(n * E.value, 1), np.int64)
    ln = np.zeros(max(n, 1), np.int32)
    check(L.dwdp_batches_from_csv(raw, C.byref(it), C.byref(N), C.byref(E), t.ctypes.data,
                                  q.ctypes.data, r.ctypes.data, ln.ctypes.data))
    out = []
    for i in range(it.value):
        rows = slice(i * N.value, (i + 1) * N.value)
        routed = [r[(i * N.value + k) * E.value:(i * N.value + k) * E.value + ln[i * N.value + k]].tolist()
                  for k in range(N.value)]
        out.append(RankBatch(t[rows].tolist(), q[rows].tolist(), routed))
    return out


def imbalance_cv(batch: RankBatch) -> float:
    """src/workload.cpp:175-189."""
    a = np.asarray(batch.tokens, np.int64)
    v = C.c_double()
    check(lib().dwdp_imbalance_cv(a.ctypes.data, len(a), C.byref(v)))
    return v.value


# --------------------------------------------------------------------------- costs


def expert_shard_bytes(model: MoeModelSpec) -> float:
    """src/modelspec.cpp:32-36."""
    v = C.c_double()
    check(lib().dwdp_expert_shard_bytes(C.byref(model.c()), C.byref(v)))
    return v.value


@dataclass
class OpCost:
    category: str
    flops: float
    bytes: float


def _cat(i: int) -> str:
    return lib().dwdp_category_name(i).decode()


def _costs(arr, n) -> list[OpCost]:
    return [OpCost(_cat(arr[i].category), arr[i].flops, arr[i].bytes) for i in range(n.value)]


def attention_entries(model: MoeModelSpec, tokens: float, mean_seq_len: float) -> list[OpCost]:
    """src/modelspec.cpp:38-55."""
    out = (OpCostC * 4)()
    n = C.c_int32()
    check(lib().dwdp_attention_entries(C.byref(model.c()), tokens, mean_seq_len, out, C.byref(n)))
    return _costs(out, n)


def moe_entries(model: MoeModelSpec, tokens: float, routed_pairs: float,
                experts_touched: int) -> list[OpCost]:
    """src/modelspec.cpp:57-86."""
    out = (OpCostC * 4)()
    n = C.c_int32()
    check(lib().dwdp_moe_entries(C.byref(model.c()), tokens, routed_pairs, experts_touched, out,
                                 C.byref(n)))
    return _costs(out, n)


@dataclass
class LayerWork:
    """modelspec.hpp:43-50."""
    attn: list[OpCost]
    moe: list[OpCost]

    def total_time(self, gpu: "GpuSpec") -> float:
        return sum(roofline_time(op.flops, op.bytes, gpu) for op in self.attn + self.moe)


def layer_costs(model: MoeModelSpec, tokens: int, mean_seq_len: int) -> LayerWork:
    """src/modelspec.cpp:88-98."""
    a, m = (OpCostC * 4)(), (OpCostC * 4)()
    na, nm = C.c_int32(), C.c_int32()
    check(lib().dwdp_layer_costs(C.byref(model.c()), tokens, mean_seq_len, a, C.byref(na), m,
                                 C.byref(nm)))
    return LayerWork(_costs(a, na), _costs(m, nm))


@dataclass
class GpuSpec:
    """hwmodel.hpp:29-38 (defaults: measured B200 peaks, NVLink 5)."""
    peak_flops: float = 1649.8e12
    mem_bw: float = 6552.6e9
    link_bw: float = 900e9


def roofline_time(flops: float, bytes_: float, gpu: GpuSpec) -> float:
    """src/hwmodel.cpp:68-73."""
    v = C.c_double()
    check(lib().dwdp_roofline_time(flops, bytes_, C.byref(GpuSpecC(gpu.peak_flops, gpu.mem_bw,
                                                                   gpu.link_bw)), C.byref(v)))
    return v.value


def analytic_compare(model: MoeModelSpec, gpu: GpuSpec, placement: PlacementPlan,
                     tokens: int, mean_seq_len: int = 0) -> dict:
    """src/simcore.cpp:882-905; mean_seq_len = 0: the MoE block alone (the
    measured stack without attention)."""
    out = AnalyticC()
    with _Placement.from_plan(placement) as p:
        check(lib().dwdp_analytic_compare(C.byref(model.c()),
                                          C.byref(GpuSpecC(gpu.peak_flops, gpu.mem_bw, gpu.link_bw)),
                                          p.h, tokens, mean_seq_len, C.byref(out)))
    return {k: getattr(out, k) for k, _ in AnalyticC._fields_ if k != "reserved"}
