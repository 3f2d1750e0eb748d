"""Accounting over measured runs: SimEvent / RunReport / breakdown /
compare_reports (reference include/dwdpsim/simcore.hpp:29-61, 177-213;
src/simcore.cpp:18-63, 766-876), computed natively by libdwdp.so
(csrc/report.cpp) from CUDA-event timestamps instead of a simulated clock."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import NC, BreakdownC, ComparisonC, LayerRecordC, SimEventC, check, lib  # noqa: F401

CATEGORIES = ["Attention", "GroupedGEMM", "DenseGEMM", "Others", "Communication", "D2DCopy",
              "P2PCopy", "SyncWait"]  # hwmodel.hpp:14-23 order (DWDP_CAT_*)
DETAILS = {"": 0, "weight_wait": 1, "dispatch": 2, "combine": 3, "barrier": 4}


def _fn(name):
    return getattr(lib(), name)


@dataclass
class BreakdownTable:
    """BreakdownTable (simcore.hpp:177-188): mean us per rank and steady
    iteration by category, compute stream and copy stream separately."""
    compute_us: dict[str, float] = field(default_factory=dict)
    copy_us: dict[str, float] = field(default_factory=dict)
    iteration_latency_us: float = 0.0
    p2p_fully_overlapped: bool = False
    tokens_per_s: float = 0.0
    c: BreakdownC | None = None

    def category_us(self, name: str) -> float:
        return self.compute_us.get(name, self.copy_us.get(name, 0.0))

    def to_csv(self) -> str:
        return _csv("dwdp_breakdown_csv", self.c)

    def as_dict(self) -> dict:
        return {"compute_us": self.compute_us, "copy_us": self.copy_us,
                "iteration_latency_us": self.iteration_latency_us,
                "p2p_fully_overlapped": self.p2p_fully_overlapped,
                "tokens_per_s": self.tokens_per_s}


@dataclass
class ComparisonTable:
    rows: list[dict]
    a_latency_us: float
    b_latency_us: float
    overall_frac: float
    gross_sync_comm_pct: float
    c: ComparisonC | None = None

    def to_csv(self) -> str:
        return _csv("dwdp_comparison_csv", self.c)

    def as_dict(self) -> dict:
        return {"rows": self.rows, "a_latency_us": self.a_latency_us,
                "b_latency_us": self.b_latency_us, "overall_frac": self.overall_frac,
                "gross_sync_comm_pct": self.gross_sync_comm_pct}


def _csv(name: str, obj) -> str:
    n = C.c_size_t(0)
    check(_fn(name)(C.byref(obj), None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    check(_fn(name)(C.byref(obj), buf, C.byref(n)))
    return buf.value.decode()


def _table(b: BreakdownC) -> BreakdownTable:
    return BreakdownTable(
        compute_us={CATEGORIES[i]: b.compute_us[i] for i in range(NC) if b.compute_present[i]},
        copy_us={CATEGORIES[i]: b.copy_us[i] for i in range(NC) if b.copy_present[i]},
        iteration_latency_us=b.iteration_latency_us,
        p2p_fully_overlapped=bool(b.p2p_fully_overlapped), tokens_per_s=b.tokens_per_s, c=b)


def breakdown_events(events: np.ndarray, num_ranks: int, iterations: int, warmup: int,
                     iter_start, iter_end, iter_tokens) -> BreakdownTable:
    """breakdown(RunReport) over an explicit SimEventC array (validates the
    per-(rank, stream) no-overlap invariant first)."""
    ev = np.ascontiguousarray(events)
    arrs = [np.ascontiguousarray(a, np.int64).reshape(-1) for a in (iter_start, iter_end, iter_tokens)]
    out = BreakdownC()
    check(_fn("dwdp_report_breakdown")(ev.ctypes.data if len(ev) else None, len(ev), num_ranks,
                                       iterations, warmup, *[a.ctypes.data for a in arrs],
                                       C.byref(out)))
    return _table(out)


def events_dtype() -> np.dtype:
    return np.dtype([(n, np.int32) for n in ("rank", "stream", "category", "layer", "iteration",
                                              "detail")] +
                    [("start_ns", np.int64), ("end_ns", np.int64), ("bytes", np.float64)])


def report_from_records(records_per_rank: list[list[dict]], num_layers: int, warmup: int,
                        with_events: bool = False):
    """Measured run -> RunReport -> BreakdownTable. records_per_rank[r] are
    rank r's drained layer records (whole iterations of num_layers layers)."""
    flat = [rec for rr in records_per_rank for rec in rr]
    arr = (LayerRecordC * max(len(flat), 1))()
    for i, rec in enumerate(flat):
        for k, _ in LayerRecordC._fields_:
            setattr(arr[i], k, rec[k])
    counts = np.array([len(rr) for rr in records_per_rank], np.uint64)
    out = BreakdownC()
    n = C.c_size_t(0)
    fn = _fn("dwdp_report_from_records")
    check(fn(arr, counts.ctypes.data, len(records_per_rank), num_layers, warmup, C.byref(out),
             None, C.byref(n)))
    table = _table(out)
    if not with_events:
        return table
    ev = np.zeros(n.value, events_dtype())
    check(fn(arr, counts.ctypes.data, len(records_per_rank), num_layers, warmup, C.byref(out),
             ev.ctypes.data, C.byref(n)))
    return table, ev


def compare_reports(a: BreakdownTable, b: BreakdownTable) -> ComparisonTable:
    """compare_reports (simcore.cpp:822-854): per-category delta as a fraction
    of a's iteration latency; P2PCopy has no delta (off the critical path)."""
    out = ComparisonC()
    check(_fn("dwdp_compare_reports")(C.byref(a.c), C.byref(b.c), C.byref(out)))
    rows = [{"category": CATEGORIES[i], "a_us": out.a_us[i], "b_us": out.b_us[i],
             "delta_frac": out.delta_frac[i] if out.has_delta[i] else None} for i in range(NC)]
    return ComparisonTable(rows, out.a_latency_us, out.b_latency_us, out.overall_frac,
                           out.gross_sync_comm_pct, out)


DETAIL_NAMES = {v: k for k, v in DETAILS.items()}


def chrome_trace(events: np.ndarray) -> list[dict]:
    """Chrome trace of measured SimEvents, in the reference's layout
    (report_to_chrome_trace, src/report_io.cpp:58-76): one complete ("X")
    event per SimEvent, pid = rank, tid 0 compute / 1 copy stream, us."""
    out = []
    for e in events:
        cat = CATEGORIES[int(e["category"])]
        det = DETAIL_NAMES.get(int(e["detail"]), "")
        name = cat + (":" + det if det else "") + " L" + str(int(e["layer"]))
        out.append({"name": name, "cat": cat, "ph": "X", "ts": float(e["start_ns"]) / 1e3,
                    "dur": float(e["end_ns"] - e["start_ns"]) / 1e3, "pid": int(e["rank"]),
                    "tid": int(e["stream"]),
                    "args": {"iteration": int(e["iteration"]), "bytes": float(e["bytes"])}})
    return out
