#!/usr/bin/env python
"""Measured-trace -> simulator calibration loop.

Takes N>1 bench.py JSON lines (DWDP with its same-box DEP baseline), fits the
reference cost model's knobs to the measured per-kernel times, and re-runs the
COMPILED reference simulator (oracle/_ref: simulate_dwdp / simulate_dep,
/root/reference/proj/src/simcore.cpp:346-761) on the identical workload
(sample_batches with the bench's spec and seed) to print, beside every point,
the model's prediction against the measurement -- uncalibrated (nominal B200
envelope) and calibrated:

* GpuSpec.peak_flops = the measured sustained bf16 peak (MEASURED_PEAKS.json);
  CostCalibration.grouped_gemm = dense_gemm = measured GEMM1+GEMM2 time over
  the roofline time of their flops at that peak (one scalar per strategy: the
  DWDP value carries the interference of the concurrent NVLink pull);
* others_bytes_factor = measured router+permute+combine time over one
  activation pass at the HBM peak (modelspec.hpp:33-36);
* link_bw (DWDP) = fitted (a few simulator runs) so the model's P2PCopy
  time per layer equals the measured in-step prefetch time; link_bw (DEP) = the
  all-to-all bytes of simcore.cpp:321-324 over the measured dispatch+combine
  time per layer.

    python scripts/calibrate.py profiles/r1_bench_n4_end.json [...] [--out f.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (the compiled reference simulator)

R1 = dict(h=7168, E=256, k=8, f=2048, fs=2048)


def _peaks():
    p = {"hbm_gbs": 6544.0, "bf16_tflops_sustained": 1408.4}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in p if k in m})
    except (OSError, ValueError):
        pass
    return p


def _last_json(path):
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1])


def _predicted(rep, layers, N):
    """Per-layer means (ms) from a simulator report."""
    bd = rep["breakdown"]
    per_layer = lambda c: bd[c] / 1e3 / layers  # noqa: E731  (us per iteration -> ms per layer)
    i32, i64, _ = rep["events"]
    steady = i32[:, 4] >= rep["dims"][2]
    wait = (i32[:, 2] == 7) & (i32[:, 5] == 1) & steady  # SyncWait "weight_wait" (simcore.cpp:684-690)
    n_layers = max(1, (rep["dims"][1] - rep["dims"][2]) * layers * N)
    exposed = float((i64[wait, 1] - i64[wait, 0]).sum()) / 1e6 / n_layers
    return {"tokens_per_s": bd[34], "ms_per_step": bd[32] / 1e3,
            "moe_compute_ms_per_layer": per_layer(1) + per_layer(2) + per_layer(3),
            "comm_ms_per_layer": per_layer(4), "prefetch_ms_per_layer": bd[8 + 6] / 1e3 / layers,
            "exposed_ms_per_layer": exposed}


def calibrate(d: dict, ref, iters: int = 6, warmup: int = 2) -> dict:
    N = d["n_gpus"]
    c = d["config"]
    layers, mnt, cv = c["layers"], c["mnt_tokens_per_rank"], c["seq_len_cv"]
    dep = d.get("dep_baseline")
    assert N > 1 and dep, "needs an N>1 line with its DEP baseline"
    wb = 2.0 if d["dtype"] == "bf16" else 1.0 if d["dtype"].startswith("e4m3") else 0.5 + 1 / 16
    pk = _peaks()
    P = pk["bf16_tflops_sustained"] * 1e12 * (2.0 / wb if wb < 2 else 1.0)  # nominal fp8/fp4 rate
    bw = pk["hbm_gbs"] * 1e9
    h, E, k, f, fs = R1["h"], R1["E"], R1["k"], R1["f"], R1["fs"]
    tok = d["value"] * d["ms_per_step"] / 1e3 / N          # mean tokens per rank per step
    flops = 2 * tok * 3 * h * (k * f + fs)                  # routed + shared, per layer
    act = tok * h * 2.0

    def fit(kms, comm_ms=None, link=None):
        gemm = (kms["gemm1"] + kms["gemm2"]) / 1e3
        other = (kms["router"] + kms["permute"] + kms["combine"]) / 1e3
        cal = {"peak_flops": P, "mem_bw": bw, "ce_inflight": 2,
               "grouped_gemm": gemm / (flops / P), "dense_gemm": gemm / (flops / P),
               "others_bytes_factor": other * bw / act, "mem_interference": 0}
        if comm_ms is not None:  # DEP: all2all_oneway_bytes = T k h act each way
            cal["link_bw"] = 2 * tok * k * h * 2.0 / (comm_ms / 1e3)
        else:
            cal["link_bw"] = link
        return cal

    nominal = {"peak_flops": P, "mem_bw": bw, "link_bw": 900e9, "ce_inflight": 2, "grouped_gemm": 1.0,
               "dense_gemm": 1.0, "others_bytes_factor": 0.0, "mem_interference": 0}
    cal_dwdp = fit(d["kernel_ms_per_layer"], link=(d["prefetch"] or {}).get("gbs", 900) * 1e9)
    cal_dep = fit(dep["kernel_ms_per_layer"], comm_ms=dep["comm_ms_per_layer"])
    spec = (2 if cv > 0 else 0, 8192.0, 1.0, cv * 8192, mnt, max(1, mnt // 8192), 7)
    slice_size = c.get("slice_size") or (1 << 20)

    def sim(dwdp, cal):
        rep = ref.simulate_report_cal(0, dwdp, layers, h, E, k, f, fs, wb, cal, N, iters, warmup, *spec,
                                      tdm=True, slice_size=slice_size, merge_elim=True)
        return _predicted(rep, layers, N)

    measured = {
        "dwdp": {"tokens_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                 "moe_compute_ms_per_layer": d["kernel_ms_per_layer"]["moe"],
                 "prefetch_ms_per_layer": d["kernel_ms_per_layer"]["prefetch"],
                 "exposed_ms_per_layer": d["exposed_prefetch_ms_per_layer"]},
        "dep": {"tokens_per_s": dep["value"], "ms_per_step": dep["ms_per_step"],
                "comm_ms_per_layer": dep["comm_ms_per_layer"],
                "moe_compute_ms_per_layer": sum(dep["kernel_ms_per_layer"].values())},
    }
    # The simulator's copy engine shares each source port between its
    # destinations (max-min fair, ce_inflight queues): refit link_bw so its
    # P2PCopy time per layer equals the measured in-step prefetch time.
    p_dwdp = sim(True, cal_dwdp)
    meas_pf = d["kernel_ms_per_layer"]["prefetch"]
    for _ in range(3):
        if p_dwdp["prefetch_ms_per_layer"] <= 0 or meas_pf <= 0:
            break
        cal_dwdp["link_bw"] *= p_dwdp["prefetch_ms_per_layer"] / meas_pf
        p_dwdp = sim(True, cal_dwdp)
    pred = {"nominal": {"dwdp": sim(True, nominal), "dep": sim(False, nominal)},
            "calibrated": {"dwdp": p_dwdp, "dep": sim(False, cal_dep)}}
    out = {"n_gpus": N, "mnt": mnt, "cv": cv, "dtype": d["dtype"], "layers": layers,
           "tokens_per_rank_mean": tok, "calibration": {"dwdp": cal_dwdp, "dep": cal_dep},
           "measured": measured, "predicted": pred,
           "dwdp_over_dep": {"measured": d["value"] / dep["value"]},
           # GEMM time per flop in DWDP (NVLink pull running) over DEP (no pull)
           "interference_gemm_slowdown": cal_dwdp["grouped_gemm"] / cal_dep["grouped_gemm"]}
    for kind in ("nominal", "calibrated"):
        p = pred[kind]
        out["dwdp_over_dep"][kind] = p["dwdp"]["tokens_per_s"] / p["dep"]["tokens_per_s"]
        out.setdefault("error_pct", {})[kind] = {
            s: (p[s]["tokens_per_s"] / measured[s]["tokens_per_s"] - 1) * 100 for s in ("dwdp", "dep")}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lines", nargs="+", help="bench.py JSON files (N>1, DEP baseline on)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ref = O.ref()
    assert ref is not None, "oracle/_ref (the compiled reference) is not built"
    res = []
    for path in a.lines:
        r = calibrate(_last_json(path), ref)
        r["source"] = os.path.relpath(path, ROOT)
        res.append(r)
        print(json.dumps({k: r[k] for k in ("source", "n_gpus", "mnt", "cv", "dwdp_over_dep", "error_pct",
                                            "interference_gemm_slowdown")}))
    if a.out:
        with open(a.out, "w") as f:
            for r in res:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
