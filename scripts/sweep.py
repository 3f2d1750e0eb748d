#!/usr/bin/env python
"""BASELINE config 4: prefill imbalance sweep (ISL 8K, seq-len CV 0-0.3) at
N GPUs, DWDP vs the same-box DEP baseline. Runs bench.py once per point under
torchrun and writes one JSON line per point to --out.

    python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 \
        --out profiles/r1_sweep_n4.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--cv", default="0,0.1,0.2,0.3")
    ap.add_argument("--tokens", default="32768,65536")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--extra", default="", help="extra bench.py flags")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    port = 29700
    with open(a.out, "a") as out:
        for mnt in [int(t) for t in a.tokens.split(",")]:
            for cv in [float(c) for c in a.cv.split(",")]:
                port += 1
                cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                       f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
                       f"--master-port={port}", os.path.join(ROOT, "bench.py"),
                       f"--gpus={a.gpus}", f"--steps={a.steps}", f"--warmup={a.warmup}",
                       f"--cv={cv}", f"--tokens={mnt}", "--no-e2e", *a.extra.split()]
                r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
                line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
                if r.returncode or not line:
                    rec = {"cv": cv, "mnt": mnt, "error": (r.stdout + r.stderr)[-600:]}
                else:
                    d = json.loads(line[-1])
                    dep = d.get("dep_baseline") or {}
                    rec = {"n_gpus": a.gpus, "cv": cv, "mnt": mnt,
                           "dwdp_tokens_per_s_per_gpu": d["tokens_per_s_per_gpu"],
                           "dep_tokens_per_s_per_gpu": dep.get("tokens_per_s_per_gpu"),
                           "dwdp_over_dep": dep.get("dwdp_over_dep"),
                           "dep_mode1_tokens_per_s_per_gpu": (dep.get("dedupe") or {}).get("tokens_per_s_per_gpu"),
                           "dep_mode2_tokens_per_s_per_gpu": (dep.get("dedupe_owners") or {}).get(
                               "tokens_per_s_per_gpu"),
                           "dwdp_over_best_dep": dep.get("dwdp_over_best_dep"),
                           "dwdp_independent_ranks_per_gpu": (d.get("value_independent_ranks") or 0) / a.gpus
                           or None,
                           "exposed_prefetch_ms_per_layer": d["exposed_prefetch_ms_per_layer"],
                           "dep_comm_ms_per_layer": dep.get("comm_ms_per_layer"),
                           "engine": d["config"].get("prefetch_engine"),
                           "prefetch_gbs": (d.get("prefetch") or {}).get("gbs"),
                           "step_roofline_frac": (d.get("step_roofline") or {}).get("frac"),
                           "attention_ms_per_layer": (d.get("attention") or {}).get("ms_per_layer"),
                           "moe_ms_per_layer": (d.get("kernel_ms_per_layer") or {}).get("moe"),
                           "extra": a.extra,
                           "clocks": d.get("clocks")}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
