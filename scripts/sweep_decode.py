#!/usr/bin/env python
"""BASELINE config 5: decode-phase batch sweep with Zipf-skewed routing, fp8
expert weights, split-weight (merge_elim) vs merged-weight fetch, DWDP vs the
same-box DEP baseline. One bench.py run per point under torchrun; one JSON
line per point to --out.

    python scripts/sweep_decode.py --gpus 4 --batch 64,256,1024,4096 --zipf 0,0.8,1.2 \
        --out profiles/r1_sweep_decode_n4.jsonl
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
    ap.add_argument("--batch", default="64,256,1024,4096")
    ap.add_argument("--zipf", default="0,0.8,1.2")
    ap.add_argument("--fetch", default="split,merged")
    ap.add_argument("--dtype", default="fp8")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--extra", default="", help="extra bench.py flags")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep_decode.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    port = 29800
    with open(a.out, "a") as out:
        for fetch in a.fetch.split(","):
            for b in [int(t) for t in a.batch.split(",")]:
                for s in [float(z) for z in a.zipf.split(",")]:
                    port += 1
                    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
                           f"--master-port={port}", os.path.join(ROOT, "bench.py"),
                           f"--gpus={a.gpus}", f"--steps={a.steps}", f"--warmup={a.warmup}",
                           f"--decode={b}", f"--zipf={s}", f"--dtype={a.dtype}", "--no-e2e",
                           *(["--merged"] if fetch == "merged" else []), *a.extra.split()]
                    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
                    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
                    if r.returncode or not line:
                        rec = {"batch": b, "zipf": s, "fetch": fetch,
                               "error": (r.stdout + r.stderr)[-600:]}
                    else:
                        d = json.loads(line[-1])
                        dep = d.get("dep_baseline") or {}
                        rec = {"n_gpus": a.gpus, "dtype": a.dtype, "batch": b, "zipf": s,
                               "fetch": fetch,
                               "dwdp_ms_per_step": d["ms_per_step"],
                               "dep_ms_per_step": dep.get("ms_per_step"),
                               "dwdp_tokens_per_s_per_gpu": d["tokens_per_s_per_gpu"],
                               "dep_tokens_per_s_per_gpu": dep.get("tokens_per_s_per_gpu"),
                               "dwdp_over_dep": dep.get("dwdp_over_dep"),
                               "dep_mode1_ms_per_step": (dep.get("dedupe") or {}).get("ms_per_step"),
                               "dep_mode2_ms_per_step": (dep.get("dedupe_owners") or {}).get("ms_per_step"),
                               "dwdp_over_best_dep": dep.get("dwdp_over_best_dep"),
                               "dep_mode_errors": [x.get("error") for x in (dep.get("dedupe") or {}, dep.get("dedupe_owners") or {})
                                                   if x.get("error")],
                               "exposed_prefetch_ms_per_layer": d["exposed_prefetch_ms_per_layer"],
                               "merge_ms_per_layer": d.get("merge_ms_per_layer"),
                               "dep_comm_ms_per_layer": dep.get("comm_ms_per_layer"),
                               "routing": d.get("routing"),
                               "engine": d["config"].get("prefetch_engine"),
                               "prefetch_gbs": (d.get("prefetch") or {}).get("gbs"),
                               "step_roofline_frac": (d.get("step_roofline") or {}).get("frac"),
                           "clocks": d.get("clocks")}
                    out.write(json.dumps(rec) + "\n")
                    out.flush()
                    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
