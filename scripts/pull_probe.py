#!/usr/bin/env python
"""Prefetch-engine probe on two GPUs of one process: rank 0 pulls one R1
layer's remote experts (128 experts x gate/up/down, 11.3 GB bf16) from rank 1
over NVLink with the chosen engine; prints achieved GB/s per plan. Used for
the ncu capture of the TMA pull kernel (one process, so ncu sees every
launch) and for engine GB/s numbers in DESIGN.md.

    python scripts/pull_probe.py --engine pull --plans 4
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2604_01621_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engine", default="pull", choices=["pull", "copy", "hybrid"])
    ap.add_argument("--plans", type=int, default=4)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp8"])
    ap.add_argument("--slice-size", type=int, default=64 << 20)
    ap.add_argument("--gpus", type=int, default=2, help="ranks (one per GPU), all pulling at once")
    ap.add_argument("--with-compute", type=int, default=0,
                    help="T tokens of MoE forward on GPU 0 while each plan runs (in-step contention)")
    a = ap.parse_args()
    assert torch.cuda.device_count() >= a.gpus >= 2, f"needs {a.gpus} GPUs"
    eng = {"pull": D.ENGINE_PULL, "copy": D.ENGINE_COPY, "hybrid": D.ENGINE_HYBRID}[a.engine]
    ctxs = [D.DwdpContext(D.DwdpConfig(num_layers=2, rank=r, group_size=a.gpus, device=r, engine=eng,
                                       slice_size=a.slice_size, weight_layers=2,
                                       max_tokens=max(128, a.with_compute),
                                       weight_dtype=D.WEIGHT_FP8 if a.dtype == "fp8" else
                                       D.WEIGHT_BF16))
            for r in range(a.gpus)]
    for c in ctxs:
        c.init_weights()
    D.DwdpContext.link_local(ctxs)
    torch.cuda.synchronize(0)
    res = []
    x = None
    if a.with_compute:
        x = torch.empty((a.with_compute, 7168), dtype=torch.bfloat16, device="cuda:0")
        D.fill_bf16(x, 7, 1.0)
        ctxs[0].moe_forward(0, x)
        torch.cuda.synchronize(0)
    for g in range(1, a.plans + 1):  # layer 0 is preloaded
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        hs = [c.prefetch_issue(g) for c in ctxs]  # every rank pulls its plan at once
        h = hs[0]
        if x is not None:  # the same device's MoE GEMMs run while the plan streams
            for _ in range(2):
                ctxs[0].moe_forward(0, x)
        ev[1].record()
        ctxs[0].prefetch_wait(h)
        for r in range(a.gpus):
            torch.cuda.synchronize(r)
        others = []
        for r in range(1, a.gpus):
            s2, e2, b2 = ctxs[r].prefetch_times(hs[r])
            others.append(round(b2 / (e2 - s2)))
        s, e, b = ctxs[0].prefetch_times(h)
        res.append({"plan": g, "bytes": b, "ms": (e - s) / 1e6, "gbs": b / (e - s), "other_ranks_gbs": others,
                    "compute_ms": ev[0].elapsed_time(ev[1]) if x is not None else None})
    print(json.dumps({"engine": a.engine, "dtype": a.dtype, "slice_size": a.slice_size,
                      "plans": res}), flush=True)
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    main()
