#!/usr/bin/env python
"""DWDP independence on hardware (the paper's "no synchronisation" claim).

Reference: tests/test_simcore.cpp:276-311 and acceptance criterion 6
(tests/acceptance_main.cpp:258-319) perturb ONE rank's batch and require every
other rank's event timeline to be unchanged in the simulator. Here, on real
GPUs (torchrun, one process per GPU, R1-shaped 8-layer stack):

  A1  every rank T0 tokens per step                    (baseline)
  B   rank N-1 gets `--factor` x T0 tokens, others T0  (perturbed peer)
  A2  baseline again                                   (run-to-run noise)

for DWDP (layer_forward: owned experts + one-sided IPC pulls, no collective)
and for the DEP baseline (same kernels + NCCL all-to-alls). Reported for rank
0 from its own CUDA events: step time, per-layer MoE time, weight_wait and the
per-layer start offsets inside the step. DWDP's rank-0 numbers should move by
no more than the A1/A2 noise; DEP's rank-0 step stretches to the slow peer.

    torchrun --nproc-per-node 2 scripts/independence.py [--tokens 32768 --factor 2]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_01621_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--factor", type=float, default=2.0)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    T0 = a.tokens
    Tmax = int(T0 * a.factor)
    ctx = D.DwdpContext(D.DwdpConfig(num_layers=a.layers, rank=rank, group_size=world, device=local,
                                     weight_layers=a.layers, kernel_timing=1, max_tokens=Tmax,
                                     slice_size=64 << 20))
    ctx.init_weights()
    blobs = [None] * world
    dist.all_gather_object(blobs, ctx.export_ipc())
    ctx.open_peers(b"".join(blobs))
    ids = [D.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    ctx.dep_init(ids[0])
    x = torch.empty((Tmax, 7168), dtype=torch.bfloat16, device=dev)
    D.fill_bf16(x, 0xC0FFEE + rank, 1.0)
    y = torch.empty_like(x)
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    dist.barrier()

    def scenario(mode, perturbed):
        T = int(T0 * a.factor) if (perturbed and rank == world - 1) else T0
        fwd = ctx.dep_stack_forward if mode == "dep" else ctx.stack_forward
        for _ in range(a.warmup):
            fwd(x[:T], y[:T])
        torch.cuda.synchronize()
        ctx.records()
        dist.barrier()
        evs = []
        for _ in range(a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fwd(x[:T], y[:T])
            e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        recs = ctx.records()
        dist.barrier()
        L = a.layers
        steps = [recs[i * L:(i + 1) * L] for i in range(a.steps)]
        offs = [[(r["start_ns"] - s[0]["start_ns"]) / 1e6 for r in s] for s in steps]
        mean = lambda v: sum(v) / max(len(v), 1)  # noqa: E731
        return {"tokens_rank0": T0 if rank == 0 else None, "tokens_this_rank": T,
                "step_ms": mean([e0.elapsed_time(e1) for e0, e1 in evs]),
                "moe_ms_per_layer": mean([r["moe_ns"] for r in recs]) / 1e6,
                "weight_wait_ms_per_layer": mean([r["gate_wait_ns"] for r in recs]) / 1e6,
                "comm_ms_per_layer": mean([r["comm_ns"] for r in recs]) / 1e6,
                "layer_start_offsets_ms": [mean([o[l] for o in offs]) for l in range(L)]}

    out = {}
    for mode in ("dwdp", "dep"):
        res = {}
        for name, pert in (("A1", False), ("B", True), ("A2", False)):
            res[name] = scenario(mode, pert)
        a1, b, a2 = res["A1"]["step_ms"], res["B"]["step_ms"], res["A2"]["step_ms"]
        base = (a1 + a2) / 2
        res["rank0_step_change_pct"] = (b / base - 1) * 100
        res["noise_pct"] = abs(a1 - a2) / base * 100
        off_a = [(p + q) / 2 for p, q in zip(res["A1"]["layer_start_offsets_ms"],
                                              res["A2"]["layer_start_offsets_ms"])]
        res["max_layer_offset_shift_ms"] = max(abs(p - q) for p, q in
                                               zip(res["B"]["layer_start_offsets_ms"], off_a))
        out[mode] = res
    allr = [None] * world
    dist.all_gather_object(allr, out)
    if rank == 0:
        line = {"what": "rank-0 timeline with rank N-1's batch x factor (B) vs unperturbed (A1, A2)",
                "n_gpus": world, "layers": a.layers, "tokens": T0, "factor": a.factor,
                "rank0": out, "last_rank": allr[-1],
                "reference": "tests/test_simcore.cpp:276-311, tests/acceptance_main.cpp:258-319"}
        s = json.dumps(line)
        print(s, flush=True)
        if a.out:
            with open(a.out, "w") as fh:
                fh.write(s + "\n")
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
