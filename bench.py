#!/usr/bin/env python
"""DWDP MoE-stack throughput on B200 (BASELINE.json metric: output tokens/s/GPU
at 1/2/4/8 B200 vs DEP; exposed prefetch ms/layer).

A step = one forward pass of the 8-layer DeepSeek-R1-shaped MoE stack
(h 7168, E 256 top-8, f 2048, 1 shared expert, bf16) over one rank's batch.
Batches come from the reference workload generator (sample_batches,
src/workload.cpp:137-173): ISL 8K with seq-len CV 0.2, MNT 32768 tokens/rank.
N = 1: config 2 (all 256 experts local; the 8 layers alias one 22.5 GB
weight set because 8 x 22.5 GB does not fit in 180 GB). N > 1: config 3
(DWDP: 256/N owned experts per layer per GPU, the rest pulled from peers one
layer ahead over NVLink, no collective, no barrier on the layer path).

    python bench.py [--gpus N --steps K --warmup W]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference      # CPU reference arm (oracle port)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output tokens/sec/GPU at 1/2/4/8 B200 vs DEP; exposed prefetch ms/layer"
R1 = dict(h=7168, E=256, k=8, f=2048, fs=2048)
# Zipf skew on the device router: bias_e = -beta*s*ln(e+1) added to the
# sigmoid scores (selection only). beta = 0.05 gives a routed-count CV of 2.05
# at s = 0.8 on the R1 router, matching the reference's Zipf(0.8) counts
# (route_tokens, src/workload.cpp:85-111: CV 1.97); calibration in DESIGN.md.
ZIPF_BETA = 0.05


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
         "source": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    except (OSError, ValueError):
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.t.join(timeout=2)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9
                          for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


REF_BUDGET_S = 150.0  # wall budget of the --impl reference arm's W + K steps


def pick_cpu_tokens(stack, steps: int, budget_s: float = REF_BUDGET_S,
                    candidates=(1024, 512, 256, 128, 64, 32, 16)) -> int:
    """Largest C2 sample (tokens per step through the whole stack) whose
    `steps` steps fit the budget, from one timed 16-token probe step (per-token
    cost only falls with T: weight streaming amortises)."""
    import time as _t
    x = stack.input(16)
    t0 = _t.perf_counter()
    stack.forward(x, 16)
    per_tok = (_t.perf_counter() - t0) / 16
    for T in candidates:
        if per_tok * T * steps <= budget_s:
            return T
    return candidates[-1]


def cpu_baseline(layers: int, tokens: int = 0):
    """Oracle port on this host's cores (bounded samples), rank 0 / N = 1 only:
    SURVEY.md §8(d) C1 layer at T in {1, 7, 64, 1000}, one C2 layer at T in
    {64, 256, 1024}, and `value` = the L-layer C2 stack at the reference arm's
    sample size."""
    from oracle import cpu_moe
    sw = cpu_moe.sweep(c2_tokens=())
    stack = cpu_moe.CpuStack(cpu_moe.r1_config(), layers)
    for T in (64, 256, 1024):
        sw["c2_layer_tokens_per_s"][str(T)] = stack.tokens_per_s(T, layers=1, min_s=0.0)
    T = tokens or pick_cpu_tokens(stack, 25)
    tps = stack.tokens_per_s(T, min_s=0.0)
    return {"value": tps, "unit": "tokens/s", "cores": sw["cores"], "kind": "port",
            "sample": f"{T} tokens/step through the {layers}-layer R1 MoE stack (fp32 math, bf16 "
                      f"resident weights); C1/C2 per-layer sweeps beside it",
            "tokens_per_step": T, "c1_layer_tokens_per_s": sw["c1_layer_tokens_per_s"],
            "c2_layer_tokens_per_s": sw["c2_layer_tokens_per_s"]}


def reference_arm(args):
    """--impl reference: the CPU path of the hot path (oracle/ C restatement of the
    MoE layer; the reference itself has no numerical MoE) on all host cores, on
    the largest C2 sample whose W + K steps fit REF_BUDGET_S."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_moe, oracle as O
    stack = cpu_moe.CpuStack(cpu_moe.r1_config(), args.layers)
    tokens = args.ref_tokens or pick_cpu_tokens(stack, args.warmup + args.steps)
    x = stack.input(tokens)
    for _ in range(max(args.warmup, 1)):
        stack.forward(x, tokens)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        stack.forward(x, tokens)
    dt = (time.perf_counter() - t0) / args.steps
    value = tokens / dt
    sim = None
    r = O.ref()
    if r is not None:  # the reference's own CPU code on this path: its simulator
        t1 = time.perf_counter()
        r.simulate(True, args.layers, 7168, 256, 8, 2048, 2048, 2.0, 1382.3e12, 6552.6e9, 900e9,
                   max(args.gpus, 2), 6, 2, 2, 8192.0, 1.0, 0.2 * 8192, args.tokens,
                   args.tokens // 8192, 7)
        sim = {"simulate_dwdp_wall_s": time.perf_counter() - t1}
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "R1 MoE stack, config 2 shapes (CPU oracle port, bounded sample)",
                       "layers": args.layers, "tokens_per_step": tokens,
                       "sample_rule": f"largest T in 1024..16 whose {args.warmup}+{args.steps} steps "
                                      f"fit {REF_BUDGET_S:.0f} s on this host"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"{tokens} tokens/step x {args.layers} layers"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_simulator": sim}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dwdp", choices=["dwdp", "reference"])
    ap.add_argument("--tokens", type=int, default=65536,
                    help="MNT tokens per rank per step (65536: the DWDP break-even regime, "
                         "SURVEY.md section 7; 32768 also reported in DESIGN.md)")
    ap.add_argument("--cv", type=float, default=0.2, help="sequence-length CV")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--engine", default="auto", choices=["auto", "copy", "pull", "hybrid"],
                    help="auto: copy engine unless it leaves prefetch exposed, then the engine "
                         "(copy, pull or hybrid) with the fastest measured step")
    ap.add_argument("--slice-size", type=int, default=64 << 20)
    ap.add_argument("--no-tdm", action="store_true")
    ap.add_argument("--merged", action="store_true", help="merge_elim off (D2D merge baseline)")
    ap.add_argument("--pull-ctas", type=int, default=148)
    ap.add_argument("--ce-inflight", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dep", action="store_true", help="skip the same-box DEP baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=0,
                    help="cpu_baseline stack sample (0: the reference arm's budget rule)")
    ap.add_argument("--ref-tokens", type=int, default=0,
                    help="--impl reference tokens per step (0: largest that fits the budget)")
    ap.add_argument("--profile", action="store_true", help="1 layer, for ncu captures")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp8", "nvfp4"],
                    help="expert weights: bf16, or e4m3 W8A8 with per-row scales (config 5)")
    ap.add_argument("--decode", type=int, default=0,
                    help="decode phase (config 5): B tokens/rank every step instead of prefill batches")
    ap.add_argument("--trace", default="", help="write a chrome trace of the timed DWDP steps here")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="code-path test: WORLD_SIZE > GPUs (ranks share GPUs, gloo, no DEP); "
                         "numbers from such a run are not bench values")
    ap.add_argument("--extra-redundancy", type=int, default=0,
                    help="experts each rank owns beyond E/N (build_placement extra; fewer bytes to pull, "
                         "more HBM per rank; SURVEY.md section 8(f) row 3)")
    ap.add_argument("--attention", action="store_true",
                    help="run a DeepSeek-V3 MLA prefill block (library ops) before every MoE layer, "
                         "in DWDP and DEP alike: the paper's prefetch window MoE(l) + Attention(l+1)")
    ap.add_argument("--no-check", dest="check", action="store_false",
                    help="skip the parity check that runs after timing at N=1: layer 0 on the first "
                         "timed batch against the CPU oracle -- routing of all T tokens bit-exact, 512 "
                         "sampled rows within 1e-2 (oracle/check.py; the checker, outside every timed "
                         "region)")
    ap.add_argument("--zipf", type=float, default=0.0,
                    help="expert-routing skew s: router bias -ZIPF_BETA*s*ln(e+1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2604_01621_b200 as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    if args.oversubscribe:  # code-path test only: several ranks per GPU, gloo plumbing, no DEP
        local = local % torch.cuda.device_count()
        args.no_dep = True
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.oversubscribe:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def allmax(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cpu" if args.oversubscribe else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            if args.oversubscribe:
                torch.cuda.synchronize()
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    layers = 1 if args.profile else args.layers
    model = D.r1_model(layers)
    iters = args.warmup + args.steps
    if args.decode:  # one output token per request, B requests per rank
        toks = [[args.decode] * world for _ in range(iters)]
    else:
        spec = D.WorkloadSpec(D.IslDist.from_cv(8192, args.cv), args.tokens,
                              max(1, args.tokens // 8192), 0.0, 7)
        batches = D.sample_batches(spec, model, world, iters, with_routing=False)
        toks = [[b.tokens[r] for r in range(world)] for b in batches]
        reqs = [[b.requests[r] for r in range(world)] for b in batches]
    if args.attention:
        assert not args.decode, "--attention models the prefill window"
        args.no_e2e = True  # the e2e leg drives dwdp_stack_forward (MoE layers only)
    fp8 = args.dtype == "fp8"
    fp4 = args.dtype == "nvfp4"
    # bytes per weight element (nvfp4: e2m1 + one e4m3 scale per 16) and the
    # dense tensor rate relative to bf16 (no measured fp8 / fp4 figure: the
    # nominal 2x / 4x of the measured sustained bf16 peak)
    wb = 2.0 if args.dtype == "bf16" else 1.0 if fp8 else 0.5 + 1.0 / 16
    rate = {"bf16": 1, "fp8": 2, "nvfp4": 4}[args.dtype]
    rate_src = "nominal"
    lt = os.path.join(ROOT, "profiles", "r1_lt_peaks.json")  # cuBLASLt fp8 / nvfp4 vs bf16 on B200
    if args.dtype != "bf16" and os.path.exists(lt):
        with open(lt) as fh:
            rate = json.load(fh)[{"fp8": "fp8_over_bf16", "nvfp4": "nvfp4_over_bf16"}[args.dtype]]
        rate_src = "measured cuBLASLt"

    cfg = D.DwdpConfig(num_layers=layers, rank=rank, group_size=world, device=local,
                       extra_redundancy=args.extra_redundancy if world > 1 else 0,
                       engine={"pull": D.ENGINE_PULL, "hybrid": D.ENGINE_HYBRID}.get(args.engine,
                                                                                      D.ENGINE_COPY),
                       tdm=0 if args.no_tdm else 1, slice_size=args.slice_size,
                       merge_elim=0 if args.merged else 1, pull_ctas=args.pull_ctas,
                       ce_inflight=args.ce_inflight,
                       weight_layers=layers if world > 1 else 1, kernel_timing=1,
                       max_tokens=args.decode or args.tokens,
                       weight_dtype=D.WEIGHT_NVFP4 if fp4 else D.WEIGHT_FP8 if fp8 else D.WEIGHT_BF16)
    ctx = D.DwdpContext(cfg)
    ctx.init_weights()
    if args.zipf > 0:
        import numpy as np
        ctx.set_bias((-ZIPF_BETA * args.zipf * np.log(np.arange(R1["E"]) + 1.0)).astype(np.float32))
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, ctx.export_ipc())
        ctx.open_peers(b"".join(blobs))
        if not args.no_dep:
            ids = [D.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            ctx.dep_init(ids[0])
    torch.cuda.synchronize()
    barrier()

    T_max = max(max(t) for t in toks)
    x = torch.empty((T_max, R1["h"]), dtype=torch.bfloat16, device=dev)
    D.fill_bf16(x, 0xC0FFEE + rank, 1.0)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    attn = None
    if args.attention:
        from paper_2604_01621_b200.attention import MlaAttention, split_sequences
        attn = MlaAttention(dev, seed=7 + rank)
    gl = [0]  # next global layer of the DWDP stack (attention mode drives the layers itself)
    attn_ms = [0.0, 0]  # attention time inside timed DWDP steps, layers
    attn_flops = [0.0]

    def step(T: int, it: int, dep: bool = False, timed: bool = False):
        """One step of the L-layer stack on rank tokens x[:T] -> y[:T]."""
        if attn is None:
            (ctx.dep_stack_forward if dep else ctx.stack_forward)(x[:T], y[:T])
            return
        seqs = split_sequences(T, reqs[it][rank])
        hcur = x[:T]
        for l in range(layers):
            if timed:
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
            hin = hcur + attn.forward(hcur, seqs)
            if timed:
                a1.record(stream)
                attn_ev.append((a0, a1))
                attn_flops[0] += attn.flops(seqs)
            if dep:
                ctx.dep_layer_forward(l, hin, y[:T], residual=True)
            else:
                ctx.layer_forward(gl[0] + l, hin, y[:T], residual=True)
            hcur = y[:T]
        if not dep:
            gl[0] += layers
    attn_ev = []
    # routed-count statistics of rank 0's first batch (skew and touched experts)
    _, _, cnt, _, _ = ctx.route(0, x[:toks[0][rank]])
    cnt = cnt.double().cpu()
    routing = {"count_cv": float(cnt.std(unbiased=False) / cnt.mean()),
               "touched_experts": int((cnt > 0).sum()), "zipf_s": args.zipf,
               "bias": f"-{ZIPF_BETA}*s*ln(e+1)" if args.zipf > 0 else "0"}

    for it in range(args.warmup):
        step(toks[it][rank], it)
    torch.cuda.synchronize()
    wrecs = ctx.records()
    engine = {D.ENGINE_COPY: "copy", D.ENGINE_PULL: "pull", D.ENGINE_HYBRID: "hybrid"}[cfg.engine]
    if world > 1 and args.engine == "auto":
        # keep the copy engine (no SM cost) while it hides the pull under the
        # compute window, else probe the engines (below)
        steady = [r for r in wrecs if r["prefetch_bytes"] > 0][len(wrecs) // 2:]
        wait = sum(r["gate_wait_ns"] for r in steady)
        moe = sum(r["moe_ns"] for r in steady)
        # one decision for all ranks (the probe below times steps across ranks)
        if allmax(wait / moe if steady and moe > 0 else 0.0) > 0.02:
            # the copy engine leaves prefetch exposed: time one step on each
            # engine (copy; TMA pull kernel; hybrid = pull kernel + copy
            # engines on alternating slices) and keep the fastest step (max
            # over ranks). The SM engines move bytes faster but take SM time
            # from the GEMMs, so in-step GB/s alone is not the criterion.
            best = None
            probe = {}
            for name, eid in (("copy", D.ENGINE_COPY), ("pull", D.ENGINE_PULL), ("hybrid", D.ENGINE_HYBRID)):
                ctx.set_engine(eid)
                t_eng = float("inf")
                for it in range(2):  # best of two steps: one step alone is noisy under the power cap
                    barrier()
                    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    p0.record(stream)
                    step(toks[it][rank], it)
                    p1.record(stream)
                    torch.cuda.synchronize()
                    t_eng = min(t_eng, allmax(p0.elapsed_time(p1)) / max(1, max(toks[it])))
                ctx.records()
                probe[name] = t_eng * 1e3  # us per token of the step's largest rank
                if best is None or t_eng < best[0]:
                    best = (t_eng, name, eid)
            ctx.set_engine(best[2])
            engine = best[1]
    engines = [None] * world
    if world > 1:
        dist.all_gather_object(engines, engine)
    engine_probe = locals().get("probe")
    n0 = ctx.launch_count()

    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for it in range(args.warmup, iters):
            step(toks[it][rank], it, timed=True)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count() - n0
    ms_local = ev0.elapsed_time(ev1)
    attention = None
    if attn is not None:
        a_ms = sum(a0.elapsed_time(a1) for a0, a1 in attn_ev)
        attention = {"block": "DeepSeek-V3 MLA prefill (q_lora 1536, kv_lora 512, 128 heads, qk 128+64, v 128) "
                              + ("on sm_100a kernels (dwdp_mla_forward: tcgen05 projections, tcgen05 causal "
                                 "flash attention)" if attn.backend == "native" else
                                 "from library ops (cuBLAS GEMMs + FlashAttention-2)")
                              + ", causal, rank tokens split into RankBatch::requests sequences",
                     "ms_per_layer": a_ms / max(len(attn_ev), 1),
                     "tflops": attn_flops[0] / (a_ms * 1e-3) / 1e12 if a_ms else None}
    ms = allmax(ms_local)
    recs = ctx.records()
    total_tokens = sum(sum(toks[it]) for it in range(args.warmup, iters))
    value = total_tokens / (ms / 1e3)

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    from paper_2604_01621_b200 import report as RP
    all_recs = gather(recs)
    # per-rank view of the timed DWDP steps (ranks never wait for each other,
    # so the step time is the slowest rank's): its own timed-region length,
    # tokens and per-layer split
    a_local = (sum(a0.elapsed_time(a1) for a0, a1 in attn_ev) / max(len(attn_ev), 1)) if attn is not None else None
    mine = {"rank": rank, "ms_per_step": ms_local / args.steps,
            "tokens_per_step": sum(toks[it][rank] for it in range(args.warmup, iters)) / args.steps,
            "attention_ms_per_layer": a_local}
    for key in ("moe_ns", "gate_wait_ns", "prefetch_ns"):
        mine[key.replace("_ns", "_ms_per_layer")] = sum(r[key] for r in recs) / 1e6 / max(len(recs), 1)
    pf_b, pf_t = sum(r["prefetch_bytes"] for r in recs), sum(r["prefetch_ns"] for r in recs)
    mine["prefetch_gbs"] = pf_b / pf_t if pf_t else None
    per_rank = gather(mine)

    # ---- per-kernel split and roofline of the dominant kernel (grouped GEMM1)
    k, h, f = R1["k"], R1["h"], R1["f"]
    g1_ns = sum(r["gemm1_ns"] for r in recs)
    g1_flops = sum(2.0 * (r["tokens"] * k + r["tokens"]) * 2 * f * h for r in recs)
    g2_ns = sum(r["gemm2_ns"] for r in recs)
    g2_flops = sum(2.0 * (r["tokens"] * k + r["tokens"]) * f * h for r in recs)
    pk = peaks()
    achieved = g1_flops / (g1_ns * 1e-9) / 1e12 if g1_ns else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "gemm1_dram.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    esz = wb
    if args.decode:
        # decode: GEMM1 streams the gate/up rows of every touched expert once
        # (+ the shared expert); token rows are noise next to 2*f*h*esz bytes
        g1_bytes = (routing["touched_experts"] + 1) * 2 * f * h * esz
        gbs = g1_bytes * len(recs) / (g1_ns * 1e-9) / 1e9 if g1_ns else 0.0
        roof = {"bound": "hbm", "kernel": "grouped GEMM1 (gate/up + SwiGLU, tcgen05), weight streaming",
                "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
                "peak_source": pk["source"] + ", HBM copy",
                "bytes_per_launch": g1_bytes, "tflops": achieved, "traffic": None}
    else:
        tpk = pk["bf16_tflops_sustained"] * rate
        roof = {"bound": "tensor", "kernel": "grouped GEMM1 (gate/up + SwiGLU, tcgen05)",
                "achieved": achieved, "peak": tpk, "unit": "TFLOP/s", "frac": achieved / tpk,
                "peak_source": pk["source"] + (f", sustained bf16 x {rate} ({rate_src} {args.dtype}/bf16 "
                                               f"dense-GEMM ratio, profiles/r1_lt_peaks.json)" if rate != 1
                                               else ", sustained bf16"),
                "flops_per_launch": g1_flops / max(len(recs), 1),
                "gemm2_tflops": g2_flops / (g2_ns * 1e-9) / 1e12 if g2_ns else None,
                "traffic": traffic if args.dtype == "bf16" else None,
                "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum of GEMM1 from one committed "
                                   "ncu --set full capture (profiles/gemm1_dram.json), not measured in this run"
                                   if args.dtype == "bf16" and traffic else None)}
    split = {key: sum(r[key] for r in recs) / 1e6 / max(len(recs), 1)
             for key in ("router_ns", "permute_ns", "gemm1_ns", "gemm2_ns", "combine_ns",
                         "moe_ns", "gate_wait_ns", "prefetch_ns", "merge_ns")}
    exposed_ms = split["gate_wait_ns"]
    pf_bytes = sum(r["prefetch_bytes"] for r in recs)
    pf_ns = sum(r["prefetch_ns"] for r in recs)

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # Serving-style pipeline through the public API: step i+1's input goes
        # host->device and step i's result device->host on a copy stream while
        # step i computes (double-buffered device x/y, pinned host buffers).
        # Every step's copies are inside the timed region.
        hx = torch.empty((T_max, h), dtype=torch.bfloat16, pin_memory=True)
        hy = [torch.empty((T_max, h), dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
        hx.copy_(x.cpu())
        xb, yb = [x, torch.empty_like(x)], [y, torch.empty_like(y)]
        cs = torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        steps = list(range(args.warmup, iters))
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d = d2h = 0
        e0.record(stream)
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            T = toks[steps[0]][rank]
            xb[0][:T].copy_(hx[:T], non_blocking=True)
            ev_in[0].record(cs)
            h2d += T * h * 2
        for i, it in enumerate(steps):
            b, T = i % 2, toks[it][rank]
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[b])  # y buffer b drained to the host
            ctx.stack_forward(xb[b][:T], yb[b][:T])
            ev_done[b].record(stream)
            with torch.cuda.stream(cs):
                if i + 1 < len(steps):
                    Tn = toks[steps[i + 1]][rank]
                    if i >= 1:
                        cs.wait_event(ev_done[1 - b])  # x buffer 1-b no longer read
                    xb[1 - b][:Tn].copy_(hx[:Tn], non_blocking=True)
                    ev_in[1 - b].record(cs)
                    h2d += Tn * h * 2
                cs.wait_event(ev_done[b])
                hy[b][:T].copy_(yb[b][:T], non_blocking=True)
                ev_out[b].record(cs)
                d2h += T * h * 2
        stream.wait_stream(cs)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = allmax(e0.elapsed_time(e1))
        e2e = {"value": total_tokens / (ems / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "api": "dwdp_stack_forward (C-ABI) with pinned host input/output; H2D of step i+1 "
                      "and D2H of step i on a copy stream overlap step i's compute"}
        ctx.records()

    # ---- DEP baseline on the same box: same kernels + NCCL all-to-alls
    dep = None
    if world > 1 and not args.no_dep:
        for it in range(args.warmup):
            step(toks[it][rank], it, dep=True)
        torch.cuda.synchronize()
        ctx.records()
        barrier()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for it in range(args.warmup, iters):
            step(toks[it][rank], it, dep=True)
        d1.record(stream)
        torch.cuda.synchronize()
        barrier()
        dms = allmax(d0.elapsed_time(d1))
        drecs = ctx.records()
        all_drecs = gather(drecs)
        dval = total_tokens / (dms / 1e3)
        what = {1: "token-deduplicated dispatch (each token row once to every peer rank) + receive-side permute "
                   "merging sources + per-rank partial combine; token counts exchanged once per step",
                2: "owner-only dispatch (each token row once to each rank owning one of its experts; per-layer "
                   "row counts exchanged) + receive-side permute + per-rank partial combine"}

        def dep_mode_run(mode):
            # the stronger DEPs (dwdp_dep_set_mode), same kernels, same box
            ctx.dep_set_mode(mode)
            for it in range(args.warmup):
                step(toks[it][rank], it, dep=True)
            torch.cuda.synchronize()
            ctx.records()
            barrier()
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(stream)
            for it in range(args.warmup, iters):
                step(toks[it][rank], it, dep=True)
            q1.record(stream)
            torch.cuda.synchronize()
            barrier()
            qms = allmax(q0.elapsed_time(q1))
            qrecs = ctx.records()
            ctx.dep_set_mode(0)
            qval = total_tokens / (qms / 1e3)
            return {"value": qval, "tokens_per_s_per_gpu": qval / world, "ms_per_step": qms / args.steps,
                    "comm_ms_per_layer": sum(r["comm_ns"] for r in qrecs) / 1e6 / max(len(qrecs), 1),
                    "kernel_ms_per_layer": {key.replace("_ns", ""): sum(r[key] for r in qrecs) / 1e6
                                            / max(len(qrecs), 1)
                                            for key in ("router_ns", "permute_ns", "gemm1_ns",
                                                        "gemm2_ns", "combine_ns")},
                    "dwdp_over_dep": value / qval, "what": what[mode]}

        def guarded(mode):
            # a stronger-DEP arm that fails (e.g. out of memory at a large N:
            # every rank allocates the same sizes, so all ranks raise together)
            # is reported instead of losing the DWDP line
            try:
                return dep_mode_run(mode)
            except Exception as exc:  # noqa: BLE001
                ctx.dep_set_mode(0)
                torch.cuda.synchronize()
                return {"value": 0.0, "error": f"{type(exc).__name__}: {exc}"[:300]}

        dep2 = guarded(1)
        dep3 = guarded(2)
        dep = {"value": dval, "unit": "tokens/s", "tokens_per_s_per_gpu": dval / world,
               "ms_per_step": dms / args.steps,
               "comm_ms_per_layer": sum(r["comm_ns"] for r in drecs) / 1e6 / max(len(drecs), 1),
               "kernel_ms_per_layer": {key.replace("_ns", ""): sum(r[key] for r in drecs) / 1e6
                                       / max(len(drecs), 1)
                                       for key in ("router_ns", "permute_ns", "gemm1_ns",
                                                   "gemm2_ns", "combine_ns")},
               "dwdp_over_dep": value / dval,
               "what": "reference DEP semantics: every (token, expert) row to the expert's rank "
                       "(simcore.cpp:321-324), per-expert counts exchanged each layer",
               "dedupe": dep2, "dedupe_owners": dep3,
               "dwdp_over_best_dep": value / max(dval, dep2.get("value") or 0.0, dep3.get("value") or 0.0)}

    # ---- whole-step roofline (north star / SURVEY.md §8(d)): per layer the
    # slower of the layer's flops at the tensor peak and the remote-expert
    # bytes over NVLink (900 GB/s per direction), summed over the timed steps
    # with each step's heaviest rank
    f_tok = 2.0 * h * (3 * k * f + 3 * R1["fs"] + R1["E"])
    p_peak = pk["bf16_tflops_sustained"] * 1e12 * rate
    c_loc = min(R1["E"], -(-R1["E"] // world) + args.extra_redundancy) if world > 1 else R1["E"]
    b_rem = (R1["E"] - c_loc) * 3.0 * h * f * wb if world > 1 else 0.0
    t_tensor = sum(layers * max(toks[it]) * f_tok / p_peak for it in range(args.warmup, iters))
    t_link = args.steps * layers * b_rem / 900e9
    t_roof = sum(layers * max(max(toks[it]) * f_tok / p_peak, b_rem / 900e9)
                 for it in range(args.warmup, iters))
    step_roof = {"t_roof_ms_per_step": t_roof * 1e3 / args.steps,
                 "t_measured_ms_per_step": ms / args.steps, "frac": t_roof / (ms * 1e-3),
                 "bound": "tensor" if t_tensor >= t_link else "nvlink",
                 "t_tensor_ms_per_step": t_tensor * 1e3 / args.steps,
                 "t_nvlink_ms_per_step": t_link * 1e3 / args.steps,
                 "flops_per_token_layer": f_tok, "remote_bytes_per_layer": b_rem,
                 "peak_tflops": p_peak / 1e12, "link_gbs": 900.0}

    # ---- RunReport accounting (simcore.hpp:29-61, 177-213) over the measured
    # events of every rank, and the analytic model beside it (a15, a16)
    acct = None
    if rank == 0:
        tab, evs = RP.report_from_records(all_recs, layers, 0, with_events=True)
        acct = {"dwdp": tab.as_dict(), "breakdown_csv": tab.to_csv()}
        if args.trace:
            with open(args.trace, "w") as fh:
                json.dump(RP.chrome_trace(evs), fh)
            acct["trace"] = args.trace
        if dep is not None:
            dtab = RP.report_from_records(all_drecs, layers, 0)
            cmp_ = RP.compare_reports(dtab, tab)  # a = DEP baseline, b = DWDP
            acct.update(dep=dtab.as_dict(), comparison_dep_vs_dwdp=cmp_.as_dict(),
                        comparison_csv=cmp_.to_csv())
        if world > 1:
            mean_t = total_tokens / (args.steps * world)
            acct["analytic_compare"] = D.analytic_compare(
                D.r1_model(layers, wb),
                D.GpuSpec(pk["bf16_tflops_sustained"] * 1e12 * rate, pk["hbm_gbs"] * 1e9,
                          900e9),
                D.build_placement(R1["E"], world, args.extra_redundancy), int(mean_t))
            acct["analytic_compare"]["tokens_per_rank"] = mean_t
            # the same model calibrated with this run's
            # measured rates (grouped-GEMM TFLOP/s, in-step prefetch GB/s) beside
            # the measured DWDP/DEP ratio
            gemm_tf = (g1_flops + g2_flops) / ((g1_ns + g2_ns) * 1e-9) if (g1_ns + g2_ns) else p_peak
            link = pf_bytes / pf_ns * 1e9 if pf_ns else 900e9
            cal = D.analytic_compare(D.r1_model(layers, wb),
                                     D.GpuSpec(gemm_tf, pk["hbm_gbs"] * 1e9, link),
                                     D.build_placement(R1["E"], world, args.extra_redundancy), int(mean_t))
            cal.update(gemm_tflops_measured=gemm_tf / 1e12, prefetch_gbs_measured=link / 1e9,
                       measured_dwdp_over_dep=(dep or {}).get("dwdp_over_dep"))
            acct["analytic_compare_calibrated"] = cal

    check = None
    if args.check and world == 1 and not args.decode and not args.profile and args.dtype == "bf16":
        from oracle import check as CK
        T0 = toks[args.warmup][rank]
        bias = None
        if args.zipf > 0:
            import numpy as np
            bias = (-ZIPF_BETA * args.zipf * np.log(np.arange(R1["E"]) + 1.0)).astype(np.float32)
        check = CK.check_layer(ctx, x[:T0], layer=0, sample_rows=512, seed=T0, bias=bias)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(layers, args.cpu_tokens)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("e4m3 (W8A8, fp32 accumulate)" if fp8 else
                      "nvfp4 (W4A4 e2m1, e4m3 per-16 scales, fp32 accumulate)" if fp4 else "bf16"),
            "data": "synthetic (counter-hash random-init weights and activations)",
            "config": {"workload": (f"R1 MoE stack, config 5 (decode B={args.decode}, "
                                    f"{args.dtype}, zipf {args.zipf}, "
                                    f"{'merged' if args.merged else 'split'} fetch)" if args.decode
                                    else "R1 MoE stack, config 2 (all experts local)" if world == 1
                                    else "R1 MoE stack, config 3 (DWDP)"),
                       "layers": layers, "hidden": h, "experts": 256, "top_k": k, "ffn": f,
                       "shared_experts": 1, "mnt_tokens_per_rank": args.tokens,
                       "isl": 8192, "seq_len_cv": args.cv,
                       "tokens_per_step_rank0": [toks[it][0] for it in range(args.warmup, iters)],
                       "weights": ("one 22.5 GB set aliased by all layers (N=1)" if world == 1
                                   else f"{min(256, -(-256 // world) + args.extra_redundancy)} owned experts/layer/GPU, {layers} layers"),
                       "prefetch_engine": (engines if world > 1 else None),
                       "engine_probe_us_per_token": engine_probe,
                       "slice_size": args.slice_size if world > 1 else None,
                       "l2": "inputs larger than L2: {} GB of expert weights per layer".format(
                           "11.3 (e4m3)" if fp8 else "6.3 (nvfp4)" if fp4 else "22.5 (bf16)"),
                       "attention_block": bool(args.attention),
                       "extra_redundancy": args.extra_redundancy,
                       "parallelism": f"dwdp{world}"},
            "tokens_per_s_per_gpu": value / world,
            "exposed_prefetch_ms_per_layer": exposed_ms,
            "per_rank": per_rank if world > 1 else None,
            # DWDP ranks never wait for each other: in serving each rank takes
            # its next batch when it finishes, so the sustained rate is the sum
            # of the ranks' own rates (not the headline value, which follows the
            # bench contract: all tokens over the slowest rank's time)
            "value_independent_ranks": (sum(r["tokens_per_step"] / (r["ms_per_step"] / 1e3) for r in per_rank)
                                        if world > 1 else None),
            # the reference's own definitions (src/simcore.cpp:35-47, SURVEY.md
            # §8(d)): tokens/s/GPU = (1/N) sum over ranks of each rank's tokens
            # over its own steady-state time; exposed = weight-wait averaged
            # over ranks
            "reference_definition": ({"tokens_per_s_per_gpu": sum(r["tokens_per_step"] / (r["ms_per_step"] / 1e3)
                                                                  for r in per_rank) / world,
                                      "exposed_prefetch_ms_per_layer": sum(r["gate_wait_ms_per_layer"]
                                                                           for r in per_rank) / world}
                                     if world > 1 else None),
            "merge_ms_per_layer": split["merge_ns"] if args.merged else None,
            "prefetch": ({"bytes_per_layer": pf_bytes / max(len(recs), 1),
                          "gbs": pf_bytes / pf_ns if pf_ns else None,
                          "ms_per_layer": split["prefetch_ns"]} if world > 1 else None),
            "kernel_ms_per_layer": {k2.replace("_ns", ""): v for k2, v in split.items()},
            "roofline": roof, "step_roofline": step_roof, "routing": routing,
            "dep_baseline": dep, "report": acct,
            "hbm_gb": {k2: round(v / 1e9, 2) for k2, v in ctx.memory().items()},
            "attention": attention,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "check": check,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    barrier()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
