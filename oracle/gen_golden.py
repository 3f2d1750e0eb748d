"""ORACLE / TEST INFRASTRUCTURE ONLY — regenerates tests/golden/*.json.

Run here (needs /root/reference built into oracle/_ref and transformers):
    python oracle/gen_golden.py

* ref_*.json  — outputs of the reference library itself (oracle/_ref,
  compiled from /root/reference/proj/src) on the reference's own KAT inputs
  (tests/test_placement.cpp, tests/test_copyplan.cpp, tests/test_workload.cpp,
  tests/test_modelspec.cpp) plus seeded random cases and the BASELINE configs'
  workload batches.
* hf_moe.json — transformers 5.5 DeepseekV3MoE (sigmoid, noaux_tc group-limited
  routing, shared expert) and Qwen2MoeTopKRouter (softmax top-k) run in fp32 on
  bf16-representable inputs: the public implementations of the MoE semantics
  that /root/reference does not contain.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def dump(name, obj):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name, os.path.getsize(os.path.join(OUT, name)), "bytes")


def gen_ref():
    r = O.ref()
    assert r is not None, "reference library not built (oracle/_ref)"
    # --- placement: reference KATs (test_placement.cpp:14-121) + random grid
    cases = [(256, 4, 0), (256, 3, 0), (4, 2, 1), (6, 3, 1), (97, 5, 2), (256, 4, 256),
             (256, 8, 0), (256, 2, 0), (16, 4, 0), (16, 4, 1), (256, 5, 0), (256, 6, 0),
             (256, 7, 0), (256, 3, 1), (61, 4, 0), (8, 1, 0), (3, 4, 0), (8, 2, -1)]
    g = np.random.default_rng(20240811)
    for _ in range(40):
        n = int(g.integers(2, 16))
        cases.append((int(n + g.integers(0, 120)), n, int(g.integers(0, 8))))
    for extra in range(0, 70, 7):
        cases.append((61, 4, extra))
    pl = []
    for E, N, x in cases:
        st, c, red, local, fetch = r.build_placement(E, N, x)
        pl.append({"E": E, "N": N, "extra": x, "status": st, "local_count": c,
                   "redundancy": red, "local_sets": local,
                   "fetch": [[list(p) for p in f] for f in fetch] if fetch else None})
    dump("ref_placement.json", pl)

    # --- copy plan: test_copyplan.cpp KATs + random shard lists
    cp_cases = [([(1, 0, 5, 0), (2, 0, 5, 0)], 2, 0), ([(1, 7, 5, 100)], 2, 0),
                ([(1, 0, 2, 0), (2, 0, 2, 0), (3, 0, 2, 0)], 4, 0),
                ([(1, 0, 300, 0), (2, 0, 200, 0), (1, 1, 250, 0)], 300, 0),
                ([(1, 0, 4, 0), (2, 0, 4, 0), (3, 0, 4, 0)], 2, 9),
                ([(1, 0, 4, 0), (2, 0, 4, 0), (3, 0, 4, 0)], 2, 10),
                ([(1, 0, 4, 0), (2, 0, 4, 0), (3, 0, 4, 0)], 2, 11),
                ([(1, 0, 10, 0), (2, 0, 10, 0), (3, 0, 6, 0)], 2, 0),
                ([(1, 3, 5, 10)], 2, 0),
                ([(1, 0, 5, 0)], 0, 0), ([(1, 0, 0, 0)], 2, 0), ([(0, 0, 5, 0)], 2, 0),
                ([(1, 0, 5, 0), (1, 0, 7, 0)], 2, 0), ([], 4, 0)]
    # DWDP per-rank shard lists for C1 (E16 N4, 1 MiB tensors) and C3-like R1 N=8 at 1 MiB
    for N, E, per_tensor in [(4, 16, 1 << 20), (8, 256, 7168 * 2048 * 2)]:
        _, c, _, _, fetch = r.build_placement(E, N, 0)
        for dst in range(N):
            per_peer = {}
            for e, s in fetch[dst]:
                per_peer[s] = per_peer.get(s, 0) + 1
            sh = [(p, t, per_tensor * cnt, 0) for t in range(3) for p, cnt in sorted(per_peer.items())]
            cp_cases.append((sh, 1 << 20, dst))
    for _ in range(80):
        peers = int(g.integers(1, 6))
        params = int(g.integers(1, 4))
        sh = []
        for p in range(params):
            for peer in range(peers):
                if g.random() < 0.2 and peers > 1:
                    continue
                sh.append((peer, p, int(g.integers(1, 5000)), int(g.integers(0, 1000))))
        if sh:
            cp_cases.append((sh, int(g.integers(1, 700)), 90))
    cp = []
    for sh, s, dst in cp_cases:
        st, slices = r.build_copy_plan(sh, s, dst)
        big = slices is not None and len(slices) > 2000
        ent = {"shards": [list(x) for x in sh], "slice": s, "dst": dst, "status": st}
        if big:  # keep fixtures small: count + a checksum over the ordered plan
            arr = np.array(slices, np.int64)
            ent["n_slices"] = len(slices)
            ent["head"] = [list(x) for x in slices[:64]]
            ent["checksum"] = int((arr * (np.arange(len(arr))[:, None] + 1) % 1000003).sum())
        else:
            ent["slices"] = [list(x) for x in slices] if slices is not None else None
        cp.append(ent)
    dump("ref_copyplan.json", cp)

    # --- workload + RNG
    wl = {"u64": {str(s): [str(v) for v in r.rng_u64(s, 64)] for s in (0, 1, 5, 12345)},
          "mix": [[str(a), str(b), str(r.mix(a, b))] for a, b in
                  [(0, 0), (1, 2), (7, 0x10000), (2**63, 5), (123456789, 987654321)]],
          "normal": {str(s): r.rng_normal(s, 32, 3.0, 2.0).tolist() for s in (1, 17)},
          "route": [], "batches": []}
    for tokens, E, k, skew, seed in [(100, 16, 2, 0.0, 1), (100, 16, 2, 1.2, 1), (1000, 256, 8, 0.0, 5),
                                     (2000, 256, 8, 10.0, 5), (509, 256, 8, 1.2, 42),
                                     (4096, 256, 8, 0.8, 3), (0, 256, 8, 0.0, 5), (64, 256, 8, 1.2, 9)]:
        st, cnt = r.route_tokens(tokens, E, k, skew, seed)
        wl["route"].append({"tokens": tokens, "E": E, "k": k, "skew": skew, "seed": seed,
                            "counts": cnt.tolist()})
    # BASELINE config 4: ISL 8K CV sweep (acceptance_main.cpp:233-239 shape), MNT 32K/64K
    specs = []
    for cv in (0.0, 0.1, 0.2, 0.3):
        for mnt in (32768, 65536):
            kind = 0 if cv == 0 else 2
            specs.append((kind, 8192.0, 1.0, cv * 8192.0, mnt, mnt // 8192, 0.0, 7))
    specs += [(1, 8192.0, 0.8, 0.0, 32768, 4, 0.0, 7), (1, 1000.0, 0.5, 0.0, 4000, 3, 1.0, 7),
              (2, 4096.0, 1.0, 512.0, 8192, 2, 0.0, 99), (0, 600.0, 1.0, 0.0, 1000, 2, 0.0, 1)]
    for spec in specs:
        for N in (2, 4, 8):
            st, t, q, routed = r.sample_batches(*spec, 256, 8, N, 6, routed=spec[6] > 0)
            ent = {"spec": list(spec), "N": N, "iters": 6, "tokens": t.tolist(),
                   "requests": q.tolist()}
            if routed is not None:
                ent["routed_rank0_iter0"] = routed[0, 0].tolist()
            wl["batches"].append(ent)
    dump("ref_workload.json", wl)

    # --- cost formulas + analytic predictor + simulator on a toy rig
    R1 = dict(h=7168, E=256, k=8, f=2048, fs=2048)
    costs = {"shard_bytes": [[h, f, wb, r.expert_shard_bytes(h, f, wb)] for h, f, wb in
                             [(8, 4, 1.0), (8, 4, 0.5), (7168, 2048, 0.5), (7168, 2048, 2.0),
                              (7168, 2048, 1.0), (512, 1024, 2.0)]],
             "moe_entries": [], "analytic": []}
    for T in (1, 64, 4096, 32768):
        costs["moe_entries"].append({"T": T, "out": r.moe_entries(R1["h"], R1["f"], R1["fs"], 2.0, 2.0,
                                                                   T, T * 8, 256).tolist()})
    for N in (2, 4, 8):
        for T in (8192, 32768, 65536):
            costs["analytic"].append({"N": N, "T": T, **r.analytic(
                R1["h"], 256, 8, 2048, 2048, 2.0, 1649.8e12, 6552.6e9, 900e9, N, T)})
    dump("ref_costs.json", costs)


def gen_hf():
    import torch
    from transformers import DeepseekV3Config
    from transformers.models.deepseek_v3.modeling_deepseek_v3 import DeepseekV3MoE
    from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeTopKRouter

    torch.manual_seed(0)

    def bf(shape, scale):  # bf16-representable fp32 values
        return (torch.rand(shape) * 2 - 1).mul(scale).to(torch.bfloat16).float()

    def bits(t):  # bf16 bit patterns, compact in JSON
        return O.bf16_round(t.numpy()).astype(int).reshape(-1).tolist()

    out = {"deepseek": [], "softmax": []}
    for case, (h, E, k, f, ng, tg, T) in enumerate([(64, 16, 4, 32, 4, 2, 24), (64, 32, 8, 32, 8, 4, 17),
                                                      (64, 16, 2, 32, 1, 1, 9)]):
        cfg = DeepseekV3Config(hidden_size=h, n_routed_experts=E, num_experts_per_tok=k,
                               moe_intermediate_size=f, n_shared_experts=1, n_group=ng,
                               topk_group=tg, norm_topk_prob=True, routed_scaling_factor=2.5,
                               hidden_act="silu", num_local_experts=E)
        moe = DeepseekV3MoE(cfg).float()
        x = bf((T, h), 1.0)
        wr = bf((E, h), 1 / np.sqrt(h))
        bias = (torch.rand(E) * 0.1 - 0.05)
        gate_up = bf((E, 2 * f, h), 1 / np.sqrt(h))
        down = bf((E, h, f), 1 / np.sqrt(f))
        sg, su, sd = bf((f, h), 1 / np.sqrt(h)), bf((f, h), 1 / np.sqrt(h)), bf((h, f), 1 / np.sqrt(f))
        with torch.no_grad():
            moe.gate.weight.copy_(wr)
            moe.gate.e_score_correction_bias.copy_(bias)
            moe.experts.gate_up_proj.copy_(gate_up)
            moe.experts.down_proj.copy_(down)
            moe.shared_experts.gate_proj.weight.copy_(sg)
            moe.shared_experts.up_proj.weight.copy_(su)
            moe.shared_experts.down_proj.weight.copy_(sd)
            logits = moe.gate(x)
            idx, wts = moe.route_tokens_to_experts(logits)
            y = moe(x.unsqueeze(0)).squeeze(0)
        order = torch.argsort(idx, dim=-1)
        out["deepseek"].append({
            "h": h, "E": E, "k": k, "f": f, "n_group": ng, "topk_group": tg, "T": T,
            "x": bits(x), "w_router": wr.tolist(), "bias": bias.tolist(),
            "gate_up": bits(gate_up), "down": bits(down), "s_gate": bits(sg),
            "s_up": bits(su), "s_down": bits(sd),
            "idx_sorted": torch.gather(idx, 1, order).tolist(),
            "wts_sorted": torch.gather(wts, 1, order).tolist(), "y": y.tolist()})
    for h, E, k, T in [(512, 16, 2, 32), (64, 8, 2, 7)]:
        from types import SimpleNamespace
        cfg = SimpleNamespace(num_experts_per_tok=k, num_experts=E, norm_topk_prob=True, hidden_size=h)
        router = Qwen2MoeTopKRouter(cfg).float()
        x = bf((T, h), 1.0)
        wr = bf((E, h), 1 / np.sqrt(h))
        with torch.no_grad():
            router.weight.copy_(wr)
            _, w, i = router(x)
        order = torch.argsort(i, dim=-1)
        out["softmax"].append({"h": h, "E": E, "k": k, "T": T, "x": bits(x), "w_router": wr.tolist(),
                               "idx_sorted": torch.gather(i, 1, order).tolist(),
                               "wts_sorted": torch.gather(w, 1, order).tolist()})
    dump("hf_moe.json", out)


if __name__ == "__main__":
    O.build()
    gen_ref()
    gen_hf()
