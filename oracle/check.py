"""ORACLE / TEST INFRASTRUCTURE ONLY — the headline-config parity check.

Used by tests/test_gpu_headline.py and by ``bench.py --check`` (outside the
timed region) to compare one MoE layer of the sm_100a path at the bench's own
batch (R1 shapes, T ~ 61K tokens) with the CPU oracle:

* routing for ALL T tokens: top-k indices, fp32 weights (bitwise), per-expert
  counts and the stable expert-major permutation rows, against oracle_route /
  oracle_permute (the DeepSeek-V3 routing restated in oracle/dwdp_oracle.c;
  rows sum to T*k as include/dwdpsim/workload.hpp:50-52 requires);
* the exact (22-bit fixed point, int64-sum) router's top-k against float64
  logits for all T tokens (fp64_agreement);
* layer outputs on a seeded sample of rows (every MoE row depends only on its
  own token, so a row subset through the oracle is exact) within the stated
  normwise relative error of the oracle's fp32 math.

The product path never imports this module.
"""
from __future__ import annotations

import time

import numpy as np

from . import oracle as O


def moe_config(c) -> O.MoeConfig:
    """oracle MoeConfig of a paper_2604_01621_b200.DwdpConfig."""
    return O.MoeConfig(c.hidden, c.num_experts, c.top_k, c.ffn, c.shared_ffn, c.scoring,
                       c.n_group, c.topk_group, c.norm_topk, c.routed_scale)


def _bf16_np(t) -> np.ndarray:
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)


def check_layer(ctx, x, layer: int = 0, sample_rows: int = 512, seed: int = 0,
                bias: np.ndarray | None = None, row_align: int = 128, y=None) -> dict:
    """Compare ctx's layer `layer` on x [T][h] (bf16, cuda) with the oracle.

    ctx must hold every expert locally (all-local config 2). y: the device
    layer output if the caller already has it (else moe_forward is run).
    Returns a dict of the comparison; `ok` is the overall verdict."""
    import torch

    cfg = ctx.cfg
    T, h = x.shape
    o = O.oracle()
    oc = moe_config(cfg)
    t0 = time.perf_counter()
    idx, wts, counts, row_of, rows = ctx.route(layer, x)
    if y is None:
        y = ctx.moe_forward(layer, x)
    torch.cuda.synchronize()
    xb = _bf16_np(x)
    sc = float(np.float32(1.0) / np.sqrt(np.float32(h)))
    wr = o.fill_bf16(o.tensor_seed(cfg.weight_seed, layer, cfg.num_experts + 1, 0),
                     cfg.num_experts * h, sc)
    _, oidx, owts = o.route(oc, xb, T, wr, bias)
    t_route = time.perf_counter() - t0
    total, ocounts, orow = o.permute(oidx, cfg.num_experts, row_align)
    gidx = idx.cpu().numpy()
    res = {
        "tokens": int(T),
        "idx_mismatch_tokens": int((gidx != oidx).any(axis=1).sum()),
        "wts_mismatch_tokens": int((wts.cpu().numpy().view(np.uint32) != owts.view(np.uint32))
                                   .any(axis=1).sum()),
        "counts_equal": bool((counts.cpu().numpy() == ocounts).all()),
        "row_of_equal": bool((row_of.cpu().numpy() == orow).all()),
        "rows_equal": int(rows) == int(total),
        "padded_rows": int(total),
        "touched_experts": int((ocounts > 0).sum()),
        "oracle_route_s": round(t_route, 2),
        # the exact router's selection vs float64 logits (weak point of a
        # quantised-exact router: near-ties between experts); first 16K tokens
        "fp64_routing": fp64_agreement(oc, xb[:min(T, 16384) * h], min(T, 16384), wr,
                                       oidx[:min(T, 16384)], bias),
    }
    # sampled rows: first, last and a seeded draw
    rng = np.random.default_rng(seed)
    n = min(sample_rows, T)
    pick = np.unique(np.concatenate([[0, T - 1], rng.choice(T, size=max(n - 2, 0), replace=False)]))
    t1 = time.perf_counter()
    xs = np.ascontiguousarray(xb.reshape(T, h)[pick]).reshape(-1)
    yo, sidx, _ = o.moe_forward_seeded(oc, cfg.weight_seed, layer, xs, len(pick), bias)
    yg = y.float()[torch.as_tensor(pick, device=y.device)].cpu().numpy()
    diff = yg - yo
    row_err = np.linalg.norm(diff, axis=1) / np.maximum(np.linalg.norm(yo, axis=1), 1e-30)
    res.update({
        "sampled_rows": int(len(pick)),
        "sample_routing_equal": bool((sidx == oidx[pick]).all()),
        "rel_err_normwise": float(np.linalg.norm(diff) / max(np.linalg.norm(yo), 1e-30)),
        "max_row_rel_err": float(row_err.max()),
        "oracle_rows_s": round(time.perf_counter() - t1, 2),
        "tolerance": 1e-2,
    })
    res["ok"] = bool(res["idx_mismatch_tokens"] == 0 and res["wts_mismatch_tokens"] == 0
                     and res["counts_equal"] and res["row_of_equal"] and res["rows_equal"]
                     and res["sample_routing_equal"] and res["rel_err_normwise"] < 1e-2
                     and res["max_row_rel_err"] < 1e-2)
    return res


def fp64_route(cfg, x_bf16: np.ndarray, T: int, w_router_bf16: np.ndarray, bias=None):
    """DeepSeek-V3 / Qwen routing with float64 logits (x . Wr^T of bf16
    values: every product exact, the 7168-term sums to ~1e-16): the
    unquantised selection the exact 22-bit router is compared against.
    Returns idx [T][k] ordered like oracle_route (descending choice score,
    ties to the lower expert)."""
    E, k, h = cfg.num_experts, cfg.top_k, cfg.hidden
    x = O.bf16_to_f32(x_bf16).reshape(T, h).astype(np.float64)
    w = O.bf16_to_f32(w_router_bf16).reshape(E, h).astype(np.float64)
    lg = x @ w.T
    if cfg.scoring == 1:
        sc = 1.0 / (1.0 + np.exp(-lg))
        ch = sc + (0.0 if bias is None else np.asarray(bias, np.float64)[None, :])
    else:
        ch = lg.copy()
    G = max(cfg.n_group, 1)
    if G > 1 and cfg.topk_group < G:
        gs = E // G
        g2 = np.sort(ch.reshape(T, G, gs), axis=-1)[..., -2:].sum(-1) if gs >= 2 else ch.reshape(T, G, gs)[..., 0]
        order = np.argsort(-g2, axis=1, kind="stable")[:, :cfg.topk_group]
        keep = np.zeros((T, G), bool)
        np.put_along_axis(keep, order, True, axis=1)
        ch = np.where(np.repeat(keep, gs, axis=1), ch, 0.0)
    return np.argsort(-ch, axis=1, kind="stable")[:, :k].astype(np.int32)


def fp64_agreement(cfg, x_bf16: np.ndarray, T: int, w_router_bf16: np.ndarray, idx_exact: np.ndarray,
                   bias=None) -> dict:
    """How often the exact 22-bit router's top-k differs from float64 routing."""
    ref = fp64_route(cfg, x_bf16, T, w_router_bf16, bias)
    same_set = (np.sort(ref, 1) == np.sort(idx_exact, 1)).all(1)
    same_order = (ref == idx_exact).all(1)
    return {"tokens": int(T), "topk_set_mismatch_tokens": int((~same_set).sum()),
            "topk_order_mismatch_tokens": int((~same_order).sum()),
            "topk_set_agreement": float(same_set.mean())}
