"""GPU parity tests of the NVFP4 (W4A4) path: kind::mxf4nvf4 block-scaled
grouped GEMM, the NVFP4 quantisers and the nvfp4 DWDP layer.

Bar: quantised codes, e4m3 block scales (in the device atom layout) and fp32
row scales bit-exact vs oracle_nvfp4_quant_row; the GEMM within 1e-2 of an
fp32 product of the dequantised operands; layer outputs within 1e-2 of the
oracle's W4A4 emulation (w8a8 = 2) and within 0.35 of the bf16 oracle
(NVFP4 quantisation error of weights and activations); DWDP with NVFP4 arenas
bit-identical to the all-local NVFP4 model.
"""
import numpy as np
import pytest
import torch

import paper_2604_01621_b200 as D
from oracle import oracle as O
from test_gpu import MID, _bf16_np, _bias, _rel, _scale, dev, make_x, oracle_cfg  # noqa: F401

pytestmark = pytest.mark.gpu

TOL_FP4 = 1e-2    # vs the oracle's W4A4 emulation (fp32 sum order, rare bf16-H flips)
TOL_FP4_Q = 0.35  # NVFP4 quantisation error vs the bf16 oracle (measured 0.254-0.264:
#                   e2m1 x, weights and H, each ~9% per element)

FP4_CONFIGS = {
    "tiny_fp4": D.DwdpConfig.tiny(weight_dtype=D.WEIGHT_NVFP4),
    "mid_fp4": D.DwdpConfig(num_layers=1, num_experts=64, hidden=1024, ffn=256, shared_ffn=256,
                            top_k=6, n_group=8, topk_group=4, max_tokens=2048,
                            weight_dtype=D.WEIGHT_NVFP4),
    "r1_fp4": D.DwdpConfig(num_layers=1, max_tokens=512, weight_dtype=D.WEIGHT_NVFP4),
}
# GEMM1 runs on CTA pairs by default (DWDP_FP4_PAIR); batches with fewer than
# 128 routed rows per expert, and contexts created with DWDP_FP4_PAIR=0, use
# the 1-SM kernel -- test_moe_forward_nvfp4_single_cta covers that path.


@pytest.fixture(scope="module")
def ctxs4(dev):
    out = {}
    for name, cfg in FP4_CONFIGS.items():
        c = D.DwdpContext(cfg)
        c.init_weights()
        if cfg.scoring == 1:
            c.set_bias(_bias(cfg))
        out[name] = c
    yield out
    for c in out.values():
        c.close()


def _rand_bf16(R, K, seed, dev, scale=1.0):
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((R, K), generator=g, device=dev) * scale
    x[0, :16] = 0.0  # an all-zero block
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("R,K", [(1, 256), (300, 512), (129, 7168), (77, 2048), (130, 1024)])
def test_nvfp4_quant_bit_exact(dev, orc, R, K):
    x = _rand_bf16(R, K, R + K, dev)
    codes, sf, s = D.quant_nvfp4(x)
    torch.cuda.synchronize()
    xo = O.bf16_to_f32(_bf16_np(x).reshape(-1)).reshape(R, K)
    oc, osf, os_ = orc.nvfp4_quant_rows(xo)
    assert (codes.cpu().numpy() == oc).all()
    assert (sf.cpu().numpy() == orc.nvfp4_sf_atoms(osf)).all()
    assert (s.cpu().numpy() == os_).all()


@pytest.mark.parametrize("pair", ["0", "1"])  # 1-SM kernel / CTA-pair kernel (cta_group::2)
@pytest.mark.parametrize("M,N,K", [(128, 256, 256), (300, 512, 1024), (1, 256, 7168),
                                   (1000, 2048, 2048)])
def test_gemm_nvfp4_vs_dequantised_fp32(dev, orc, monkeypatch, M, N, K, pair):
    monkeypatch.setenv("DWDP_FP4_PAIR", pair)
    a = _rand_bf16(M, K, M + 3 * K, dev)
    b = _rand_bf16(N, K, N + 5 * K, dev, scale=0.05)
    qa, qb = D.quant_nvfp4(a), D.quant_nvfp4(b)
    d = D.gemm_nvfp4(qa, qb)
    torch.cuda.synchronize()
    ao = O.bf16_to_f32(_bf16_np(a).reshape(-1)).reshape(M, K)
    bo = O.bf16_to_f32(_bf16_np(b).reshape(-1)).reshape(N, K)
    ca, sa_, ra = orc.nvfp4_quant_rows(ao)
    cb, sb_, rb = orc.nvfp4_quant_rows(bo)
    ref = (orc.nvfp4_dequant(ca, sa_).astype(np.float64) @ orc.nvfp4_dequant(cb, sb_).T.astype(np.float64))
    ref = ref * ra[:, None] * rb[None, :]
    assert _rel(d.float().cpu().numpy(), ref) < TOL_FP4


@pytest.mark.parametrize("name", ["tiny_fp4", "mid_fp4"])
def test_nvfp4_weights_bit_exact(dev, ctxs4, orc, name):
    """Resident e2m1 codes, e4m3 block scales (atom layout) and row scales ==
    oracle quantisation of the same counter-hash bf16 rows."""
    cfg = FP4_CONFIGS[name]
    h, f = cfg.hidden, cfg.ffn
    for e in (0, cfg.num_experts - 1) + ((cfg.num_experts,) if cfg.shared_ffn else ()):
        for t in range(3):
            rows, K = (f, h) if t < 2 else (h, f)
            sc = _scale(h) if t < 2 else _scale(f)
            w = O.bf16_to_f32(orc.fill_bf16(orc.tensor_seed(cfg.weight_seed, 0, e, t), rows * K, sc))
            oc, osf, os_ = orc.nvfp4_quant_rows(w.reshape(rows, K))
            assert (ctxs4[name].read_expert(0, e, t) == oc).all(), (e, t)
            assert (ctxs4[name].read_expert(0, e, 3 + t) == os_).all(), (e, t)
            assert (ctxs4[name].read_expert(0, e, 6 + t) == orc.nvfp4_sf_atoms(osf)).all(), (e, t)


@pytest.mark.parametrize("name,T", [("tiny_fp4", 1), ("tiny_fp4", 300), ("mid_fp4", 200),
                                    ("mid_fp4", 1), ("mid_fp4", 2000), ("r1_fp4", 16)])
def test_moe_forward_nvfp4_vs_oracle(dev, ctxs4, orc, name, T):
    cfg = FP4_CONFIGS[name]
    x = make_x(T, cfg.hidden, 11 + T, dev)
    y = ctxs4[name].moe_forward(0, x)
    idx, wts, _, _, _ = ctxs4[name].route(0, x)
    torch.cuda.synchronize()
    oc = oracle_cfg(cfg)
    oc.w8a8 = 2
    yo4, oidx, owts = orc.moe_forward_seeded(oc, cfg.weight_seed, 0, _bf16_np(x).reshape(-1), T,
                                             _bias(cfg))
    yo, _, _ = orc.moe_forward_seeded(oracle_cfg(cfg), cfg.weight_seed, 0, _bf16_np(x).reshape(-1), T,
                                      _bias(cfg))
    assert (idx.cpu().numpy() == oidx).all() and (wts.cpu().numpy() == owts).all()
    yd = y.float().cpu().numpy()
    assert _rel(yd, yo4) < TOL_FP4, _rel(yd, yo4)
    assert _rel(yd, yo) < TOL_FP4_Q, _rel(yd, yo)


def test_moe_forward_nvfp4_single_cta(dev, orc, monkeypatch):
    """GEMM1 on the 1-SM kernel (DWDP_FP4_PAIR=0) vs the oracle and bitwise vs
    the CTA-pair build of the same layer (rows are independent)."""
    cfg = FP4_CONFIGS["mid_fp4"]
    x = make_x(2000, cfg.hidden, 2011, dev)
    pair = D.DwdpContext(cfg)
    monkeypatch.setenv("DWDP_FP4_PAIR", "0")
    single = D.DwdpContext(cfg)
    for c in (pair, single):
        c.init_weights()
        c.set_bias(_bias(cfg))
    y1, y0 = pair.moe_forward(0, x), single.moe_forward(0, x)
    torch.cuda.synchronize()
    oc = oracle_cfg(cfg)
    oc.w8a8 = 2
    yo4, _, _ = orc.moe_forward_seeded(oc, cfg.weight_seed, 0, _bf16_np(x).reshape(-1), 2000, _bias(cfg))
    assert _rel(y0.float().cpu().numpy(), yo4) < TOL_FP4
    assert _rel(y1.float().cpu().numpy(), yo4) < TOL_FP4
    pair.close()
    single.close()


def test_dwdp_nvfp4_group_of_two_matches_all_local(dev):
    """NVFP4 arenas (codes + row scales + block scales) prefetched over both
    engines, and with the merged-weight fetch (D2D merge of all nine
    tensors), give bit-identical outputs to the all-local NVFP4 model."""
    kw = dict(MID, weight_dtype=D.WEIGHT_NVFP4)
    full = D.DwdpContext(D.DwdpConfig(**kw))
    full.init_weights()
    for engine, merge in ((D.ENGINE_COPY, 1), (D.ENGINE_PULL, 1), (D.ENGINE_COPY, 0)):
        ranks = [D.DwdpContext(D.DwdpConfig(**kw, rank=r, group_size=2, engine=engine, merge_elim=merge,
                                            slice_size=1 << 18)) for r in range(2)]
        for c in ranks:
            c.init_weights()
        D.DwdpContext.link_local(ranks)
        xs = [make_x(90 + 41 * r, MID["hidden"], 70 + r, dev) for r in range(2)]
        for g in range(4):
            for r in range(2):
                y = ranks[r].layer_forward(g, xs[r], residual=False)
                yf = full.moe_forward(g % 3, xs[r])
                torch.cuda.synchronize()
                assert torch.equal(y, yf), (engine, g, r)
        recs = ranks[0].records()
        # (E - c) experts x (3 code tensors + 3 fp32 row-scale vectors + 3 block-scale tensors)
        h, f = MID["hidden"], MID["ffn"]
        assert recs[1]["prefetch_bytes"] == 32 * (3 * h * f // 2 + 4 * (2 * f + h) + 3 * h * f // 16)
        for c in ranks:
            c.close()
    full.close()


@pytest.mark.parametrize("group,extra,engine,T0", [(3, 1, D.ENGINE_PULL, 64), (2, 0, D.ENGINE_COPY, 1900)])
def test_dwdp_nvfp4_placements_and_large_batches(dev, group, extra, engine, T0):
    """NVFP4 arenas under a non-divisible redundant placement (multi-run
    shards over all nine tensors) and at batches whose GEMM1 runs on CTA pairs
    (>= 128 routed rows per expert): bit-identical to the all-local model."""
    kw = dict(MID, weight_dtype=D.WEIGHT_NVFP4, max_tokens=4096)
    full = D.DwdpContext(D.DwdpConfig(**kw))
    full.init_weights()
    ranks = [D.DwdpContext(D.DwdpConfig(**kw, rank=r, group_size=group, extra_redundancy=extra,
                                        engine=engine, slice_size=1 << 19)) for r in range(group)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    plan = D.build_placement(MID["num_experts"], group, extra)
    xs = [make_x(T0 + 29 * r, MID["hidden"], 90 + r, dev) for r in range(group)]
    for g in range(4):
        for r in range(group):
            y = ranks[r].layer_forward(g, xs[r], residual=False)
            yf = full.moe_forward(g % 3, xs[r])
            torch.cuda.synchronize()
            assert torch.equal(y, yf), (group, extra, g, r)
    h, f = MID["hidden"], MID["ffn"]
    for r in range(group):
        fetched = len(plan.fetch_lists[r])
        assert ranks[r].records()[1]["prefetch_bytes"] == fetched * (3 * h * f // 2 + 4 * (2 * f + h) + 3 * h * f // 16)
    for c in ranks + [full]:
        c.close()
