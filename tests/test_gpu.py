"""GPU parity tests: the sm_100a path through the C-ABI against the oracle.

Bar: routing indices, weights, expert counts and permutation rows bit-exact;
layer outputs within normwise relative error 1e-2 of the oracle's fp32
(bf16 storage of H, O and y), GEMM within 1e-2 of a torch fp32 reference.
"""
import numpy as np
import pytest
import torch

import paper_2604_01621_b200 as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2  # normwise relative error vs the oracle's fp32 (stated in BASELINE.md §3)


def _bf16_np(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _scale(n):
    return float(np.float32(1.0) / np.sqrt(np.float32(n)))


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    assert torch.cuda.get_device_capability(0) == (10, 0), "sm_100 required"
    return torch.device("cuda:0")


def make_x(T, h, seed, dev):
    x = torch.empty((T, h), dtype=torch.bfloat16, device=dev)
    if T:
        D.fill_bf16(x, seed, 1.0)
    torch.cuda.synchronize()
    return x


def oracle_cfg(c: D.DwdpConfig):
    return O.MoeConfig(c.hidden, c.num_experts, c.top_k, c.ffn, c.shared_ffn, c.scoring,
                       c.n_group, c.topk_group, c.norm_topk, c.routed_scale)


CONFIGS = {
    "tiny": D.DwdpConfig.tiny(),  # BASELINE config 1 layer (softmax top-2, E16, h512)
    "tiny_shared": D.DwdpConfig.tiny(shared_ffn=1024),
    # T = 2000: ~190 rows per expert, so expert segments span a full CTA pair
    "mid_sigmoid": D.DwdpConfig(num_layers=1, num_experts=64, hidden=1024, ffn=256, shared_ffn=256,
                                top_k=6, n_group=8, topk_group=4, max_tokens=2048),
    "r1": D.DwdpConfig(num_layers=1, max_tokens=512),  # BASELINE config 2 shapes
    # top-k kernel variants: contiguous-lane layout with 8 lanes per group, and
    # softmax over all E without renormalisation (norm_topk = 0)
    "e128_g4": D.DwdpConfig(num_layers=1, num_experts=128, hidden=512, ffn=256, shared_ffn=256,
                            top_k=4, n_group=4, topk_group=2, max_tokens=512),
    "e32_softmax": D.DwdpConfig(num_layers=1, num_experts=32, hidden=512, ffn=256, shared_ffn=0, top_k=3,
                                scoring=0, n_group=1, topk_group=1, norm_topk=0, routed_scale=1.0,
                                max_tokens=512),
}


@pytest.fixture(scope="module")
def ctxs(dev):
    out = {}
    for name, cfg in CONFIGS.items():
        c = D.DwdpContext(cfg)
        c.init_weights()
        if cfg.scoring == 1:
            c.set_bias((np.arange(cfg.num_experts) % 7 - 3).astype(np.float32) * 0.01)
        out[name] = c
    yield out
    for c in out.values():
        c.close()


def _bias(cfg):
    if cfg.scoring != 1:
        return None
    return (np.arange(cfg.num_experts) % 7 - 3).astype(np.float32) * 0.01


# ---------------------------------------------------------------- kernels

def test_fill_matches_oracle(dev, orc):
    t = torch.empty(100_003, dtype=torch.bfloat16, device=dev)
    D.fill_bf16(t, 12345, 0.37)
    torch.cuda.synchronize()
    assert (_bf16_np(t) == orc.fill_bf16(12345, t.numel(), 0.37)).all()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 1024), (1, 256, 7168),
                                   (2048, 7168, 2048), (1000, 4096, 7168)])
def test_gemm_vs_torch(dev, M, N, K):
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    A = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    B = (torch.randn((N, K), device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    Dm = D.gemm_bf16(A, B)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    assert _rel(Dm.float().cpu().numpy(), ref.cpu().numpy()) < TOL


# ---------------------------------------------------------------- routing

@pytest.mark.parametrize("name,T", [("tiny", 1), ("tiny", 7), ("tiny", 64), ("tiny", 1000),
                                    ("mid_sigmoid", 1), ("mid_sigmoid", 333),
                                    ("r1", 1), ("r1", 37), ("r1", 256), ("e128_g4", 77),
                                    ("e32_softmax", 129)])
def test_route_bit_exact(dev, ctxs, orc, name, T):
    cfg = CONFIGS[name]
    ctx = ctxs[name]
    x = make_x(T, cfg.hidden, 99 + T, dev)
    idx, wts, counts, row_of, rows = ctx.route(0, x)
    torch.cuda.synchronize()
    wr = orc.fill_bf16(orc.tensor_seed(cfg.weight_seed, 0, cfg.num_experts + 1, 0),
                       cfg.num_experts * cfg.hidden, _scale(cfg.hidden))
    _, oidx, owts = orc.route(oracle_cfg(cfg), _bf16_np(x).reshape(-1), T, wr, _bias(cfg))
    assert (idx.cpu().numpy() == oidx).all()
    assert (wts.cpu().numpy().view(np.uint32) == owts.view(np.uint32)).all()  # bitwise
    total, ocounts, orow = orc.permute(oidx, cfg.num_experts, 128)
    assert (counts.cpu().numpy() == ocounts).all()
    assert (row_of.cpu().numpy() == orow).all()
    assert rows == total


# ---------------------------------------------------------------- layer forward

@pytest.mark.parametrize("name,T", [("tiny", 1), ("tiny", 64), ("tiny", 1000), ("tiny_shared", 129),
                                    ("mid_sigmoid", 200), ("mid_sigmoid", 2000),
                                    ("r1", 16), ("r1", 300)])
def test_moe_forward_vs_oracle(dev, ctxs, orc, name, T):
    cfg = CONFIGS[name]
    ctx = ctxs[name]
    x = make_x(T, cfg.hidden, 7 + T, dev)
    y = ctx.moe_forward(0, x)
    torch.cuda.synchronize()
    yo, _, _ = orc.moe_forward_seeded(oracle_cfg(cfg), cfg.weight_seed, 0,
                                      _bf16_np(x).reshape(-1), T, _bias(cfg))
    err = _rel(y.float().cpu().numpy(), yo)
    assert err < TOL, err


# ---------------------------------------------------------------- fp8 W8A8

TOL_FP8 = 1e-2   # vs the oracle's W8A8 emulation (fp32 sum order, rare bf16-H ulp flips)
TOL_FP8_Q = 8e-2  # quantisation error vs the bf16 oracle (e4m3 weights + activations)

FP8_CONFIGS = {
    "tiny_fp8": D.DwdpConfig.tiny(weight_dtype=D.WEIGHT_FP8),
    "mid_fp8": D.DwdpConfig(num_layers=1, num_experts=64, hidden=1024, ffn=256, shared_ffn=256,
                            top_k=6, n_group=8, topk_group=4, max_tokens=2048,
                            weight_dtype=D.WEIGHT_FP8),
    "r1_fp8": D.DwdpConfig(num_layers=1, max_tokens=512, weight_dtype=D.WEIGHT_FP8),
}


@pytest.fixture(scope="module")
def ctxs8(dev):
    out = {}
    for name, cfg in FP8_CONFIGS.items():
        c = D.DwdpContext(cfg)
        c.init_weights()
        if cfg.scoring == 1:
            c.set_bias(_bias(cfg))
        out[name] = c
    yield out
    for c in out.values():
        c.close()


@pytest.mark.parametrize("name", ["tiny_fp8", "mid_fp8"])
def test_fp8_weights_bit_exact(dev, ctxs8, orc, name):
    """Resident e4m3 expert rows + per-row scales == oracle quantisation of
    the same counter-hash bf16 rows."""
    cfg = FP8_CONFIGS[name]
    h, f = cfg.hidden, cfg.ffn
    for e in (0, cfg.num_experts - 1) + ((cfg.num_experts,) if cfg.shared_ffn else ()):
        for t in range(3):
            rows, K = (f, h) if t < 2 else (h, f)
            sc = _scale(h) if t < 2 else _scale(f)
            w = O.bf16_to_f32(orc.fill_bf16(orc.tensor_seed(cfg.weight_seed, 0, e, t), rows * K, sc))
            q = ctxs8[name].read_expert(0, e, t)
            s = ctxs8[name].read_expert(0, e, 3 + t)
            for r in (0, 1, rows // 2, rows - 1):
                oq, os_ = orc.quant_row_e4m3(w[r * K:(r + 1) * K])
                assert (q[r] == oq).all(), (e, t, r)
                assert np.float32(s[r]) == np.float32(os_), (e, t, r)


@pytest.mark.parametrize("name,T", [("tiny_fp8", 1), ("tiny_fp8", 300), ("mid_fp8", 200),
                                    ("mid_fp8", 1), ("mid_fp8", 2000), ("r1_fp8", 16)])
def test_moe_forward_fp8_vs_oracle(dev, ctxs8, orc, name, T):
    cfg = FP8_CONFIGS[name]
    x = make_x(T, cfg.hidden, 11 + T, dev)
    y = ctxs8[name].moe_forward(0, x)
    torch.cuda.synchronize()
    oc = oracle_cfg(cfg)
    oc.w8a8 = 1
    yo8, _, _ = orc.moe_forward_seeded(oc, cfg.weight_seed, 0, _bf16_np(x).reshape(-1), T, _bias(cfg))
    yo, _, _ = orc.moe_forward_seeded(oracle_cfg(cfg), cfg.weight_seed, 0, _bf16_np(x).reshape(-1), T,
                                      _bias(cfg))
    yd = y.float().cpu().numpy()
    assert _rel(yd, yo8) < TOL_FP8, _rel(yd, yo8)
    assert _rel(yd, yo) < TOL_FP8_Q, _rel(yd, yo)


def test_dwdp_fp8_group_of_two_matches_all_local(dev):
    """fp8 arenas (weights + scale tensors) prefetched over the pull kernel
    give bit-identical outputs to the all-local fp8 model."""
    kw = dict(MID, weight_dtype=D.WEIGHT_FP8)
    full = D.DwdpContext(D.DwdpConfig(**kw))
    full.init_weights()
    for engine in (D.ENGINE_COPY, D.ENGINE_PULL):
        ranks = [D.DwdpContext(D.DwdpConfig(**kw, rank=r, group_size=2, engine=engine,
                                            slice_size=1 << 20)) for r in range(2)]
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
        # (E - c) experts x (3 e4m3 tensors + 3 fp32 scale vectors)
        h, f = MID["hidden"], MID["ffn"]
        assert recs[1]["prefetch_bytes"] == 32 * (3 * h * f + 4 * (2 * f + h))
        for c in ranks:
            c.close()
    full.close()


def test_empty_batch_is_a_noop(dev, ctxs):
    x = torch.empty((0, 512), dtype=torch.bfloat16, device=dev)
    ctxs["tiny"].moe_forward(0, x)
    torch.cuda.synchronize()


def test_stack_forward_residual(dev, orc):
    cfg = D.DwdpConfig.tiny(num_layers=2, max_tokens=256)
    ctx = D.DwdpContext(cfg)
    ctx.init_weights()
    x = make_x(50, cfg.hidden, 3, dev)
    y = ctx.stack_forward(x)
    torch.cuda.synchronize()
    xf = _bf16_np(x).reshape(-1)
    h = O.bf16_to_f32(xf).reshape(50, -1)
    for layer in range(2):
        yo, _, _ = orc.moe_forward_seeded(oracle_cfg(cfg), cfg.weight_seed, layer,
                                          O.bf16_round(h).reshape(-1), 50, None)
        h = h + yo
    assert _rel(y.float().cpu().numpy(), h) < TOL
    recs = ctx.records()
    assert [r["global_layer"] for r in recs] == [0, 1]
    assert ctx.launch_count() > 0
    ctx.close()


# ---------------------------------------------------------------- DWDP on one GPU

MID = dict(num_layers=3, num_experts=64, hidden=1024, ffn=256, shared_ffn=256, top_k=6,
           n_group=8, topk_group=4, max_tokens=512, weight_layers=3)


@pytest.mark.parametrize("engine,tdm,slice_size,merge", [(D.ENGINE_COPY, 1, 1 << 20, 1),
                                                          (D.ENGINE_PULL, 1, 1 << 20, 1),
                                                          (D.ENGINE_HYBRID, 1, 1 << 20, 1),
                                                          (D.ENGINE_COPY, 0, 1 << 20, 1),
                                                          (D.ENGINE_COPY, 1, 300_000, 0)])
def test_dwdp_group_of_two_matches_all_local(dev, engine, tdm, slice_size, merge):
    """Two DWDP ranks (one process, one GPU) pulling from each other give the
    same layer outputs, bit for bit, as the all-local model (same seed)."""
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = [D.DwdpContext(D.DwdpConfig(**MID, rank=r, group_size=2, engine=engine, tdm=tdm,
                                        slice_size=slice_size, merge_elim=merge))
             for r in range(2)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    xs = [make_x(100 + 37 * r, MID["hidden"], 50 + r, dev) for r in range(2)]
    for g in range(5):  # crosses an iteration boundary (L = 3)
        for r in range(2):
            y = ranks[r].layer_forward(g, xs[r], residual=False)
            yf = full.moe_forward(g % 3, xs[r])
            torch.cuda.synchronize()
            assert torch.equal(y, yf), (g, r)
    # received experts are byte-identical to the owner's copy
    plan = D.build_placement(64, 2)
    for r in range(2):
        for e, src in plan.fetch_lists[r][:4]:
            for t in range(3):
                layer = 4 % 3
                assert (ranks[r].read_expert(layer, e, t) == ranks[src].read_expert(layer, e, t)).all()
    recs = ranks[0].records()
    assert len(recs) == 5
    pf = recs[1]["prefetch_bytes"]
    assert pf == 32 * 3 * MID["hidden"] * MID["ffn"] * 2  # (E - c) * expert_shard_bytes
    assert all(r["gate_wait_ns"] >= 0 for r in recs)
    for c in ranks + [full]:
        c.close()


def test_prefetch_handles(dev):
    ranks = [D.DwdpContext(D.DwdpConfig(**MID, rank=r, group_size=2)) for r in range(2)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    h = ranks[0].prefetch_issue(0)
    assert h >= 0
    ranks[0].prefetch_wait(h)
    torch.cuda.synchronize()
    assert ranks[0].prefetch_query(h)
    s, e, b = ranks[0].prefetch_times(h)
    assert 0 <= s <= e and b == 32 * 3 * MID["hidden"] * MID["ffn"] * 2
    with pytest.raises(D.InvariantViolation):
        ranks[0].prefetch_issue(0)  # double issue (simcore.cpp:624)
    plan = ranks[0].copy_plan()
    assert sum(s.length for s in plan) == b
    for c in ranks:
        c.close()


@pytest.mark.parametrize("name,mode", [("mid_sigmoid", "1"), ("mid_fp8", "1"), ("mid_sigmoid", "3"),
                                       ("mid_fp8", "3"), ("mid_sigmoid", "4")])
def test_gemm_pair_matches_single_cta(dev, monkeypatch, name, mode):
    """The CTA-pair GEMM (cta_group::2, 256-row segments; DWDP_GEMM_PAIR=1 for
    every GEMM, =3 for GEMM2 and the router only, =4 the split layout: GEMM1
    1-SM on 128-row segments writing H into 256-row segments, GEMM2 on pairs)
    gives the
    same layer outputs as the all-1-SM kernels (DWDP_GEMM_PAIR=0; bf16 and
    e4m3 weights; routing included)."""
    cfg = CONFIGS.get(name) or FP8_CONFIGS[name]
    outs = []
    for pair in (mode, "0"):
        monkeypatch.setenv("DWDP_GEMM_PAIR", pair)
        c = D.DwdpContext(cfg)
        c.init_weights()
        c.set_bias(_bias(cfg))
        x = make_x(2000, cfg.hidden, 5, dev)  # >= 128 rows per expert: the pair path is taken
        outs.append(c.moe_forward(0, x).float().cpu().numpy())
        torch.cuda.synchronize()
        c.close()
    assert _rel(outs[0], outs[1]) < 1e-3


@pytest.mark.parametrize("group,extra,engine", [(3, 0, D.ENGINE_COPY), (3, 1, D.ENGINE_PULL),
                                                (2, 5, D.ENGINE_COPY), (5, 0, D.ENGINE_HYBRID)])
def test_dwdp_non_divisible_and_redundant_placements(dev, group, extra, engine):
    """non-divisible (N = 3, 5) and redundant (extra > 0)
    placements. Ranks own overlapping expert arcs, fetch sources come from
    assign_fetch_sources and a peer's slots can form several contiguous runs
    (multi-run shards); outputs stay bit-identical to the all-local model."""
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = [D.DwdpContext(D.DwdpConfig(**MID, rank=r, group_size=group, extra_redundancy=extra,
                                        engine=engine, slice_size=1 << 20))
             for r in range(group)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    plan = D.build_placement(MID["num_experts"], group, extra)
    xs = [make_x(64 + 29 * r, MID["hidden"], 90 + r, dev) for r in range(group)]
    for g in range(4):
        for r in range(group):
            y = ranks[r].layer_forward(g, xs[r], residual=False)
            yf = full.moe_forward(g % 3, xs[r])
            torch.cuda.synchronize()
            assert torch.equal(y, yf), (group, extra, g, r)
    for r in range(group):
        recs = ranks[r].records()
        fetched = len(plan.fetch_lists[r])
        assert recs[1]["prefetch_bytes"] == fetched * 3 * MID["hidden"] * MID["ffn"] * 2
        for e, src in plan.fetch_lists[r][:3]:
            assert (ranks[r].read_expert(3 % 3, e, 0) == ranks[src].read_expert(3 % 3, e, 0)).all()
    for c in ranks + [full]:
        c.close()


@pytest.mark.parametrize("engine", [D.ENGINE_COPY, D.ENGINE_PULL])
def test_dwdp_large_batch_bitwise(dev, engine):
    """DWDP at ~180-350 rows per expert (segments spanning CTA pairs, several
    permute chunks) stays bit-identical to the all-local model."""
    kw = dict(MID, max_tokens=4096)
    full = D.DwdpContext(D.DwdpConfig(**kw))
    full.init_weights()
    ranks = [D.DwdpContext(D.DwdpConfig(**kw, rank=r, group_size=2, engine=engine)) for r in range(2)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    xs = [make_x(1900 + 1800 * r, MID["hidden"], 300 + r, dev) for r in range(2)]
    for g in range(3):
        for r in range(2):
            y = ranks[r].layer_forward(g, xs[r], residual=False)
            yf = full.moe_forward(g % 3, xs[r])
            torch.cuda.synchronize()
            assert torch.equal(y, yf), (engine, g, r)
    for c in ranks + [full]:
        c.close()


def test_gemm1_gather_matches_permuted_copy(dev, monkeypatch):
    """GEMM1 gathering the routed rows from x (cp.async into the swizzled
    tile, no X_perm copy; DWDP_GATHER=1) gives bit-identical layer outputs."""
    cfg = CONFIGS["mid_sigmoid"]
    outs = []
    for g in ("1", "0"):
        monkeypatch.setenv("DWDP_GATHER", g)
        c = D.DwdpContext(cfg)
        c.init_weights()
        c.set_bias(_bias(cfg))
        x = make_x(1500, cfg.hidden, 21, dev)
        outs.append(c.moe_forward(0, x))
        torch.cuda.synchronize()
        c.close()
    assert torch.equal(outs[0], outs[1])


# ---------------------------------------------------------------- error contract

@pytest.mark.parametrize("bad", [dict(hidden=300), dict(ffn=100), dict(top_k=0), dict(top_k=17),
                                 dict(num_experts=600), dict(rank=2, group_size=2),
                                 dict(n_group=5), dict(topk_group=9), dict(scoring=3),
                                 dict(engine=7), dict(slice_size=1000), dict(shared_ffn=512),
                                 dict(weight_dtype=5), dict(max_tokens=0)])
def test_config_errors_are_config_errors(dev, bad):
    """Invalid configurations fail with ConfigError (status 2, reference
    errors.hpp:11-15) before touching the GPU, never with a CUDA error."""
    kw = dict(num_layers=1, num_experts=64, hidden=1024, ffn=256, shared_ffn=256, top_k=6,
              n_group=8, topk_group=4, max_tokens=64)
    kw.update(bad)
    with pytest.raises(D.ConfigError):
        D.DwdpContext(D.DwdpConfig(**kw))


def test_call_errors(dev, ctxs):
    ctx = ctxs["tiny"]
    x = make_x(2000, 512, 1, dev)
    with pytest.raises(D.ConfigError):
        ctx.moe_forward(0, x)  # T > max_tokens
    with pytest.raises(D.ConfigError):
        ctx.moe_forward(5, x[:10])  # layer out of range
    with pytest.raises(D.ConfigError):
        ctx.read_expert(0, 99, 0)
    lonely = D.DwdpContext(D.DwdpConfig(**MID, rank=0, group_size=2))
    with pytest.raises(D.ConfigError):
        lonely.prefetch_issue(1)  # peers not wired
    lonely.close()


def test_stack_matches_layer_by_layer_bitwise(dev):
    """stack_forward (ping-pong buffers, prefetch chain) against the same
    layers called one by one with residual, bit for bit."""
    cfg = D.DwdpConfig(**MID)
    a, b = D.DwdpContext(cfg), D.DwdpContext(cfg)
    a.init_weights()
    b.init_weights()
    x = make_x(300, cfg.hidden, 5, dev)
    y_stack = a.stack_forward(x)
    h = x
    for g in range(cfg.num_layers):
        h = b.layer_forward(g, h, residual=True)
    torch.cuda.synchronize()
    assert torch.equal(y_stack, h)
    a.close()
    b.close()
