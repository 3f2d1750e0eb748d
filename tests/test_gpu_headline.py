"""Parity at the headline configuration (BASELINE config 2 as bench.py runs it).

bench.py's default N=1 step runs one rank's batch of ~61K tokens (ISL 8K, CV
0.2, MNT 65536: sample_batches, reference src/workload.cpp:137-173) through
R1-shaped layers. These tests run THAT batch -- the same T, the same x
(counter hash 0xC0FFEE), the same weights -- and check it against the CPU
oracle (oracle/check.py):

* routing of all T tokens bit-exact (indices, fp32 weights, per-expert counts,
  permutation rows; rows sum to T*k, include/dwdpsim/workload.hpp:50-52). At
  this T the permute runs with its large-batch chunk size (128 pairs per warp
  chunk, T >= 37,888; kernels.cu), which no smaller test reaches, and the
  shared-expert segment (T rows, 480+ m-blocks) takes the m-block-major raster;
* the layer output on 512 sampled rows within normwise and per-row relative
  error 1e-2 of the oracle's fp32 (each MoE row depends only on its token);
* DWDP with two ranks (one GPU, link_local) at full R1 shapes -- 128 owned
  experts each, 128 x 88 MB pulled per layer -- bit-identical to the
  all-local model across an iteration boundary (simcore.cpp:486-515 shards,
  :640-733 gate / double buffer).
"""
import numpy as np
import pytest
import torch

import paper_2604_01621_b200 as D
from oracle import check as CK

pytestmark = pytest.mark.gpu

TOL = 1e-2


def bench_tokens(it: int = 5, mnt: int = 65536, cv: float = 0.2) -> int:
    """Rank 0's token count of bench.py's step `it` (default: the first timed
    step of `bench.py --steps 20 --warmup 5`)."""
    spec = D.WorkloadSpec(D.IslDist.from_cv(8192, cv), mnt, max(1, mnt // 8192), 0.0, 7)
    batches = D.sample_batches(spec, D.r1_model(8), 1, it + 1, with_routing=False)
    return int(batches[it].tokens[0])


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def test_bench_batch_is_large():
    T = bench_tokens()
    assert 37_888 <= T <= 65_536, T


@pytest.mark.parametrize("bias", [None, "ramp"])
def test_headline_layer_vs_oracle(dev, bias):
    T = bench_tokens()
    cfg = D.DwdpConfig(num_layers=8, weight_layers=1, max_tokens=65536)
    ctx = D.DwdpContext(cfg)
    try:
        ctx.init_weights()
        b = None
        if bias == "ramp":  # noaux_tc selection bias (e.g. the Zipf-skew bias of bench --zipf)
            b = (-0.04 * np.log(np.arange(cfg.num_experts) + 1.0)).astype(np.float32)
            ctx.set_bias(b)
        x = torch.empty((T, cfg.hidden), dtype=torch.bfloat16, device=dev)
        D.fill_bf16(x, 0xC0FFEE, 1.0)
        res = CK.check_layer(ctx, x, layer=0, sample_rows=512, seed=T, bias=b)
        print(res)
        assert res["idx_mismatch_tokens"] == 0, res
        assert res["wts_mismatch_tokens"] == 0, res
        assert res["counts_equal"] and res["row_of_equal"] and res["rows_equal"], res
        assert res["sample_routing_equal"], res
        assert res["rel_err_normwise"] < TOL, res
        assert res["max_row_rel_err"] < TOL, res
        assert res["ok"]
    finally:
        ctx.close()


def test_headline_stack_rows_finite_and_deterministic(dev):
    """The 8-layer stack bench.py times: finite outputs and run-to-run
    bit-identical (fixed combine order, no atomics in the data path)."""
    T = bench_tokens()
    cfg = D.DwdpConfig(num_layers=8, weight_layers=1, max_tokens=65536)
    ctx = D.DwdpContext(cfg)
    try:
        ctx.init_weights()
        x = torch.empty((T, cfg.hidden), dtype=torch.bfloat16, device=dev)
        D.fill_bf16(x, 0xC0FFEE, 1.0)
        y1 = ctx.stack_forward(x)
        y2 = ctx.stack_forward(x)
        torch.cuda.synchronize()
        assert torch.isfinite(y1.float()).all()
        assert torch.equal(y1, y2)
    finally:
        ctx.close()


def test_dwdp_two_ranks_r1_shapes_bitwise(dev):
    """DWDP(N=2) at full R1 shapes on one GPU (two contexts wired with
    link_local, TMA pull and copy engine) == the all-local layer, bitwise."""
    L = 2
    kw = dict(num_layers=L, weight_layers=L, max_tokens=4096)
    full = D.DwdpContext(D.DwdpConfig(**kw))
    ranks = []
    try:
        full.init_weights()
        ranks = [D.DwdpContext(D.DwdpConfig(**kw, rank=r, group_size=2,
                                            engine=(D.ENGINE_PULL, D.ENGINE_COPY)[r],
                                            slice_size=64 << 20))
                 for r in range(2)]
        for c in ranks:
            c.init_weights()
        D.DwdpContext.link_local(ranks)
        xs = []
        for r, T in enumerate((4096, 1531)):
            x = torch.empty((T, 7168), dtype=torch.bfloat16, device=dev)
            D.fill_bf16(x, 0xC0FFEE + r, 1.0)
            xs.append(x)
        for g in range(2 * L + 1):  # crosses the iteration boundary twice
            for r in range(2):
                y = ranks[r].layer_forward(g, xs[r], residual=False)
                yf = full.moe_forward(g % L, xs[r])
                torch.cuda.synchronize()
                assert torch.equal(y, yf), (g, r)
        for r in range(2):
            recs = ranks[r].records()
            assert recs[1]["prefetch_bytes"] == 128 * D.expert_shard_bytes(D.r1_model(L))
            for e, src in D.build_placement(256, 2).fetch_lists[r][:2]:
                for t in range(3):
                    assert (ranks[r].read_expert((2 * L) % L, e, t)
                            == ranks[src].read_expert((2 * L) % L, e, t)).all()
    finally:
        for c in ranks + [full]:
            c.close()
