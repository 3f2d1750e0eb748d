"""Pins the C restatement oracle (oracle/dwdp_oracle.c) before trusting it:
against golden outputs of the compiled reference library (tests/golden/ref_*),
against the live reference library when present, and the MoE numerics against
transformers' DeepseekV3MoE / Qwen2MoeTopKRouter (tests/golden/hf_moe.json)."""
import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O


def test_rng_mix_and_mt64_golden(orc):
    g = load_golden("ref_workload.json")
    for seed, seq in g["u64"].items():
        assert orc.rng_u64(int(seed), len(seq)).tolist() == [int(v) for v in seq]
    for a, b, m in g["mix"]:
        assert orc.mix(int(a), int(b)) == int(m)
    for seed, seq in g["normal"].items():
        assert orc.rng_normal(int(seed), len(seq), 3.0, 2.0).tolist() == seq


def test_placement_golden(orc):
    for c in load_golden("ref_placement.json"):
        st, lc, red, local, fetch = orc.build_placement(c["E"], c["N"], c["extra"])
        assert st == c["status"], c
        if st:
            continue
        assert (lc, red) == (c["local_count"], c["redundancy"])
        assert local == c["local_sets"]
        assert [[list(p) for p in f] for f in fetch] == (c["fetch"] or [[] for _ in local])


def _plan_checksum(slices):
    arr = np.array(slices, np.int64)
    return int((arr * (np.arange(len(arr))[:, None] + 1) % 1000003).sum())


def test_copy_plan_golden(orc):
    for c in load_golden("ref_copyplan.json"):
        st, slices = orc.build_copy_plan([tuple(s) for s in c["shards"]], c["slice"], c["dst"])
        assert st == c["status"], c
        if st:
            continue
        if "slices" in c:
            assert [list(s) for s in slices] == c["slices"]
        else:
            assert len(slices) == c["n_slices"]
            assert [list(s) for s in slices[:64]] == c["head"]
            assert _plan_checksum(slices) == c["checksum"]


def test_workload_golden(orc):
    g = load_golden("ref_workload.json")
    for c in g["route"]:
        st, cnt = orc.route_tokens(c["tokens"], c["E"], c["k"], c["skew"], c["seed"])
        assert st == 0 and cnt.tolist() == c["counts"]
    for c in g["batches"]:
        spec = c["spec"]
        st, t, q, r = orc.sample_batches(*spec, 256, 8, c["N"], c["iters"], routed=spec[6] > 0)
        assert st == 0
        assert t.tolist() == c["tokens"] and q.tolist() == c["requests"]
        if "routed_rank0_iter0" in c:
            assert r[0, 0].tolist() == c["routed_rank0_iter0"]


def test_costs_golden(orc):
    g = load_golden("ref_costs.json")
    for h, f, wb, b in g["shard_bytes"]:
        assert orc.expert_shard_bytes(h, f, wb) == b
    for c in g["moe_entries"]:
        T = c["T"]
        assert orc.moe_entries(7168, 2048, 2048, 2.0, 2.0, T, T * 8, 256).tolist() == c["out"]


def test_live_reference_matches_oracle(orc, ref):
    """Randomised cross-check against the reference library itself."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        N = int(rng.integers(2, 12))
        E = N + int(rng.integers(0, 300))
        x = int(rng.integers(0, 6))
        assert orc.build_placement(E, N, x) == ref.build_placement(E, N, x)
    for _ in range(100):
        sh = [(int(p), int(t), int(rng.integers(1, 3000)), int(rng.integers(0, 50)))
              for t in range(int(rng.integers(1, 4))) for p in range(1, int(rng.integers(2, 6)))]
        s, d = int(rng.integers(1, 500)), int(rng.integers(0, 7))
        assert orc.build_copy_plan(sh, s, d) == ref.build_copy_plan(sh, s, d)
    for seed in range(20):
        a = orc.route_tokens(777, 64, 4, 0.9, seed)[1]
        b = ref.route_tokens(777, 64, 4, 0.9, seed)[1]
        assert (a == b).all()


def _cfg(c, scoring):
    if scoring == 1:
        return O.MoeConfig(c["h"], c["E"], c["k"], c["f"], c["f"], 1, c["n_group"],
                           c["topk_group"], 1, 2.5)
    return O.MoeConfig(c["h"], c["E"], c["k"], 64, 0, 0, 1, 1, 1, 1.0)


@pytest.mark.parametrize("case", range(3))
def test_oracle_matches_hf_deepseek_v3_moe(orc, case):
    c = load_golden("hf_moe.json")["deepseek"][case]
    h, E, f, T = c["h"], c["E"], c["f"], c["T"]
    B = lambda n: O.bf16_to_f32(np.array(c[n], np.uint16))  # noqa: E731
    gu = B("gate_up").reshape(E, 2 * f, h)
    y, idx, w = orc.moe_forward_explicit(
        _cfg(c, 1), B("x").reshape(T, h), np.array(c["w_router"], np.float32),
        np.array(c["bias"], np.float32), gu[:, :f], gu[:, f:], B("down").reshape(E, h, f),
        B("s_gate").reshape(f, h), B("s_up").reshape(f, h), B("s_down").reshape(h, f))
    order = np.argsort(idx, 1)
    assert (np.take_along_axis(idx, order, 1) == np.array(c["idx_sorted"])).all()
    np.testing.assert_allclose(np.take_along_axis(w, order, 1), c["wts_sorted"], rtol=0, atol=1e-6)
    yref = np.array(c["y"], np.float32)
    assert np.abs(y - yref).max() <= 1e-5 * np.abs(yref).max()


@pytest.mark.parametrize("case", range(2))
def test_oracle_matches_hf_softmax_router(orc, case):
    c = load_golden("hf_moe.json")["softmax"][case]
    x = np.array(c["x"], np.uint16)
    wr = O.bf16_round(np.array(c["w_router"], np.float32))
    _, idx, w = orc.route(_cfg(c, 0), x, c["T"], wr, None)
    order = np.argsort(idx, 1)
    assert (np.take_along_axis(idx, order, 1) == np.array(c["idx_sorted"])).all()
    np.testing.assert_allclose(np.take_along_axis(w, order, 1), c["wts_sorted"], atol=1e-6)


def test_oracle_permute_is_stable_expert_major(orc):
    rng = np.random.default_rng(0)
    idx = np.stack([rng.choice(16, 2, replace=False) for _ in range(100)]).astype(np.int32)
    total, counts, row_of = orc.permute(idx, 16, 128)
    assert counts.sum() == 200 and total == sum((c + 127) // 128 * 128 for c in counts)
    # rows are a bijection onto each expert's segment, ordered by (t, j)
    for e in range(16):
        t, j = np.nonzero(idx == e)
        rows = row_of[t, j]
        assert (np.diff(rows) == 1).all()


def test_det_expf_accuracy(orc):
    for v in np.linspace(-20, 20, 101, dtype=np.float32):
        assert abs(orc.expf(float(v)) - np.exp(np.float64(v))) <= 4e-7 * np.exp(np.float64(v))


def test_e4m3_encode_matches_torch(orc):
    """The oracle's integer e4m3 encoder (shared bit for bit with the device
    quantisers) equals torch's float8_e4m3fn cast inside +-448."""
    import torch
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * s
                        for s in (1e-3, 0.1, 1.0, 10.0, 100.0)])
    x = np.concatenate([x, np.float32([0.0, -0.0, 448.0, -448.0, 2 ** -9, 2 ** -10,
                                       3 * 2 ** -10, 1.5 * 2 ** -9, 2 ** -6, 0.9 * 2 ** -6])])
    x = x[np.abs(x) <= 448]
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert (orc.e4m3_encode(x) == ref).all()
    assert orc.e4m3_encode(np.float32([1e6, -1e6]))[0] == 0x7E  # saturates (no inf in e4m3fn)
