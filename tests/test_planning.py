"""Product host planners (libdwdp.so through the C-ABI) against the reference:
golden outputs of the compiled reference library plus the reference's own
unit-test KATs (tests/test_placement.cpp, test_copyplan.cpp, test_workload.cpp,
test_modelspec.cpp under /root/reference/proj), restated."""
import numpy as np
import pytest

import paper_2604_01621_b200 as D
from conftest import load_golden


def test_placement_matches_reference_golden():
    for c in load_golden("ref_placement.json"):
        if c["status"]:
            with pytest.raises(D.ConfigError):
                D.build_placement(c["E"], c["N"], c["extra"])
            continue
        p = D.build_placement(c["E"], c["N"], c["extra"])
        assert (p.local_count, p.redundancy) == (c["local_count"], c["redundancy"])
        assert p.local_sets == c["local_sets"]
        assert [[list(x) for x in f] for f in p.fetch_lists] == (c["fetch"] or [[] for _ in p.local_sets])


def test_placement_kats():
    # test_placement.cpp:14-28 exact division
    p = D.build_placement(256, 4, 0)
    assert p.local_count == 64 and p.redundancy == 0
    for r in range(4):
        per = {}
        for e, s in p.fetch_lists[r]:
            per[s] = per.get(s, 0) + 1
        assert sorted(per.values()) == [64, 64, 64]
    # :30-39 non-divisible
    p = D.build_placement(256, 3, 0)
    assert (p.local_count, p.redundancy) == (86, 2)
    # :41-49 redundancy E4 N2 extra1
    p = D.build_placement(4, 2, 1)
    assert p.local_count == 3 and p.redundancy == 2
    assert all(len(f) == 1 and f[0][1] == 1 - r for r, f in enumerate(p.fetch_lists))
    # :51-65 greedy balance
    p = D.build_placement(6, 3, 1)
    for f in p.fetch_lists:
        per = {}
        for _, s in f:
            per[s] = per.get(s, 0) + 1
        assert max(per.values()) - min(per.values()) <= 1
    # :67-71 determinism
    assert D.build_placement(97, 5, 2) == D.build_placement(97, 5, 2)
    # :106-112 invalid arguments
    for args in [(8, 1, 0), (3, 4, 0), (8, 2, -1)]:
        with pytest.raises(D.ConfigError):
            D.build_placement(*args)


def test_prefetch_bytes_and_full_replication():
    m = D.MoeModelSpec(1, 8, 256, 1, 2, 0, 1.0, 2.0)
    assert D.expert_shard_bytes(m) == 48
    assert D.prefetch_bytes(D.build_placement(256, 4, 0), m) == 192 * 48
    full = D.build_placement(256, 4, 256)
    assert full.local_count == 256 and D.prefetch_bytes(full, m) == 0
    assert all(not f for f in full.fetch_lists)
    assert D.prefetch_bytes(D.build_placement(256, 3, 0), m) == 170 * 48
    prev = 1e300
    m2 = D.MoeModelSpec(1, 64, 61, 1, 16, 0, 0.5, 2.0)
    for extra in range(0, 70, 7):
        b = D.prefetch_bytes(D.build_placement(61, 4, extra), m2)
        assert b <= prev
        prev = b


def test_assign_fetch_sources_and_describe():
    p = D.build_placement(97, 5, 2)
    assert D.assign_fetch_sources(97, p.local_sets) == p.fetch_lists
    text = D.describe_placement(D.build_placement(16, 4, 1))
    for r in range(4):
        assert f"rank {r}" in text
    p.validate()


def test_copy_plan_matches_reference_golden():
    for c in load_golden("ref_copyplan.json"):
        shards = [D.ShardRef(*s) for s in c["shards"]]
        if c["status"]:
            with pytest.raises(D.ConfigError):
                D.build_copy_plan(shards, c["slice"], c["dst"])
            continue
        plan = D.build_copy_plan(shards, c["slice"], c["dst"])
        got = [[s.param_id, s.src_rank, s.src_offset, s.dst_offset, s.length] for s in plan.slices]
        if "slices" in c:
            assert got == c["slices"]
        else:
            arr = np.array(got, np.int64)
            assert len(got) == c["n_slices"] and got[:64] == c["head"]
            assert int((arr * (np.arange(len(arr))[:, None] + 1) % 1000003).sum()) == c["checksum"]


def test_copy_plan_kats():
    plan = D.build_copy_plan([D.ShardRef(1, 0, 5, 0), D.ShardRef(2, 0, 5, 0)], 2, 0)
    assert [(s.src_rank, s.dst_offset, s.length) for s in plan.slices] == [
        (1, 0, 2), (2, 0, 2), (1, 2, 2), (2, 2, 2), (1, 4, 1), (2, 4, 1)]
    plan = D.build_copy_plan([D.ShardRef(1, 7, 5, 100)], 2, 0)
    assert [s.length for s in plan.slices] == [2, 2, 1]
    assert plan.slices[0].src_offset == 100 and plan.slices[2].src_offset == 104
    sh = [D.ShardRef(p, 0, 4, 0) for p in (1, 2, 3)]
    assert [D.build_copy_plan(sh, 2, d).slices[0].src_rank for d in (9, 10, 11)] == [1, 2, 3]
    q = D.source_queues([plan], 1)
    assert list(q) == [0] and [s.dst_offset for s in q[0]] == [0, 2, 4]
    a = D.build_copy_plan([D.ShardRef(9, 0, 4, 0)], 2, 0)
    b = D.build_copy_plan([D.ShardRef(9, 0, 4, 0)], 2, 1)
    m = D.source_queues([a, b], 9)
    assert len(m[0]) == 2 and len(m[1]) == 2
    assert D.source_queues([], 3) == {}
    csv = D.build_copy_plan([D.ShardRef(1, 3, 5, 10)], 2, 0).to_csv()
    assert csv.startswith("param_id,src_rank,src_offset,dst_offset,length") and "3,1,10,0,2" in csv


def test_copy_plan_byte_reconstruction():
    """test_copyplan.cpp:178-219: slices applied in any order rebuild the shards."""
    rng = np.random.default_rng(1234)
    for _ in range(50):
        peers = int(rng.integers(1, 5))
        shards, src = [], {}
        for p in range(peers):
            size, base = int(rng.integers(1, 2000)), int(rng.integers(0, 64))
            shards.append(D.ShardRef(p, 0, size, base))
            src[p] = rng.integers(0, 256, base + size).astype(np.uint8)
        plan = D.build_copy_plan(shards, int(rng.integers(1, 300)), peers)
        dst = {s.peer: np.full(s.size, 0xEE, np.uint8) for s in shards}
        for i in rng.permutation(len(plan.slices)):
            s = plan.slices[i]
            dst[s.src_rank][s.dst_offset:s.dst_offset + s.length] = \
                src[s.src_rank][s.src_offset:s.src_offset + s.length]
        for s in shards:
            assert (dst[s.peer] == src[s.peer][s.src_offset:s.src_offset + s.size]).all()


def test_workload_matches_reference_golden():
    g = load_golden("ref_workload.json")
    for c in g["route"]:
        m = D.MoeModelSpec(1, 8, c["E"], c["k"], 8)
        assert D.route_tokens(c["tokens"], m, c["skew"], c["seed"]) == c["counts"]
    for c in g["batches"]:
        kind, length, ratio, sd, mnt, bpr, skew, seed = c["spec"]
        spec = D.WorkloadSpec(D.IslDist(int(kind), length, ratio, sd), mnt, bpr, skew, seed)
        bs = D.sample_batches(spec, D.r1_model(), c["N"], c["iters"], with_routing=skew > 0)
        assert [b.tokens for b in bs] == c["tokens"]
        assert [b.requests for b in bs] == c["requests"]
        if "routed_rank0_iter0" in c:
            assert bs[0].routed[0] == c["routed_rank0_iter0"]


def test_workload_kats():
    b = D.RankBatch([80, 120], [1, 1], [])
    assert abs(D.imbalance_cv(b) - 0.2) < 1e-12
    with pytest.raises(D.ConfigError):
        D.imbalance_cv(D.RankBatch([7], [1], []))
    with pytest.raises(D.ConfigError):
        D.imbalance_cv(D.RankBatch([0, 0], [1, 1], []))
    r = 0.5
    assert abs(D.IslDist.uniform_ratio(8192, r).cv() - (1 - r) / ((1 + r) * np.sqrt(3))) < 1e-12
    assert abs(D.IslDist.from_cv(10000, 0.2).cv() - 0.2) < 1e-12
    with pytest.raises(D.ConfigError):  # MNT below request size
        D.sample_batches(D.WorkloadSpec(D.IslDist.fixed(2000), 1000), D.r1_model(), 2, 1)
    spec = D.WorkloadSpec(D.IslDist.fixed(600), 1000, 2)
    for b in D.sample_batches(spec, D.r1_model(), 2, 4):
        assert b.tokens == [600, 600] and b.requests == [1, 1]
    m = D.MoeModelSpec(1, 64, 256, 8, 16)
    c = D.route_tokens(2000, m, 10.0, 5)
    assert sum(c) == 16000 and c[0] / 16000 >= 0.9


def test_costs_match_reference_golden():
    g = load_golden("ref_costs.json")
    for h, f, wb, b in g["shard_bytes"]:
        assert D.expert_shard_bytes(D.MoeModelSpec(1, h, 1, 1, f, 0, wb)) == b
    for c in g["moe_entries"]:
        T = c["T"]
        e = D.moe_entries(D.r1_model(), T, T * 8, 256)
        assert [e[0].flops, e[0].bytes, e[1].flops, e[1].bytes] == c["out"]
    for c in g["analytic"]:
        r = D.analytic_compare(D.r1_model(), D.GpuSpec(), D.build_placement(256, c["N"]), c["T"])
        # the reference adds a ~0 attention term (calib 1e-12) and 1 ns floors
        for k in ("t_compute_s", "t_prefetch_s", "t_all2all_s", "dep_dwdp_speedup"):
            assert abs(r[k] - c[k]) <= 1e-9 * max(1.0, abs(c[k])) + 1e-12, k
    assert D.roofline_time(1e12, 0, D.GpuSpec(1e12, 1e12, 1e9)) == 1.0
    with pytest.raises(D.ConfigError):
        D.roofline_time(0, 0, D.GpuSpec())


def test_batches_csv_round_trip_and_errors():
    """workload.hpp:77-79: exact workload replay through the reference's CSV
    format (src/workload.cpp:191-247)."""
    spec = D.WorkloadSpec(D.IslDist.uniform_ratio(1000, 0.5), 4000, 3, 1.0, 7)
    model = D.MoeModelSpec(1, 64, 256, 8, 16, 0, 1.0, 2.0, attn_proj_params=100)
    b = D.sample_batches(spec, model, 3, 5)
    csv = D.batches_to_csv(b)
    assert csv.startswith("iteration,rank,tokens,requests,expert_counts\n")
    back = D.batches_from_csv(csv)
    assert [x.tokens for x in back] == [x.tokens for x in b]
    assert [x.requests for x in back] == [x.requests for x in b]
    assert [x.routed for x in back] == [x.routed for x in b]
    assert D.batches_to_csv(back) == csv
    nr = D.sample_batches(spec, model, 2, 2, with_routing=False)
    assert D.batches_from_csv(D.batches_to_csv(nr))[1].tokens == nr[1].tokens
    for bad in ("bogus", "", "iteration,rank,tokens,requests,expert_counts\n0,0,x,1,\n"):
        with pytest.raises(D.ConfigError):
            D.batches_from_csv(bad)
    with pytest.raises(D.ConfigError):
        D.WorkloadSpec(D.IslDist.fixed(2000), 1000).validate()


def test_layer_costs_and_model_validate():
    """modelspec.cpp:6-98: attention + MoE entries, calibration scalars."""
    m = D.r1_model(1)
    m.validate()
    w = D.layer_costs(m, 4096, 2048)
    assert [op.category for op in w.attn] == ["Attention"]
    assert [op.category for op in w.moe] == ["GroupedGEMM", "DenseGEMM"]
    assert w.moe[0].flops == pytest.approx(2.0 * 4096 * 8 * 3 * 7168 * 2048)
    m2 = D.r1_model(1)
    m2.calib = D.CostCalibration(grouped_gemm=0.5)
    assert D.layer_costs(m2, 4096, 2048).moe[0].flops == pytest.approx(0.5 * w.moe[0].flops)
    with pytest.raises(D.ConfigError):
        D.MoeModelSpec(1, 8, 4, 2, 4).validate()  # attn_proj_params must be > 0
    with pytest.raises(D.ConfigError):
        D.layer_costs(m, 0, 1)
