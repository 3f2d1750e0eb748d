"""RunReport accounting (a15): breakdown / compare_reports of libdwdp.so are
pinned bit for bit against the reference library's own implementation on the
reference simulator's event lists, then exercised on measured-style records."""
import numpy as np
import pytest

import paper_2604_01621_b200 as D
from paper_2604_01621_b200 import report as R

# small R1-like runs so the reference simulator finishes in well under a second
SIM = dict(layers=3, h=7168, E=64, k=8, f=2048, fs=2048, wb=2.0, peak=1382.3e12, mem_bw=6552.6e9,
           link_bw=900e9, iters=5, warmup=2, kind=0, length=8192.0, ratio=1.0, sd=0.2 * 8192,
           mnt=16384, bpr=2, seed=7)


def _sim(refl, slot, dwdp, N, **kw):
    a = dict(SIM, **kw)
    return refl.simulate_report(slot, dwdp, a["layers"], a["h"], a["E"], a["k"], a["f"], a["fs"],
                                a["wb"], a["peak"], a["mem_bw"], a["link_bw"], N, a["iters"],
                                a["warmup"], a["kind"], a["length"], a["ratio"], a["sd"], a["mnt"],
                                a["bpr"], a["seed"])


def _to_events(ref_ev):
    i32a, i64a, by = ref_ev
    ev = np.zeros(len(by), R.events_dtype())
    for j, n in enumerate(("rank", "stream", "category", "layer", "iteration", "detail")):
        ev[n] = i32a[:, j]
    ev["start_ns"], ev["end_ns"], ev["bytes"] = i64a[:, 0], i64a[:, 1], by
    return ev


def _pack(t: R.BreakdownTable) -> np.ndarray:
    c = t.c
    return np.array(list(c.compute_us) + list(c.copy_us) + list(c.compute_present) +
                    list(c.copy_present) + [c.iteration_latency_us, c.p2p_fully_overlapped,
                                            c.tokens_per_s], np.float64)


def _ours(rep):
    ranks, iters, warmup = rep["dims"]
    return R.breakdown_events(_to_events(rep["events"]), ranks, iters, warmup, rep["iter_start"],
                              rep["iter_end"], rep["iter_tokens"])


@pytest.mark.parametrize("N", [2, 4])
def test_breakdown_and_compare_bit_exact_vs_reference(ref, N):
    refl = ref
    dwdp = _sim(refl, 0, True, N, mnt=8192, bpr=1)  # 8K/rank: prefetch partly exposed
    dep = _sim(refl, 1, False, N, mnt=8192, bpr=1)
    a, b = _ours(dep), _ours(dwdp)
    pa, pb = _pack(a), _pack(b)
    assert (pa.view(np.uint64) == dep["breakdown"].view(np.uint64)).all()
    assert (pb.view(np.uint64) == dwdp["breakdown"].view(np.uint64)).all()
    assert a.to_csv() == dep["csv"] and b.to_csv() == dwdp["csv"]
    cmp_ = R.compare_reports(a, b)
    ref_out, ref_csv = refl.compare(dep["breakdown"], dwdp["breakdown"])
    ours = np.array([r["a_us"] for r in cmp_.rows] + [r["b_us"] for r in cmp_.rows] +
                    [r["delta_frac"] or 0.0 for r in cmp_.rows] +
                    [float(r["delta_frac"] is not None) for r in cmp_.rows] +
                    [cmp_.a_latency_us, cmp_.b_latency_us, cmp_.overall_frac,
                     cmp_.gross_sync_comm_pct])
    assert (ours.view(np.uint64) == ref_out.view(np.uint64)).all()
    assert cmp_.to_csv() == ref_csv
    assert "P2PCopy" in b.copy_us and "Communication" in a.compute_us


def test_overlap_on_one_stream_is_an_invariant_violation():
    ev = np.zeros(2, R.events_dtype())
    ev["start_ns"], ev["end_ns"] = [0, 50], [100, 150]
    with pytest.raises(D.InvariantViolation):
        R.breakdown_events(ev, 1, 1, 0, [0], [150], [10])


def _rec(g, tokens, t0, wait, kern, pf=None, dep=None):
    r = {k: 0.0 for k, _ in D._lib.LayerRecordC._fields_}
    r.update(global_layer=g, tokens=tokens, routed_rows=0, gate_wait_ns=wait, start_ns=t0,
             router_ns=kern[0], permute_ns=kern[1], gemm1_ns=kern[2], gemm2_ns=kern[3],
             combine_ns=kern[4], prefetch_start_ns=-1.0, prefetch_end_ns=-1.0)
    body = wait + sum(kern)
    if dep is not None:
        r.update(dispatch_ns=dep[0], comm_ns=dep[0] + dep[1])
        body += dep[0] + dep[1]
    if pf is not None:
        r.update(prefetch_start_ns=pf[0], prefetch_end_ns=pf[1], prefetch_bytes=1e9)
    r["end_ns"] = t0 + body
    return r


def test_report_from_records_dwdp_and_dep():
    L, kern = 2, (100.0, 50.0, 400.0, 200.0, 50.0)
    recs, t = [], 0.0
    for g in range(6):  # 3 iterations of 2 layers; layer 3 waits 300 ns on its weights
        wait = 300.0 if g == 3 else 0.0
        recs.append(_rec(g, 1000, t, wait, kern, pf=(t - 500, t + wait)))
        t = recs[-1]["end_ns"] + 10
    tab, ev = R.report_from_records([recs], L, 1, with_events=True)
    assert tab.compute_us["SyncWait"] == pytest.approx(0.15)  # 300 ns over 2 steady iterations
    assert tab.compute_us["GroupedGEMM"] == pytest.approx(1.2)  # 2 layers x 600 ns
    assert not tab.p2p_fully_overlapped and "P2PCopy" in tab.copy_us
    assert (ev["detail"][ev["category"] == 7] == 1).all()
    span = recs[5]["end_ns"] - recs[2]["start_ns"]
    assert tab.tokens_per_s == pytest.approx(2000 / (span / 1e9), rel=1e-9)
    deprecs, t = [], 0.0
    for g in range(6):
        deprecs.append(_rec(g % L, 1000, t, 0.0, kern, dep=(80.0, 120.0)))
        t = deprecs[-1]["end_ns"] + 10
    dtab = R.report_from_records([deprecs], L, 1)
    assert dtab.compute_us["Communication"] == pytest.approx(0.4)  # 2 layers x 200 ns
    cmp_ = R.compare_reports(dtab, tab)
    comm = [r for r in cmp_.rows if r["category"] == "Communication"][0]
    assert comm["delta_frac"] == pytest.approx(0.4 / dtab.iteration_latency_us)
    assert [r for r in cmp_.rows if r["category"] == "P2PCopy"][0]["delta_frac"] is None
    assert "GrossSyncComm" in cmp_.to_csv()
    with pytest.raises(D.ConfigError):
        R.report_from_records([recs[:5]], L, 1)  # partial iteration


def test_chrome_trace_layout():
    recs, t = [], 0.0
    for g in range(4):
        recs.append(_rec(g, 100, t, 50.0 if g == 2 else 0.0, (10.0, 5.0, 40.0, 20.0, 5.0),
                         pf=(t - 30, t + 1)))
        t = recs[-1]["end_ns"] + 10
    _, ev = R.report_from_records([recs], 2, 0, with_events=True)
    tr = R.chrome_trace(ev)
    assert len(tr) == len(ev)
    w = [x for x in tr if x["name"].startswith("SyncWait:weight_wait")]
    assert w and all(x["tid"] == 0 and x["ph"] == "X" for x in w)
    p = [x for x in tr if x["cat"] == "P2PCopy"]
    assert p and all(x["tid"] == 1 for x in p) and p[0]["args"]["bytes"] == 1e9
