"""Runtime contract of the prefetch engine and receive buffers (GPU).

The double-buffer protocol of simulate_dwdp (reference src/simcore.cpp:
640-733: plan(l+1) issued at MoeGate(l), buffer l%2 reused by l+2) made safe
for the public handle API (dwdp_prefetch_issue, dwdp_moe_forward,
dwdp_layer_forward): misuse that would compute on another layer's weights
fails loudly instead, per-layer state stays bounded in a serving loop, and
one host thread per GPU can drive contexts concurrently.
"""
import threading

import pytest
import torch

import paper_2604_01621_b200 as D

pytestmark = pytest.mark.gpu

MID = dict(num_layers=3, num_experts=64, hidden=1024, ffn=256, shared_ffn=256, top_k=6,
           n_group=8, topk_group=4, max_tokens=512, weight_layers=3)


def _x(T, h, seed):
    x = torch.empty((T, h), dtype=torch.bfloat16, device="cuda:0")
    D.fill_bf16(x, seed, 1.0)
    return x


def _group(n=2, **kw):
    ranks = [D.DwdpContext(D.DwdpConfig(**dict(MID, **kw), rank=r, group_size=n)) for r in range(n)]
    for c in ranks:
        c.init_weights()
    D.DwdpContext.link_local(ranks)
    return ranks


def test_prefetch_cannot_overwrite_an_unread_buffer():
    ranks = _group()
    try:
        r = ranks[0]
        r.prefetch_issue(0)
        r.prefetch_issue(1)
        with pytest.raises(D.ConfigError, match="still holds global layer 0"):
            r.prefetch_issue(2)  # buffer 0 holds layer 0, whose MoE never ran
    finally:
        for c in ranks:
            c.close()


def test_prefetch_order_and_double_issue():
    ranks = _group()
    try:
        r = ranks[0]
        r.prefetch_issue(3)
        with pytest.raises(D.InvariantViolation):
            r.prefetch_issue(3)  # simcore.cpp:624
        with pytest.raises(D.ConfigError, match="increasing order"):
            r.prefetch_issue(1)
    finally:
        for c in ranks:
            c.close()


def test_layer_forward_rewind_is_refused():
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = _group()
    try:
        x = _x(96, MID["hidden"], 5)
        for g in range(4):
            y = ranks[0].layer_forward(g, x, residual=False)
            assert torch.equal(y, full.moe_forward(g % 3, x))
        with pytest.raises(D.ConfigError, match="behind the prefetch cursor|no longer holds"):
            ranks[0].layer_forward(1, x, residual=False)
        with pytest.raises(D.ConfigError, match="no longer holds"):
            ranks[0].layer_forward(2, x, residual=False)  # buffer 0 now holds layer 4
        y = ranks[0].layer_forward(3, x, residual=False)  # the resident layer replays fine
        assert torch.equal(y, full.moe_forward(0, x))
    finally:
        for c in ranks + [full]:
            c.close()


def test_stack_iteration_may_skip_a_prefetched_layer():
    """layer_forward(0..4) prefetches layer 5; stack_forward then starts the
    next iteration at global layer 6, abandoning 5: its buffer is reusable and
    every layer stays exact."""
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = _group()
    try:
        x = _x(64, MID["hidden"], 21)
        for g in range(5):
            ranks[0].layer_forward(g, x, residual=False)
        y = ranks[0].stack_forward(x)
        yf = full.stack_forward(x)  # all-local stack: layers 0, 1, 2 with residual
        torch.cuda.synchronize()
        assert torch.equal(y, yf)
        recs = ranks[0].records()
        assert [r["global_layer"] for r in recs][-3:] == [6, 7, 8]
        assert torch.isfinite(y.float()).all()
        with pytest.raises(D.ConfigError):
            ranks[0].layer_forward(5, x, residual=False)  # abandoned and refilled by layer 7
    finally:
        for c in ranks + [full]:
            c.close()


def test_moe_forward_needs_resident_experts_and_records_its_read():
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = _group()
    try:
        x = _x(80, MID["hidden"], 9)
        with pytest.raises(D.ConfigError, match="not resident"):
            ranks[0].moe_forward(0, x)
        h = ranks[0].prefetch_issue(0)
        y = ranks[0].moe_forward(0, x)  # waits for plan 0 on the stream
        assert torch.equal(y, full.moe_forward(0, x))
        ranks[0].prefetch_issue(1)
        ranks[0].prefetch_issue(2)  # legal now: layer 0's buffer was read
        torch.cuda.synchronize()
        assert ranks[0].prefetch_query(h)
        with pytest.raises(D.ConfigError, match="not resident"):
            ranks[0].moe_forward(0, x)  # buffer 0 now holds layer 2
        assert torch.equal(ranks[0].moe_forward(2, x), full.moe_forward(2, x))
        assert torch.equal(ranks[0].moe_forward(1, x), full.moe_forward(1, x))
    finally:
        for c in ranks + [full]:
            c.close()


def test_state_stays_bounded_in_a_long_undrained_loop():
    """2,100 layers without draining records: the oldest records and their
    plans are recycled (kMaxRecords = 2048), old handles retire, outputs stay
    exact and the newest records carry the right routed rows."""
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    ranks = _group(kernel_timing=1)
    try:
        x = _x(64, MID["hidden"], 11)
        ref = [full.moe_forward(l, x) for l in range(3)]
        h0 = None
        for g in range(2100):
            y = ranks[0].layer_forward(g, x, residual=False)
            if g == 0:
                torch.cuda.synchronize()
                h0 = 0
            if g % 700 == 0 or g == 2099:
                torch.cuda.synchronize()
                assert torch.equal(y, ref[g % 3]), g
        torch.cuda.synchronize()
        with pytest.raises(D.ConfigError, match="retired"):
            ranks[0].prefetch_times(h0)
        assert ranks[0].prefetch_query(h0)  # retired plans report done
        recs = ranks[0].records()
        assert len(recs) == 2048
        assert recs[-1]["global_layer"] == 2099
        _, _, _, _, rows = full.route(2099 % 3, x)
        assert recs[-1]["routed_rows"] == rows
        assert all(r["prefetch_bytes"] > 0 for r in recs)
    finally:
        for c in ranks + [full]:
            c.close()


def test_two_host_threads_drive_two_groups_concurrently():
    """One host thread per group (the one-thread-per-GPU deployment, here two
    groups on one GPU): the pull engine's launch path is thread-safe and
    every layer stays bit-identical to the all-local model."""
    full = D.DwdpContext(D.DwdpConfig(**MID))
    full.init_weights()
    groups = [_group(engine=D.ENGINE_PULL), _group(engine=D.ENGINE_PULL)]
    xs = [_x(128 + 64 * i, MID["hidden"], 40 + i) for i in range(2)]
    refs = [[full.moe_forward(l, xs[i]) for l in range(3)] for i in range(2)]
    torch.cuda.synchronize()
    errors = []

    def drive(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for g in range(30):
                    for r in range(2):
                        y = groups[i][r].layer_forward(g, xs[i], residual=False, stream=st)
                        st.synchronize()
                        if not torch.equal(y, refs[i][g % 3]):
                            errors.append((i, g, r))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=drive, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    try:
        assert not errors, errors[:5]
    finally:
        for c in groups[0] + groups[1] + [full]:
            c.close()


def test_open_peers_rejects_mismatched_geometry():
    a = D.DwdpContext(D.DwdpConfig(**MID, rank=0, group_size=2))
    b = D.DwdpContext(D.DwdpConfig(**dict(MID, num_layers=2, weight_layers=2), rank=1, group_size=2))
    try:
        with pytest.raises(D.ConfigError, match="geometry"):
            a.open_peers(a.export_ipc() + b.export_ipc())
    finally:
        a.close()
        b.close()
