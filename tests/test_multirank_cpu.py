"""N > 1 host logic on CPU: world_size-2 (and 4) gloo process groups, one
process per simulated rank, exchanging what the GPU ranks exchange at setup
(placement tables, copy plans, workload batches). No GPU needed."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2604_01621_b200 as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, f, h = 256, 2048, 7168
        plan = D.build_placement(E, world)
        # every rank must derive the identical table
        tables = [None] * world
        dist.all_gather_object(tables, (plan.local_sets, plan.fetch_lists))
        assert all(t == tables[0] for t in tables)
        # this rank's prefetch plan in the runtime's layout: per (tensor, peer)
        # one shard of the peer's whole owned block (prefetch_transfers,
        # simcore.cpp:486-515), 1 MiB TDM slices
        slot = h * f * 2
        per_peer = {}
        for e, src in plan.fetch_lists[rank]:
            per_peer[src] = per_peer.get(src, 0) + 1
        shards = [D.ShardRef(p, t, n * slot, 0) for t in range(3) for p, n in sorted(per_peer.items())]
        cp = D.build_copy_plan(shards, 1 << 20, rank)
        plans = [None] * world
        dist.all_gather_object(plans, cp)
        # source view: every source serves each destination exactly its block
        for src in range(world):
            qs = D.source_queues(plans, src)
            for dst, sl in qs.items():
                want = 0 if dst == src else 3 * (E // world) * slot
                assert sum(s.length for s in sl) == want
        # TDM rotation staggers the first peer of every destination
        firsts = [p.slices[0].src_rank for p in plans]
        assert len(set(firsts)) == world
        # the workload generator is rank-consistent (each rank can sample all)
        spec = D.WorkloadSpec(D.IslDist.from_cv(8192, 0.2), 32768, 4, 0.0, 7)
        b = D.sample_batches(spec, D.r1_model(), world, 3, with_routing=False)
        bs = [None] * world
        dist.all_gather_object(bs, [x.tokens for x in b])
        assert all(x == bs[0] for x in bs)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_setup_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
