"""World-size-2 gloo tests of the data-parallel host logic (CPU): request sharding, barrier +
max-over-ranks timing, and per-rank host-only planners agreeing with the oracle planner on their
shard (the GPU path shards the same way under torchrun + NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import seedgen as sg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from oracle import model as M
    from oracle import pic as P
    from paper_2410_15332_b200 import dist as D
    from paper_2410_15332_b200 import pic as B
    try:
        r, w, _ = D.env_rank()
        D.init("gloo")
        wl = sg.cfg4(n_requests=8, corpus=12, per_req=3, chunk_len=32, query_len=8, n_layers=1)
        mine = D.shard(list(range(len(wl.requests))), r, w)
        # per-rank host-only engine with the rank's own compiled corpus, plans checked vs the oracle
        eng = B.Engine(wl.model, num_blocks=512, max_rows=512, max_tokens=1024, max_requests=8, device=None)
        ids = eng.generate_context_cache(wl.chunks)
        st = P.Store(M.Weights(wl.model))
        oids = st.compile(wl.chunks, compiled_override=[(None, None)] * len(wl.chunks))
        ok = True
        for i in mine:
            segs = wl.requests[i]
            pe = eng.plan([("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs], wl.alg)
            po = P.plan(st, [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs], wl.alg)
            ok &= bool(np.array_equal(pe["sel"], po.sel))
        D.barrier()
        mx = D.max_over_ranks(10.0 * (r + 1))
        tot = D.sum_over_ranks(len(mine))
        q.put((r, mine, ok, mx, tot))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), False, 0, 0))


def test_dp_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(r[2] for r in res), res
    shards = [set(r[1]) for r in res]
    assert shards[0].isdisjoint(shards[1]) and shards[0] | shards[1] == set(range(8))
    assert all(r[3] == 20.0 for r in res)          # max over ranks
    assert all(r[4] == 8 for r in res)             # every request handled exactly once


def test_shard_properties():
    from paper_2410_15332_b200 import dist as D
    items = list(range(13))
    for world in (1, 2, 3, 8):
        parts = [D.shard(items, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == items
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        D.shard(items, 2, 2)
