"""Tensor parallelism: two ranks share one B200 here (CUDA IPC works within a device;
on an 8-GPU box the same code reads peers over NVLink).  Each rank holds exact slices of the global
weights; the O/down partials are all-reduced by the residual kernel reading peer memory.  The ranks'
logits must be bit-identical and match the unsharded oracle (and a tp=1 engine)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import seedgen as sg

pytestmark = pytest.mark.gpu
CFG = sg.TINY_TP


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist
        from paper_2410_15332_b200 import dist as D
        from paper_2410_15332_b200 import pic as B
        dist.init_process_group("gloo")
        torch.cuda.set_device(0)
        eng = B.Engine(CFG, num_blocks=256, max_rows=512, max_tokens=1024, device=0, tp_rank=rank, tp_size=world)
        D.tp_connect(eng)
        w = sg.cfg1(model=CFG)
        ids = eng.generate_context_cache(w.chunks)
        segs = [("cached", i) for i in ids] + [("tokens", w.requests[0][-1].tokens)]
        out = {}
        for alg in ("legolink:4", "fr", "naive"):
            o = eng.link(segs, alg)
            g = eng.link(segs, alg, use_graph=True)      # graph replay path too
            out[alg] = (o.logits, g.logits, o.first_token)
            out["shared " + alg] = eng.link(segs, alg, kv_share=True).logits   # f3 shared-block link, sharded
        kq = eng.read_weights(0, 1, 0, 2 * 128)          # this rank's q-head rows of layer 1
        # decode over the linked cache (f1) and LegoLink-0 (f2) under tensor parallelism
        h = eng.link(segs, "legolink:4", keep_linked=True)
        out["decode"] = [eng.decode([h.linked], [t]).logits[0] for t in (5, 77, 300, 2)]
        eng.release(h.linked)
        ids0 = eng.generate_context_cache(w.chunks, dummy_prefix=4)
        segs0 = [("cached", i) for i in ids0] + [("tokens", w.requests[0][-1].tokens)]
        out["legolink0"] = eng.link(segs0, "legolink0").logits
        q.put((rank, out, kq))
        eng.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None))


def test_tp2_matches_oracle_and_tp1():
    from oracle import model as M
    from oracle import pic as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert isinstance(r[1], dict), r[1]
    Wt = M.Weights(CFG)
    w = sg.cfg1(model=CFG)
    store = P.Store(Wt)
    oids = store.compile(w.chunks)
    segs = [("cached", i) for i in oids] + [("tokens", w.requests[0][-1].tokens)]
    for alg in ("legolink:4", "fr", "naive"):
        l0, g0, t0 = res[0][1][alg]
        l1, g1, t1 = res[1][1][alg]
        assert np.array_equal(l0, l1) and t0 == t1                 # ranks agree bit for bit
        assert np.array_equal(l0, g0) and np.array_equal(l1, g1)   # graph == eager
        ref = P.link(store, segs, alg)
        err = np.linalg.norm(l0 - ref.logits) / np.linalg.norm(ref.logits)
        assert err < 2e-2, (alg, err)
        for r in range(2):                                          # shared-block link: bit-identical
            assert np.array_equal(res[r][1]["shared " + alg], res[r][1][alg][0]), (alg, r)
    # decode steps after a LegoLink-4 link (f1) and LegoLink-0 (f2), both sharded
    r4 = P.link(store, segs, "legolink:4")
    K, V = r4.K, r4.V
    for i, t in enumerate((5, 77, 300, 2)):
        lg, K, V = P.decode(Wt, K, V, t)
        a, b = res[0][1]["decode"][i], res[1][1]["decode"][i]
        assert np.array_equal(a, b)
        assert np.linalg.norm(a - lg) / np.linalg.norm(lg) < 2e-2, i
    store0 = P.Store(Wt)
    oids0 = store0.compile(w.chunks, dummy_prefix=4)
    ref0 = P.link(store0, [("cached", i) for i in oids0] + [("tokens", w.requests[0][-1].tokens)], "legolink0")
    assert np.array_equal(res[0][1]["legolink0"], res[1][1]["legolink0"])
    assert np.linalg.norm(res[0][1]["legolink0"] - ref0.logits) / np.linalg.norm(ref0.logits) < 2e-2
    # shard-exact weights: rank r's q rows are rows [r*256, (r+1)*256) of the global W_q
    for r in range(2):
        ref = sg.matrix(CFG.seed, sg.layer_tag(1, sg.TAG_Q), 4 * 128, 256, row0=r * 256, nrows=256)
        bits = (sg.bf16_rne(ref).view(np.uint32) >> 16).astype(np.uint16)
        assert np.array_equal(res[r][2], bits)
