"""Tensor parallelism: TP = 2, 4 and 8 ranks share one B200 here (CUDA IPC works within
a device; on an 8-GPU box the same code reads peers over NVLink).  Each rank holds exact slices of the
global weights; the O/down partials are all-reduced by the residual kernel reading peer memory.  The
ranks' logits must be bit-identical and match the unsharded oracle.  TP = 8 is also run at the cfg5
shape (Llama-3-70B: one kv-head and 8 q-heads per rank) at truncated depth against the oracle on
sampled rows."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import seedgen as sg

pytestmark = pytest.mark.gpu
CFGS = {2: sg.TINY_TP, 4: sg.TINY_TP8, 8: sg.TINY_TP8}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, cfg_name):
    CFG = sg.MODELS[cfg_name]
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
        kq = eng.read_weights(0, 1, 0, CFG.n_heads // world * 128)   # this rank's q-head rows of layer 1
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


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=1200) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tp_matches_oracle(world):
    from oracle import model as M
    from oracle import pic as P
    CFG = CFGS[world]
    res = _spawn(_rank, world, CFG.name)
    for r in res:
        assert isinstance(r[1], dict), r[1]
    Wt = M.Weights(CFG)
    w = sg.cfg1(model=CFG)
    store = P.Store(Wt)
    oids = store.compile(w.chunks)
    segs = [("cached", i) for i in oids] + [("tokens", w.requests[0][-1].tokens)]
    for alg in ("legolink:4", "fr", "naive"):
        l0, g0, t0 = res[0][1][alg]
        for r in range(world):
            lr, gr, tr = res[r][1][alg]
            assert np.array_equal(l0, lr) and t0 == tr              # ranks agree bit for bit
            assert np.array_equal(lr, gr)                           # graph == eager
        ref = P.link(store, segs, alg)
        err = np.linalg.norm(l0 - ref.logits) / np.linalg.norm(ref.logits)
        assert err < 2e-2, (alg, err)
        for r in range(world):                                      # shared-block link: bit-identical
            assert np.array_equal(res[r][1]["shared " + alg], res[r][1][alg][0]), (alg, r)
    # decode steps after a LegoLink-4 link (f1) and LegoLink-0 (f2), both sharded
    r4 = P.link(store, segs, "legolink:4")
    K, V = r4.K, r4.V
    for i, t in enumerate((5, 77, 300, 2)):
        lg, K, V = P.decode(Wt, K, V, t)
        a = res[0][1]["decode"][i]
        assert all(np.array_equal(a, res[r][1]["decode"][i]) for r in range(world))
        assert np.linalg.norm(a - lg) / np.linalg.norm(lg) < 2e-2, i
    store0 = P.Store(Wt)
    oids0 = store0.compile(w.chunks, dummy_prefix=4)
    ref0 = P.link(store0, [("cached", i) for i in oids0] + [("tokens", w.requests[0][-1].tokens)], "legolink0")
    assert all(np.array_equal(res[0][1]["legolink0"], res[r][1]["legolink0"]) for r in range(world))
    assert np.linalg.norm(res[0][1]["legolink0"] - ref0.logits) / np.linalg.norm(ref0.logits) < 2e-2
    # shard-exact weights: rank r's q rows are rows [r*256, (r+1)*256) of the global W_q
    rows = CFG.n_heads // world * 128
    for r in range(world):
        ref = sg.matrix(CFG.seed, sg.layer_tag(1, sg.TAG_Q), CFG.n_heads * 128, CFG.d_model, row0=r * rows, nrows=rows)
        bits = (sg.bf16_rne(ref).view(np.uint32) >> 16).astype(np.uint16)
        assert np.array_equal(res[r][2], bits)


def _rank_cfg5(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist
        from paper_2410_15332_b200 import dist as D
        from paper_2410_15332_b200 import pic as B
        dist.init_process_group("gloo")
        torch.cuda.set_device(0)
        w = sg.cfg5(n_layers=2)
        N = sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])
        eng = B.Engine(w.model, num_blocks=(sum(len(c) for c in w.chunks) + 2 * N) // 16 + 64, max_rows=2048,
                       max_tokens=N + 16, device=0, tp_rank=rank, tp_size=world)
        D.tp_connect(eng)
        eng.kv_share = True                                    # the bench's configuration
        ids = eng.generate_context_cache(w.chunks)
        segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
        g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)
        d = eng.link(segs, w.alg, keep_linked=True, use_graph=False, debug_hidden=True, want_selected=True)
        out = {"logits": g.logits, "logits_eager": d.logits, "sel": g.selected,
               "kv": [eng.linked_export(g.linked, l) for l in range(2)]}
        if rank == 0:
            sub = np.unique(np.r_[np.arange(0, len(g.selected), 16), len(g.selected) - 1])
            out["sub"] = sub
            out["hidden"] = d.hidden[:, sub].copy()
            out["tok"] = eng.plan(segs, w.alg)["tok"]
        eng.release(g.linked)
        eng.release(d.linked)
        q.put((rank, out))
        eng.close()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


def test_tp8_cfg5_truncated_depth_vs_oracle():
    """cfg5 (Llama-3-70B shape, N = 32832, LegoLink-16, shared-block link) at L = 2 under TP = 8 on one
    GPU: every rank owns one kv-head and 8 q-heads.  Ranks agree bit for bit; the oracle recomputes both
    layers on sampled rows from the GPU's layer input and the union of the ranks' linked K/V slices."""
    from oracle import model as M
    res = _spawn(_rank_cfg5, 8)
    for r in res:
        assert isinstance(r[1], dict), r[1]
    o0 = res[0][1]
    for _, o in res:
        assert np.array_equal(o["logits"], o0["logits"]) and np.array_equal(o["logits"], o["logits_eager"])
        assert np.array_equal(o["sel"], o0["sel"])
    w = sg.cfg5(n_layers=2)
    cfg = w.model
    sel, sub, hid = o0["sel"], o0["sub"], o0["hidden"]
    assert len(sel) == 1072
    Wt = M.Weights(cfg, cache_layers=1)

    def f64(bits):
        return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)

    def rel(a, b):
        return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))

    for l in range(2):
        K = np.concatenate([f64(o["kv"][l][0]) for _, o in res], axis=1)     # [N][8 kv-heads][D], rank order
        V = np.concatenate([f64(o["kv"][l][1]) for _, o in res], axis=1)
        K0 = K.copy()
        h_in = Wt.embed_rows(o0["tok"][sel[sub]]) if l == 0 else hid[l - 1].astype(np.float64)
        h_out = M.layer_rows(Wt.layer(l), cfg, h_in, sel[sub], sel[sub], K, V)
        assert rel(hid[l], h_out) < 5e-3, (l, rel(hid[l], h_out))
        assert rel(K0[sel[sub]], K[sel[sub]]) < 5e-3, l
    logits = M.logits_of(Wt, hid[1, -1].astype(np.float64))
    assert rel(o0["logits"], logits) < 5e-3
