"""f4 open-loop Poisson serving: the arrival generator (host, CPU) and the
scheduler on the GPU path."""
import math

import numpy as np
import pytest

import seedgen as sg
from paper_2410_15332_b200 import pic as B


def test_poisson_arrivals_statistics_and_determinism():
    lam, T, users = 400.0, 5.0, 8
    t, u = B.serve_arrivals(users, lam, T, 11)
    t2, u2 = B.serve_arrivals(users, lam, T, 11)
    t3, _ = B.serve_arrivals(users, lam, T, 12)
    assert np.array_equal(t, t2) and np.array_equal(u, u2)
    assert len(t3) != len(t) or not np.array_equal(t, t3)
    n = len(t)
    assert abs(n - lam * T) < 5 * math.sqrt(lam * T)                 # Poisson count
    assert np.all(np.diff(t) >= 0) and t[0] >= 0 and t[-1] < T
    per = np.bincount(u, minlength=users)
    assert np.all(np.abs(per - lam * T / users) < 5 * math.sqrt(lam * T / users))
    gaps = np.diff(t)
    assert abs(gaps.mean() * lam - 1) < 0.05                          # merged process: rate lam
    assert abs((gaps > 1 / lam).mean() - math.exp(-1)) < 0.03         # exponential inter-arrivals
    t0, _ = B.serve_arrivals(users, 0.0, T, 11)
    assert len(t0) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["legolink:4", "cacheblend:15"])
def test_serve_poisson_tiny(alg):
    cfg = sg.TINY_D128
    w = sg.cfg1(model=cfg)
    eng = B.Engine(cfg, num_blocks=1024, max_rows=1024, max_tokens=512, max_requests=8, device=0)
    ids = eng.generate_context_cache(w.chunks)
    reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r]
            for r in [w.requests[0]] + sg.permuted_requests(w, 3)]
    st = eng.serve_poisson(reqs, alg, rate=2000.0, duration_s=0.25, seed=3)
    t, _ = B.serve_arrivals(len(reqs), 2000.0, 0.25, 3)
    assert st["n_requests"] == len(t) and st["n_completed"] == len(t)
    assert 0 < st["ttft_p50_ms"] <= st["ttft_p90_ms"] <= st["ttft_p99_ms"] <= st["ttft_max_ms"]
    assert st["throughput_rps"] > 0 and 0 < st["ccr"] < 1
    if alg.startswith("cacheblend"):
        assert st["mean_batch"] == 1.0
    else:
        assert st["mean_batch"] > 1.0                                  # queued requests were batched
    assert eng.stats()["free_blocks"] == 1024 - sum((len(c) + 15) // 16 for c in w.chunks)
    eng.close()


@pytest.mark.gpu
def test_serve_poisson_shared_block_link_admits_more():
    """f3 x f4: with the shared-block link the server admits by fresh blocks, so a pool that fits only
    one copied link at a time batches several shared links; every request completes and the pool is
    whole again afterwards (shared references dropped)."""
    cfg = sg.TINY_D128
    w = sg.cfg1(model=cfg)
    n_chunk_blocks = sum((len(c) + 15) // 16 for c in w.chunks)
    link_blocks = (sum(len(c) for c in w.chunks) + len(w.requests[0][-1].tokens) + 15) // 16
    eng = B.Engine(cfg, num_blocks=n_chunk_blocks + link_blocks + 2, max_rows=1024, max_tokens=512,
                   max_requests=8, device=0)
    ids = eng.generate_context_cache(w.chunks)
    reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r]
            for r in [w.requests[0]] + sg.permuted_requests(w, 3)]
    out = {}
    for share in (False, True):
        st = eng.serve_poisson(reqs, "legolink:4", rate=2000.0, duration_s=0.25, seed=5, kv_share=share)
        assert st["n_completed"] == st["n_requests"] > 0
        assert eng.stats()["free_blocks"] == link_blocks + 2
        out[share] = st["mean_batch"]
    assert out[False] == 1.0 and out[True] > 1.0
    eng.close()
