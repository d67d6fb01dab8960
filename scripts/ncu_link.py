"""One link step of a bench workload inside a cudaProfilerStart/Stop range, for
`ncu --profile-from-start off` captures of the LINK step only (not the compile forwards).

    python scripts/ncu_link.py [--config cfg4|cfg2|cfg3|cfg5] [--requests 32] [--layers L] [--graph 0|1]

cfg4 = one wave of 32 requests (the bench's pic_link_batch), shared-block link, as bench.py times it."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--requests", type=int, default=32)
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--alg", default=None)
ap.add_argument("--kv-share", type=int, default=3)
a = ap.parse_args()
w = {"cfg2": lambda: sg.cfg2(a.alg or "legolink:16", a.layers), "cfg3": lambda: sg.cfg3(a.alg or "legolink:32", a.layers),
     "cfg5": lambda: sg.cfg5(a.alg or "legolink:16", a.layers),
     "cfg4": lambda: sg.cfg4(n_requests=a.requests, alg=a.alg or "legolink:16", n_layers=a.layers)}[a.config]()
Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
eng = B.Engine(w.model, num_blocks=(sum(len(c) for c in w.chunks) + sum(Ns)) // 16 + 64 * len(Ns) + 64,
               max_rows=max(4096, sum(Ns) if (a.alg or "").startswith("cacheblend") else 8192),
               max_tokens=max(Ns) + 16, max_requests=len(Ns), device=0)
eng.kv_share = int(a.kv_share)
ids = eng.generate_context_cache(w.chunks)
reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
run = (lambda: eng.link_batch(reqs, w.alg, want_logits=False, use_graph=bool(a.graph))) if len(reqs) > 1 else \
      (lambda: eng.link(reqs[0], w.alg, use_graph=bool(a.graph)))
for _ in range(3):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("kernels per link step:", eng.stats()["kernels_last_call"])
eng.close()
