"""Decode TPOT A/B on one engine: copy-path links vs shared-block links vs shared + materialized links
(cfg4 batch of 32 requests, or cfg2 with one), CUDA events, interleaved repetitions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

w = sg.cfg4(n_requests=32) if (len(sys.argv) > 1 and sys.argv[1] == "cfg4") else sg.cfg2()
m = w.model
Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
stream = torch.cuda.Stream(0)
with torch.cuda.stream(stream):
    eng = B.Engine(m, num_blocks=(sum(len(c) for c in w.chunks) + 4 * sum(Ns)) // 16 + 4096, max_rows=8192,
                   max_tokens=max(Ns) + 256, max_requests=len(w.requests), device=0, stream=stream)
    ids = eng.generate_context_cache(w.chunks)
    reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
    sets = {}
    for name, share in (("copy", False), ("shared", True), ("materialized", True)):
        outs = eng.link_batch(reqs, w.alg, keep_linked=True, kv_share=share, want_logits=False)
        hs = [o.linked for o in outs]
        if name == "materialized":
            for h in hs:
                eng.materialize(h)
        sets[name] = hs
    toks = [7] * len(reqs)
    dl = torch.empty((len(reqs), m.vocab), dtype=torch.float32, device="cuda:0")
    for name, hs in sets.items():
        for _ in range(3):
            eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr())
    res = {k: [] for k in sets}
    for rep in range(3):
        for name, hs in sets.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr())
            e1.record(stream)
            e1.synchronize()
            res[name].append(e0.elapsed_time(e1) / 10)
    for k, v in res.items():
        print(k, " ".join(f"{x:.3f}" for x in v), "ms/step", flush=True)
