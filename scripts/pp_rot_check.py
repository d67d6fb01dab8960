"""Debug: tiny-D128 naive/legolink links, copy vs shared on each attention kernel, against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

cfg = sg.TINY_D128
w = sg.cfg1(model=cfg)
eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=4096, max_requests=4, device=0)
ids = eng.generate_context_cache(w.chunks)
store = P.Store(M.Weights(cfg))
oids = store.compile(w.chunks)
segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
osegs = [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
for alg in ("naive", "legolink:4"):
    ref = P.link(store, osegs, alg)
    for k in (1, 2):
        B.set_attention_kernel(k)
        for share in (False, True):
            o = eng.link(segs, alg, kv_share=share)
            err = np.linalg.norm(o.logits - ref.logits) / np.linalg.norm(ref.logits)
            print(f"{alg} kernel{k} share={share} rel {err:.3e} first {o.first_token} ref {ref.first_token}")
B.set_attention_kernel(0)
eng.close()

# where do copy and shared diverge on the ping-pong kernel?  per-layer hidden states of the selected rows
eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=4096, max_requests=4, device=0)
ids = eng.generate_context_cache(w.chunks)
for segsw in [w.requests[0]] + sg.permuted_requests(w, 6):
    segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segsw]
    for alg in ("naive", "legolink:4"):
        B.set_attention_kernel(2)
        a = eng.link(segs, alg, kv_share=False, debug_hidden=True)
        b = eng.link(segs, alg, kv_share=True, debug_hidden=True)
        diff = [float(np.nanmax(np.abs(a.hidden[l] - b.hidden[l]))) for l in range(cfg.n_layers)]
        print(alg, "layer max|diff|", diff, "logits equal", bool(np.array_equal(a.logits, b.logits)))
B.set_attention_kernel(0)
eng.close()
