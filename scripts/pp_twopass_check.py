import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import seedgen as sg
from paper_2410_15332_b200 import pic as B
cfg = sg.TINY_D128
w = sg.cfg1(model=cfg)
eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=4096, max_requests=4, device=0)
ids = eng.generate_context_cache(w.chunks)
B.set_attention_kernel(2)
out = {}
for i, segsw in enumerate([w.requests[0]] + sg.permuted_requests(w, 6)):
    segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segsw]
    for alg in ("naive", "legolink:4"):
        out[f"{i}_{alg}"] = eng.link(segs, alg, kv_share=False).logits
np.savez(sys.argv[1], **out)
