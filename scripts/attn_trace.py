"""Per-CTA attention timeline of the last layer of one link (PIC_ATTN_TRACE=1 must be set).
    python scripts/attn_trace.py [cfg2|cfg3|cfg5] [n_layers] [alg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen as sg
from paper_2410_15332_b200 import pic as B

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
kw = {"n_layers": int(sys.argv[2])} if len(sys.argv) > 2 and name != "cfg2" else {}
if len(sys.argv) > 3:
    kw["alg"] = sys.argv[3]
w = getattr(sg, name)(**kw)
N = sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])
eng = B.Engine(w.model, num_blocks=(sum(len(c) for c in w.chunks) + 3 * N) // 16 + 64, max_rows=max(4096, N),
               max_tokens=N + 16, device=0)
eng.kv_share = bool(int(os.environ.get("KV_SHARE", "1")))
ids = eng.generate_context_cache(w.chunks)
segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
for i in range(3):
    print(f"--- link {i} (graph)", file=sys.stderr, flush=True)
    eng.link(segs, w.alg)
print("--- eager", file=sys.stderr, flush=True)
eng.link(segs, w.alg, use_graph=False)
