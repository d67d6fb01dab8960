"""compute-sanitizer target (memcheck / racecheck / synccheck): the tiny-D128 link through every kernel
family — copy path and shared-block link (K-tile re-base warps), CacheBlend selection, a batched link,
LegoLink-0 compile, decode over the linked cache, materialize, and (PIC_PAIR=1) the CTA-pair GEMM.
Eager launches so every kernel is checked individually, then one graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

cfg = sg.TINY_D128
w = sg.cfg1(model=cfg)
eng = B.Engine(cfg, num_blocks=256, max_rows=512, max_tokens=1024, max_requests=4, device=0)
ids = eng.generate_context_cache(w.chunks)
q = w.requests[0][-1].tokens
segs = [("cached", i) for i in ids] + [("tokens", q)]
for alg in ("legolink:4", "naive", "fr", "cacheblend:15"):
    eng.link(segs, alg, use_graph=False)
a = eng.link(segs, "legolink:4", use_graph=False, kv_share=True, keep_linked=True)
eng.linked_export(a.linked, 1)
perm = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in sg.permuted_requests(w, 3)]
outs = eng.link_batch(perm, "legolink:4", use_graph=False, kv_share=True, keep_linked=True)
eng.decode([o.linked for o in outs], [3, 5, 7], use_graph=False)
for o in outs:
    eng.materialize(o.linked)
eng.decode([o.linked for o in outs], [4, 6, 8], use_graph=False)
for o in outs + [a]:
    eng.release(o.linked)
ids0 = eng.generate_context_cache(w.chunks, dummy_prefix=4)
eng.link([("cached", i) for i in ids0] + [("tokens", q)], "legolink0", use_graph=False)
eng.link(segs, "legolink:4", use_graph=True, kv_share=True)
print("sanitize target done, pair =", os.environ.get("PIC_PAIR", "0"))
eng.close()
