"""compute-sanitizer target (memcheck / racecheck / synccheck): the tiny-D128 link through every kernel
family — copy path and shared-block link (K-tile re-base warps), CacheBlend selection, a batched link,
LegoLink-0 compile, decode over the linked cache, materialize; both attention kernels (one-lane and the
persistent ping-pong kernel, copy and rotating variants); an FR batch (M = 336 rows: the CTA-pair
gate/up GEMM, unsplit fused epilogues and the fused RMSNorm; PIC_PAIR_FUSED=1 adds the pair residual /
QKV epilogues).  Eager launches so every kernel is checked individually, then one graph replay."""
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
for kern in (2, 1):  # ping-pong kernel forced (copy and rotating variants), then the one-lane kernel
    B.set_attention_kernel(kern)
    eng.link(segs, "legolink:4", use_graph=False, kv_share=False)
    eng.link(segs, "legolink:4", use_graph=False, kv_share=True)
    eng.link(segs, "legolink:4", use_graph=False, kv_share=3)
    eng.link_batch(perm, "fr", use_graph=False)  # M = 336: pair SwiGLU GEMM, fused epilogues and norm
B.set_attention_kernel(0)
eng.close()
# Llama-3.1-8B width, one layer, a 2-request cfg4 batch (M = 416): the default CTA-pair gate/up + SwiGLU
# GEMM (N-tile 224), the fused-norm epilogues and the staged residual epilogue at the bench's shapes
w4 = sg.cfg4(n_requests=2, n_layers=1)
Ns = [sum(len(w4.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w4.requests]
e4 = B.Engine(w4.model, num_blocks=(sum(len(c) for c in w4.chunks) + 2 * sum(Ns)) // 16 + 64, max_rows=4096,
              max_tokens=max(Ns) + 16, max_requests=2, device=0)
i4 = e4.generate_context_cache(w4.chunks)
r4 = [[("cached", i4[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w4.requests]
for share in (1, 0, 3):  # 3: chunk-frame link, Q-side re-base (QROT) at the bench's tile sizes
    e4.link_batch(r4, w4.alg, use_graph=False, kv_share=share)
e4.close()
print("sanitize target done, pair fused =", os.environ.get("PIC_PAIR_FUSED", "0"))
