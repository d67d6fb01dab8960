"""Per-kernel-class breakdown of one decode step (f1) over a cfg4 wave of linked caches (profiling on:
graphs off, CUDA events around every launch), next to the TPOT of the graph path.
    python scripts/decode_profile.py [n_requests] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = sg.cfg4(n_requests=nr)
Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
eng = B.Engine(w.model, num_blocks=(sum(len(c) for c in w.chunks) + 2 * sum(Ns)) // 16 + 64 * nr + 64, max_rows=8192,
               max_tokens=max(Ns) + 160, max_requests=nr, device=0)
ids = eng.generate_context_cache(w.chunks)
reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
hs = [o.linked for o in eng.link_batch(reqs, w.alg, keep_linked=True, want_logits=False, kv_share=3)]
if not os.environ.get("DECODE_FRAMES"):  # DECODE_FRAMES=1: decode the chunk-frame links as linked (q rotation)
    for h in hs:
        eng.materialize(h)
toks = [int(t) for t in sg.tokens(0xDEC0DE, 7, nr, w.model.vocab, None)]
dl = torch.empty((nr, w.model.vocab), dtype=torch.float32, device="cuda:0")
for _ in range(3):
    eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr())
e1.record()
e1.synchronize()
print(f"decode TPOT (graph) {e0.elapsed_time(e1) / steps:.3f} ms at batch {nr}, context ~{Ns[0]}")
if os.environ.get("DECODE_NCU"):  # one eager decode step inside a profiler range (ncu --profile-from-start off)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr(), use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
eng.set_profiling(True)
eng.profile(reset=True)
for _ in range(steps):
    eng.decode(hs, toks, want_logits=False, logits_dev=dl.data_ptr(), use_graph=False)
torch.cuda.synchronize()
prof = eng.profile(reset=True)
tot = sum(v["ms"] for v in prof.values()) / steps
print(f"profiled (graphs off) sum {tot:.3f} ms per step")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    ms = v["ms"] / steps
    print(f"  {k:18s} {ms:7.3f} ms  {v['launches'] // steps:4d} launches  {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s"
          f"  {v['flops'] / max(v['ms'], 1e-9) / 1e9:8.1f} TFLOP/s")
