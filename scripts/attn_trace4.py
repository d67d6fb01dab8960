"""Per-CTA attention accounting of the one-lane kernel on a cfg4 batch (PIC_ATTN_TRACE=1 must be set):
the last layer's launch of one eager link_batch per mode.
    python scripts/attn_trace4.py [n_requests] [n_layers] [modes, e.g. 0,1,3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
modes = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,1,3").split(",")]
w = sg.cfg4(n_requests=nr, n_layers=nl)
Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
eng = B.Engine(w.model, num_blocks=sum(len(c) for c in w.chunks) // 16 + 2 * sum(Ns) // 16 + 256, max_rows=8192,
               max_tokens=max(Ns) + 16, max_requests=nr, device=0)
ids = eng.generate_context_cache(w.chunks)
reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
B.set_attention_kernel(int(os.environ.get("ATTN_KERNEL", "1")))
for m in modes:
    for i in range(2):
        print(f"--- kv_share {m} eager {i}", file=sys.stderr, flush=True)
        eng.link_batch(reqs, w.alg, use_graph=False, kv_share=m)
B.set_attention_kernel(0)
eng.close()
