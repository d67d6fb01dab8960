"""compute-sanitizer target for the session-3 kernels: a chunk-frame link over 128-token chunks (the persistent
Q-side re-base attention, attention_qp.cu: split pieces on a small batch, multi-item CTAs), the one-CTA QROT
kernel beside it, and decode steps through the split-KV decode kernel (attention_decode.cu) at G = 2 and 4;
eager launches so every kernel is checked on its own."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

for cfg in (sg.TINY_D128, replace(sg.TINY_TP8, name="tiny-tp8-g4", n_kv_heads=4)):
    ws = sg.workload_seed(0x54)
    chunks = sg.make_chunks(ws, 5, 128, cfg.vocab, cfg.bos_id)
    q = sg.make_query(ws, 0, 24, cfg.vocab)
    eng = B.Engine(cfg, num_blocks=1024, max_rows=1024, max_tokens=2048, max_requests=4, device=0)
    ids = eng.generate_context_cache(chunks)
    reqs = [[("cached", ids[c]) for c in o] + [("tokens", q)] for o in ([0, 1, 2, 3, 4], [4, 2, 0, 3], [1, 3])]
    eng.link_batch(reqs, "legolink:16", kv_share=3, use_graph=False)          # persistent QROT
    os.environ["PIC_NO_ATTN_PERSIST"] = "1"
    eng.link_batch(reqs, "legolink:16", kv_share=3, use_graph=False)          # one-CTA QROT
    os.environ.pop("PIC_NO_ATTN_PERSIST")
    outs = eng.link_batch(reqs, "legolink:16", keep_linked=True, use_graph=False)
    hs = [o.linked for o in outs]
    for t in (3, 5, 7):
        eng.decode(hs, [t] * len(hs), use_graph=False)                       # split-KV decode kernel
    for h in hs:
        eng.release(h)
    eng.close()
print("sanitize_s3 target done")
