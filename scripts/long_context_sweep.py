"""SURVEY §8(f) f3 / PAPER.md:307-316 (Fig. 8): TTFT vs context length at a fixed 512-token chunk for
FR, CacheBlend-15 and LegoLink-16 on the Llama-3.1-8B shape, one B200, synchronous requests.

    python scripts/long_context_sweep.py [--chunks 4,8,16,32,64,94] [--reps 3] [--out FILE]

Prints one JSON line per (algorithm, N): device TTFT (CUDA events around pic_link, graphs on,
inputs resident), rows recomputed at layer 0 / in the last layer, and the linked tokens/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", default="4,8,16,32,64,94")
ap.add_argument("--algs", default="legolink:16,cacheblend:15,fr")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
ap.add_argument("--kv-share", default="0", help="comma list of kv_share settings to sweep (f3 shared-block link)")
args = ap.parse_args()
chunk_counts = [int(x) for x in args.chunks.split(",")]
algs = args.algs.split(",")
big = sg.long_context(max(chunk_counts))
m = big.model
N_max = sum(len(c) for c in big.chunks) + 64
dev = 0
torch.cuda.set_device(dev)
stream = torch.cuda.Stream(dev)
rows = []
with torch.cuda.stream(stream):
    eng = B.Engine(m, num_blocks=(2 * N_max) // 16 + 256, max_rows=N_max + 64, max_tokens=N_max + 64,
                   max_requests=1, device=dev, stream=stream)
    ids = eng.generate_context_cache(big.chunks)
    logits_dev = torch.empty((1, m.vocab), dtype=torch.float32, device=f"cuda:{dev}")
    for n_chunks in chunk_counts:
        w = sg.long_context(n_chunks)
        segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
        N = sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])
        for alg, share in [(a, int(k)) for a in algs for k in args.kv_share.split(",")]:
            eng.kv_share = int(share)
            try:
                pl = eng.plan(segs, alg)
                kv_row = m.n_layers * m.n_kv_heads * m.head_dim * 2 * 2       # K + V bf16 per token, all layers
                linked_gb = (len(pl["block_table"]) - pl["n_shared"]) * 16 * kv_row / 1e9
                o = eng.link(segs, alg, want_logits=False, logits_dev=logits_dev[0])    # warm-up + graph capture
                stream.synchronize()
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                for _ in range(args.reps):
                    o = eng.link(segs, alg, want_logits=False, logits_dev=logits_dev[0])
                ev1.record(stream)
                ev1.synchronize()
                ms = ev0.elapsed_time(ev1) / args.reps
                r = {"alg": alg, "kv_share": share, "N": N, "chunks": n_chunks, "ttft_ms": ms,
                     "tokens_per_s": N / ms * 1e3, "rows_layer0": o.n_selected_layer0, "rows_last": o.n_selected,
                     "linked_kv_gb_allocated": linked_gb}
            except B.PicError as e:
                r = {"alg": alg, "kv_share": share, "N": N, "chunks": n_chunks, "error": str(e)}
            rows.append(r)
            print(json.dumps(r), flush=True)
    eng.close()
if args.out:
    cols = [(a, int(k)) for a in algs for k in args.kv_share.split(",")]
    name = lambda a, k: f"{a}{' shared' if k else ''}"
    with open(args.out, "w") as f:
        f.write("# Long-context sweep (f3; PAPER.md:307-316): TTFT vs N, 512-token chunks, Llama-3.1-8B shape, 1 B200\n\n")
        f.write("TTFT ms (linked KV GB allocated by the link)\n\n")
        f.write("| N | " + " | ".join(name(a, k) for a, k in cols) + " |\n|---|" + "---|" * len(cols) + "\n")
        for n_chunks in chunk_counts:
            rs = [r for r in rows if r["chunks"] == n_chunks]
            f.write(f"| {rs[0]['N']} | " + " | ".join(
                f"{r['ttft_ms']:.1f} ({r['linked_kv_gb_allocated']:.2f})" if "ttft_ms" in r else r["error"][:40]
                for r in rs) + " |\n")
