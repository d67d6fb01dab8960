"""SURVEY §8(f) f4 / PAPER.md:258, :293-305 (Fig. 7): open-loop Poisson serving of LegoLink-16 vs
CacheBlend-15 on the Llama-3.1-8B shape, one B200.  d users each own 10 x 512-token chunks (compiled
once) and resend their RAG request (the chunks + a 64-token query); the pool is sized so that the
resident context cache takes a given share of it (CCR).  Reports TTFT and throughput vs rate.

    python scripts/serve_sweep.py [--users 16] [--rates 25,50,100,200,400] [--ccr 0.2,0.5,0.8] [--duration 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seedgen as sg  # noqa: E402
from paper_2410_15332_b200 import pic as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--users", type=int, default=16)
ap.add_argument("--rates", default="25,50,100,200,400")
ap.add_argument("--ccr", default="0.2,0.5,0.8")
ap.add_argument("--algs", default="legolink:16,cacheblend:15")
ap.add_argument("--duration", type=float, default=3.0)
ap.add_argument("--max-batch", type=int, default=32)
ap.add_argument("--out", default=None)
ap.add_argument("--kv-share", default="0", help="comma list of kv_share settings (f3 shared-block link)")
args = ap.parse_args()
m = sg.LLAMA31_8B
d = args.users
ws = sg.workload_seed(7)
user_chunks = [sg.make_chunks(ws ^ (u << 20), 10, 512, m.vocab, m.bos_id) for u in range(d)]
queries = [sg.make_query(ws, u, 64, m.vocab) for u in range(d)]
resident = d * 10 * 32                      # blocks of the users' compiled chunks
link_blocks = (10 * 512 + 64 + 15) // 16
torch.cuda.set_device(0)
stream = torch.cuda.Stream(0)
rows = []
with torch.cuda.stream(stream):
    for ccr in [float(x) for x in args.ccr.split(",")]:
        total = max(int(resident / ccr), resident + link_blocks)
        eng = B.Engine(m, num_blocks=total, max_rows=8192, max_tokens=5248, max_requests=args.max_batch, device=0,
                       stream=stream)
        ids = [eng.generate_context_cache(c) for c in user_chunks]
        reqs = [[("cached", i) for i in ids[u]] + [("tokens", queries[u])] for u in range(d)]
        for alg, share in [(a, int(k)) for a in args.algs.split(",") for k in args.kv_share.split(",")]:
            eng.kv_share = int(share)
            eng.link(reqs[0], alg)                                   # warm-up
            for rate in [float(x) for x in args.rates.split(",")]:
                st = eng.serve_poisson(reqs, alg, rate, args.duration, seed=int(rate * 1000) ^ 0x5E12E,
                                       max_batch=args.max_batch)
                r = {"alg": alg, "kv_share": share, "ccr": round(st["ccr"], 3), "rate": rate, **{k: st[k] for k in
                     ("n_completed", "throughput_rps", "ttft_mean_ms", "ttft_p50_ms", "ttft_p99_ms", "mean_batch",
                      "tokens_per_s")}}
                rows.append(r)
                print(json.dumps(r), flush=True)
        eng.close()
if args.out:
    with open(args.out, "w") as f:
        f.write(f"# Open-loop Poisson serving (f4; PAPER.md:258, 293-305): {d} users x (10 x 512-token chunks + 64-token "
                f"query), Llama-3.1-8B shape, 1 B200, {args.duration:.0f} s windows, eager launches\n\n")
        f.write("| alg | kv_share | CCR | rate (req/s) | throughput (req/s) | TTFT mean ms | p50 | p99 | mean batch |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['alg']} | {r['kv_share']} | {r['ccr']:.2f} | {r['rate']:.0f} | {r['throughput_rps']:.1f} | {r['ttft_mean_ms']:.1f} | "
                    f"{r['ttft_p50_ms']:.1f} | {r['ttft_p99_ms']:.1f} | {r['mean_batch']:.2f} |\n")
