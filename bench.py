#!/usr/bin/env python
"""Linked-prefill benchmark (BASELINE.json metric: linked-prefill TTFT and linked tokens/s,
with % of HBM / tensor roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg3|cfg4] [--alg ALG]
                    [--impl ours|reference]

A step = one linked prefill (pic_link, all rows of SURVEY §8(a)) of the workload's request(s)
on synthetic random-init weights of the named shape.  Multi-GPU (torchrun): one process per
GPU, each links its own independent requests (data parallel by request, no collective on the
path; "scaling": "weak"); timing is the max over ranks of CUDA-event time.

--impl reference times the fp64 CPU oracle (oracle/) on a bounded sample of the same workload
(there is no reference implementation to install: the paper ships no code)."""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import seedgen as sg  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return FALLBACK, "fallback"


def workload(name: str, alg: str | None, world: int = 1, per_gpu: int = 32):
    if name == "cfg2":
        w = sg.cfg2(alg or "legolink:16")
    elif name == "cfg3":
        w = sg.cfg3(alg or "legolink:32")
    elif name == "cfg5":
        w = sg.cfg5(alg or "legolink:16")             # 70B shape, 32K context: fits one B200 (141 GB bf16)
    elif name == "cfg4":
        # weak scaling: `per_gpu` independent requests per GPU, request r -> rank r mod world
        w = sg.cfg4(n_requests=per_gpu * world, alg=alg or "legolink:16")
    else:
        raise SystemExit(f"unknown config {name}")
    return w


def describe(w) -> dict:
    m = w.model
    n_chunks = len(w.requests[0]) - (0 if w.requests[0][-1].cached else 1)
    q = 0 if w.requests[0][-1].cached else len(w.requests[0][-1].tokens)
    return {"workload": f"{w.name}: {m.name}-shaped random-init bf16, {n_chunks} chunks x {len(w.chunks[0])} tokens"
                        f" + {q}-token query, {w.alg}, {len(w.requests)} request(s) per GPU",
            "model": m.name, "n_layers": m.n_layers, "d_model": m.d_model, "vocab": m.vocab,
            "chunk_len": len(w.chunks[0]), "n_chunks": n_chunks, "query_len": q, "alg": w.alg,
            "requests_per_gpu_step": len(w.requests),
            "l2": "inputs larger than L2 (weights 14+ GB re-read every step), no flush"}


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dummy_prefix(alg):
    """LegoLink-0 links chunks compiled behind 4 dummy BOS tokens; every other
    algorithm uses the plain compile."""
    return 4 if alg == "legolink0" else 0


# ------------------------------------------------------------------------------------- CPU oracle
class OracleSample:
    """The fp64 oracle's link on a bounded sample: layer 0 of one request (all its work: re-base of
    every cached row of that layer, the layer on the k' rows) plus the LM head, extrapolated to all
    L layers.  Weights are generated once (not timed); each run() is one timed sample."""

    def __init__(self, w):
        from oracle import model as M
        from oracle import pic as P
        self.M, self.P, self.w = M, P, w
        cfg = w.model
        self.Wt = M.Weights(sg.truncated(cfg, 1))
        self.Wt.layer(0)
        self.Wt.lm_head
        self.store = P.Store(self.Wt)
        over = [(np.zeros((1, len(c), cfg.n_kv_heads, cfg.head_dim)), np.zeros((1, len(c), cfg.n_kv_heads, cfg.head_dim)))
                for c in w.chunks]
        oids = self.store.compile(w.chunks, compiled_override=over, dummy_prefix=dummy_prefix(w.alg))
        self.segs = [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
        self.N = sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])

    def run(self):
        cfg = self.w.model
        t0 = time.perf_counter()
        r = self.P.link(self.store, self.segs, self.w.alg, layers=1)
        tl = time.perf_counter() - t0
        t0 = time.perf_counter()
        self.M.logits_of(self.Wt, r.hidden[-1][-1])
        th = time.perf_counter() - t0
        per_req = cfg.n_layers * (tl - th) + th
        return self.N / per_req, per_req, (f"oracle fp64 link of 1 request (N={self.N}): layer 0 of {cfg.n_layers} "
                                           f"+ LM head timed ({tl:.2f} s), extrapolated x{cfg.n_layers} layers")


def oracle_sample(w, min_seconds: float = 10.0):
    """cpu_baseline: the sampled oracle link repeated until >= min_seconds of CPU work,
    reported as the mean over the repetitions."""
    osamp = OracleSample(w)
    vals, spent, sample = [], 0.0, ""
    while spent < min_seconds or not vals:
        t0 = time.perf_counter()
        v, per_req, sample = osamp.run()
        spent += time.perf_counter() - t0
        vals.append(per_req)
    per_req = float(np.mean(vals))
    return osamp.N / per_req, per_req, f"{sample}; {len(vals)} repetitions, {spent:.1f} s of CPU work"


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------------------------- main
def ncu_traffic(kernel_class):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel class from the committed
    ncu --set full capture (profiles/ncu_r1_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_r1_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_class, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def roofline(prof, P, src, nsteps):
    """Dominant kernel class of the profiled steps against its roofline."""
    tot = sum(v["ms"] for v in prof.values())
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    intensity = dom["flops"] / max(dom["bytes"], 1)
    ridge = P["bf16_tflops"] * 1e12 / (P["hbm_gbs"] * 1e9)
    if intensity < ridge:
        achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": P["hbm_gbs"], "unit": "GB/s"}
    else:
        achieved = dom["flops"] / (dom["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": P["bf16_tflops"], "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    if roof["bound"] == "tensor" and P.get("bf16_tflops_sustained"):
        # the driver's sustained figure (back-to-back matmuls for seconds, power-capped clocks) applies to a
        # kernel timed inside a long step; "peak" stays the burst figure (the conservative denominator)
        roof["peak_sustained"] = P["bf16_tflops_sustained"]
        roof["frac_sustained"] = roof["achieved"] / P["bf16_tflops_sustained"]
    roof["traffic"] = ncu_traffic(dom_name)
    roof["kernel"] = dom_name
    roof["share_of_step"] = dom["ms"] / tot
    roof["peak_source"] = f"{src} (MEASURED_PEAKS.json burst)" if src == "measured" else "fallback (B200_PROFILING.md)"
    roof["launches_per_step"] = dom["launches"] / nsteps
    roof["how"] = (f"algorithmic bytes/FLOPs per launch (SURVEY §8(d)) over CUDA-event durations of every launch, "
                   f"{nsteps} profiled steps on the bench stream (graphs off)")
    breakdown = {k: {"ms_per_step": v["ms"] / nsteps, "launches_per_step": v["launches"] / nsteps,
                     "GB/s": v["bytes"] / max(v["ms"], 1e-9) / 1e6, "TFLOP/s": v["flops"] / max(v["ms"], 1e-9) / 1e9}
                 for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
    return roof, breakdown


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--alg", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--tp", action="store_true",
                    help="tensor parallel over all ranks (heads/MLP columns sharded, fused peer-memory all-reduce); "
                         "strong scaling of one request instead of data parallel requests")
    ap.add_argument("--layers", type=int, default=None, help="truncate depth (functional runs only; marked in config)")
    ap.add_argument("--kv-share", type=int, default=1, choices=[0, 1],
                    help="f3 shared-block link: chunk-store blocks linked by reference, keys re-based in the "
                         "attention K-tile load (pic_link_params.kv_share)")
    ap.add_argument("--decode-steps", type=int, default=32,
                    help="f1: decode steps over the linked caches after the link measurement (0 = skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2410_15332_b200 import dist as D
    rank, world, local = D.env_rank()
    w = workload(args.config, args.alg, 1 if args.tp else world)
    if args.layers:
        w.model = sg.truncated(w.model, args.layers)
    if not args.tp:
        if len(w.requests) == 1:
            w.requests = w.requests * world            # single-request configs: one copy per GPU
        w.requests = D.shard(w.requests, rank, world)   # data parallel by independent request
    cfgd = describe(w)
    cfgd["kv_share"] = bool(args.kv_share)
    N_tok = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        osamp = OracleSample(w)
        for i in range(args.warmup + args.steps):
            v, per_req, sample = osamp.run()
            if i >= args.warmup:
                vals.append((v, per_req))
        v = float(np.median([x[0] for x in vals]))
        ms = float(np.median([x[1] for x in vals])) * 1e3 * len(w.requests)
        line = {"impl": "reference", "metric": "linked_prefill_tokens_per_s", "value": v, "unit": "tokens/s",
                "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfgd,
                "cpu_baseline": {"kind": "oracle", "value": v, "unit": "tokens/s", "cores": cores_used(),
                                 "sample": sample},
                "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    from paper_2410_15332_b200 import pic as B

    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    red_dev = f"cuda:{dev}"
    if world > 1:
        if args.tp:
            D.init("gloo")        # TP data moves through peer memory; the group only exchanges handles/timings
            red_dev = None
        else:
            D.init("nccl", device_id=torch.device(f"cuda:{dev}"))
    stream = torch.cuda.Stream(dev)
    m = w.model
    total_tokens = sum(len(c) for c in w.chunks)
    max_N = max(N_tok)
    # rows recomputed per forward: Σ k' of the batch (host-only planner), N for CacheBlend
    planner = B.Engine(m, num_blocks=(total_tokens + max_N) // 16 + 2 * len(w.chunks) + 64, max_rows=64,
                       max_tokens=max(max_N, 512) + 16, max_requests=1, device=None)
    pids = planner.generate_context_cache(w.chunks, dummy_prefix=dummy_prefix(w.alg))
    rows_link = sum(N_tok) if w.alg.startswith("cacheblend") else sum(
        len(planner.plan([("cached", pids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r], w.alg)["sel"])
        for r in w.requests)
    planner.close()
    with torch.cuda.stream(stream):
        tp_kw = dict(tp_rank=rank, tp_size=world) if args.tp else {}
        eng = B.Engine(m, num_blocks=(total_tokens + sum(N_tok)) // 16 + 2 * len(w.chunks) + 64 * len(w.requests),
                       max_rows=max(4096, rows_link), max_tokens=max(max_N + 2 * args.decode_steps + 16, 512) + 16,
                       max_requests=len(w.requests), device=dev, stream=stream, **tp_kw)
        eng.kv_share = bool(args.kv_share)
        if args.tp and world > 1:
            D.tp_connect(eng)
        ids = eng.generate_context_cache(w.chunks, dummy_prefix=dummy_prefix(w.alg))
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
        logits_dev = torch.empty((len(reqs), m.vocab), dtype=torch.float32, device=f"cuda:{dev}")

        def step():
            if len(reqs) == 1:
                return [eng.link(reqs[0], w.alg, want_logits=False, logits_dev=logits_dev[0])]
            return eng.link_batch(reqs, w.alg, want_logits=False)

        for _ in range(args.warmup):
            step()
        stream.synchronize()
        kernels_per_step = eng.stats()["kernels_last_call"]

        barrier = D.barrier

        # ---------------- timed region: device-resident inputs, CUDA events on our stream
        barrier()
        torch.cuda.synchronize(dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]   # per-step boundaries
        with ClockSampler(dev) as clk:
            ev0.record(stream)
            for i in range(args.steps):
                outs = step()
                evs[i].record(stream)
            ev1.record(stream)
            ev1.synchronize()
        torch.cuda.synchronize(dev)
        barrier()
        ms_max = D.max_over_ranks(ev0.elapsed_time(ev1), device=red_dev)
        ms_per_step = ms_max / args.steps
        step_ms = sorted([ev0.elapsed_time(evs[0])] + [evs[i - 1].elapsed_time(evs[i]) for i in range(1, args.steps)])
        ttft_dist = {"p50": float(np.percentile(step_ms, 50)), "p90": float(np.percentile(step_ms, 90)),
                     "min": step_ms[0], "max": step_ms[-1], "how": "per-step CUDA events inside the timed region (rank 0)"}
        tokens_all = (sum(N_tok) if args.tp else D.sum_over_ranks(sum(N_tok), device=red_dev)) * args.steps
        value = tokens_all / (ms_max / 1e3)

        # ---------------- e2e: the public call with host buffers (plan H2D + logits D2H per step)
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            if len(reqs) == 1:
                o = eng.link(reqs[0], w.alg, want_logits=True)
            else:
                o = eng.link_batch(reqs, w.alg, want_logits=True)[0]
        e1.record(stream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        st = eng.stats()
        wall_max = D.max_over_ranks(wall, device=red_dev)
        e2e_value = tokens_all / wall_max

        # ---------------- f1: decode over the linked caches (TPOT); batch = this rank's requests
        dec = None
        if args.decode_steps > 0 and not args.tp:
            held = (eng.link_batch(reqs, w.alg, keep_linked=True) if len(reqs) > 1
                    else [eng.link(reqs[0], w.alg, keep_linked=True)])
            hs = [o.linked for o in held]
            # shared-block links: re-base the shared blocks into owned ones once, instead of re-rotating
            # them in every decode step (pic_linked_materialize; timed on its own)
            mat_ms = None
            if args.kv_share:
                torch.cuda.synchronize(dev)
                m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                m0.record(stream)
                for h in hs:
                    eng.materialize(h)
                m1.record(stream)
                m1.synchronize()
                mat_ms = m0.elapsed_time(m1)
            forced = [int(t) for t in sg.tokens(0xDEC0DE, 7, len(hs), m.vocab, None)]
            dl = torch.empty((len(hs), m.vocab), dtype=torch.float32, device=f"cuda:{dev}")
            for _ in range(3):
                eng.decode(hs, forced, want_logits=False, logits_dev=dl.data_ptr())
            dec_launches = eng.stats()["kernels_last_call"]
            barrier()
            torch.cuda.synchronize(dev)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            for _ in range(args.decode_steps):                    # teacher-forced: no host round trip
                eng.decode(hs, forced, want_logits=False, logits_dev=dl.data_ptr())
            d1.record(stream)
            d1.synchronize()
            barrier()
            tpot = D.max_over_ranks(d0.elapsed_time(d1), device=red_dev) / args.decode_steps
            t0 = time.perf_counter()
            toks = forced
            for _ in range(args.decode_steps // 2):               # greedy through the public call
                toks = [int(t) for t in eng.decode(hs, toks, want_logits=False).next_token]
            tpot_host = (time.perf_counter() - t0) / max(1, args.decode_steps // 2) * 1e3
            batch_all = D.sum_over_ranks(len(hs), device=red_dev)
            dec = {"tpot_ms": tpot, "tokens_per_s": batch_all / (tpot / 1e3), "batch_per_gpu": len(hs),
                   "context_tokens": int(max_N), "steps": args.decode_steps, "tpot_ms_host_greedy": tpot_host,
                   "gpu_launches_per_step": int(dec_launches), "materialize_ms": mat_ms,
                   "how": "pic_decode over the linked caches of this rank's requests (f1), one token per cache per "
                          "step, CUDA events on the bench stream (teacher-forced), then a greedy host loop; "
                          "shared-block links are materialized first (pic_linked_materialize, materialize_ms)"}
            for h in hs:
                eng.release(h)

        # ---------------- per-kernel CUDA-event profile (separate pass, same stream)
        eng.set_profiling(True)
        eng.profile(reset=True)
        for _ in range(args.profile_steps):
            step()
        prof = eng.profile(reset=True)
        eng.set_profiling(False)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    P, src = peaks()
    roof, breakdown = roofline(prof, P, src, args.profile_steps) if prof else (None, {})
    line = {"metric": "linked_prefill_tokens_per_s", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ttft_ms_device": ms_per_step if len(reqs) == 1 else None,
            "step_ms_distribution": ttft_dist,
            "ttft_ms_requests": ({"mean": ms_per_step, "p99": float(np.percentile(step_ms, 99)),
                                  "how": "SURVEY 8(d) cfg4: every request of a wave arrives at t=0, its TTFT is the "
                                         "wave's completion (one wave per step)"} if len(reqs) > 1 else None),
            "higher_is_better": True, "scaling": "strong" if args.tp else "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": dict(cfgd, parallelism=(f"tp{world} (heads/MLP sharded, fused peer-memory all-reduce)" if args.tp
                                              else f"dp{world} (independent requests)"),
                           **({"truncated_layers": args.layers} if args.layers else {})),
            "clocks": clk.summary(), "gpu_launches": int(kernels_per_step * args.steps),
            "e2e": {"value": e2e_value, "unit": "tokens/s", "ttft_ms_host": wall_max / args.steps * 1e3,
                    "h2d_bytes_per_step": int(st["h2d_bytes_last_call"]),
                    "d2h_bytes_per_step": int(st["d2h_bytes_last_call"])},
            "roofline": roof, "kernel_breakdown": breakdown, "decode": dec,
            "context": "paper (A100-80GB, vLLM 0.4.1): LegoLink-16 up to 8x lower TTFT and 7x throughput vs "
                       "CacheBlend-15 under load (P:303-305); not comparable hardware/workload"}
    if world == 1 and not args.no_cpu_baseline:
        v, per_req, sample = oracle_sample(w)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores_used(), "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
