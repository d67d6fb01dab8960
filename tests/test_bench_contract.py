"""The bench.py JSON-line contract on CPU: `--impl reference` (the fp64 oracle arm, the one leg besides
tests and smoke that may run oracle/) prints one line with the contract's keys, on the same metric and
workload config as the GPU arm, with its bounded-sample baseline description and zero-byte e2e."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) >= 1
    d = json.loads(lines[-1])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == "linked_prefill_tokens_per_s" and d["unit"] == "tokens/s" and d["higher_is_better"]
    assert d["config"]["workload"].startswith("cfg4: 256 request(s)")
    assert d["config"]["kv_share"] == 3 and d["config"]["alg"] == "legolink:16"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] >= 3


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm on one 32-request wave: every key of the contract, a live roofline measured from CUDA
    events, the clocks sample, the engine's own launch count, an e2e with the bytes it copied."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--requests", "32", "--steps", "2",
                        "--warmup", "3", "--decode-steps", "2", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.strip().splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "e2e", "roofline", "ttft_ms"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "bf16"
    assert d["gpu_launches"] > 0 and d["value"] > 0
    roof = d["roofline"]
    assert roof["bound"] in ("tensor", "hbm") and 0 < roof["frac"] < 1.2 and roof["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["clocks"]["sm_mhz"] > 0 and d["ttft_ms"]["requests"] == 32
    assert d["decode"]["tpot_ms"] > 0
