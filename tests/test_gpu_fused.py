"""Fused consumers in the GEMM epilogues and the attention output (tensor-bound shapes, split-K = 1):
the a5 RoPE + scatter in the QKV GEMM epilogue, the a7/a8 residual add in the O / down GEMM epilogues,
and unsplit attention q-tiles writing their normalised bf16 output directly.  The fused path performs
the same fp32 operations on the same accumulators as the separate kernels (qkv_rope_scatter,
residual_rmsnorm), so the link must be BIT-IDENTICAL to PIC_NO_EPI_FUSE=1 (the separate kernels),
at the tiny D=128 shape and at a cfg4 wave (Llama-3.1-8B width, 2 layers, 8 requests).

The a4 RMSNorm fused across the GEMM boundary (the residual epilogue writes bf16(h·g) and Σh² partials,
the consumer scales its accumulator rows by rsqrt(mean h² + eps)) rounds x = h·g instead of h·r·g to bf16,
so it is compared at tolerance against the residual_rmsnorm kernel (PIC_NO_NORM_FUSE=1); the bit-identity
test above runs with it off.  Its parity against the fp64 oracle at bench size is test_gpu_parity_bench's
cfg4 wave."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r)
import seedgen as sg
from paper_2410_15332_b200 import pic as B
which, out = sys.argv[1], sys.argv[2]
w = sg.cfg1(model=sg.TINY_D128) if which == "tiny" else sg.cfg4(n_requests=8, n_layers=2)
Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
eng = B.Engine(w.model, num_blocks=(sum(len(c) for c in w.chunks) + 2 * sum(Ns)) // 16 + 64, max_rows=4096,
               max_tokens=max(Ns) + 16, max_requests=len(Ns), device=0)
ids = eng.generate_context_cache(w.chunks)
reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
res = {}
for share in (False, True):
    outs = eng.link_batch(reqs, "legolink:4" if which == "tiny" else w.alg, keep_linked=True, kv_share=share)
    for i, o in enumerate(outs):
        res[f"logits{int(share)}_{i}"] = o.logits
        for l in range(w.model.n_layers):
            k, v = eng.linked_export(o.linked, l)
            res[f"k{int(share)}_{i}_{l}"] = k
            res[f"v{int(share)}_{i}_{l}"] = v
        eng.release(o.linked)
ck, cv = eng.cache_export(ids[0], w.model.n_layers - 1)   # compile forward (fused too)
res["ck"], res["cv"] = ck, cv
np.savez(out, **res)
"""


def _run(tmp_path, which, tag, env_set):
    script = tmp_path / "run.py"
    script.write_text(SCRIPT % {"root": ROOT})
    env = dict(os.environ)
    for k in ("PIC_NO_EPI_FUSE", "PIC_NO_NORM_FUSE"):
        env.pop(k, None)
    env.update(env_set)
    out = tmp_path / f"{which}_{tag}.npz"
    r = subprocess.run([sys.executable, str(script), which, str(out)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("which", ["tiny", "cfg4"])
def test_fused_epilogues_bit_identical_to_separate_kernels(which, tmp_path):
    a = _run(tmp_path, which, "fused", {"PIC_NO_NORM_FUSE": "1"})
    b = _run(tmp_path, which, "separate", {"PIC_NO_NORM_FUSE": "1", "PIC_NO_EPI_FUSE": "1"})
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _f32(x):
    x = np.asarray(x)
    return (x.astype(np.uint32) << 16).view(np.float32) if x.dtype == np.uint16 else x


@pytest.mark.parametrize("which", ["tiny", "cfg4"])
def test_fused_norm_matches_rmsnorm_kernel(which, tmp_path):
    """Layer-0 K/V are produced before any fused norm (bit-identical); later layers and the logits agree
    with the residual_rmsnorm path to bf16 rounding of x (well inside the 2e-2 oracle bar)."""
    a = _run(tmp_path, which, "normfused", {})
    b = _run(tmp_path, which, "kernel", {"PIC_NO_NORM_FUSE": "1"})
    assert sorted(a.files) == sorted(b.files)
    worst = 0.0
    for k in a.files:
        if k.endswith("_0") and k[0] in "kv":      # layer 0 of every request: before the first fused norm
            assert np.array_equal(a[k], b[k]), k
        err = _rel(_f32(a[k]), _f32(b[k]))
        worst = max(worst, err)
        assert err < 1e-2, (k, err)
    print(f"fused-norm vs rmsnorm kernel: worst rel-L2 {worst:.2e}")
