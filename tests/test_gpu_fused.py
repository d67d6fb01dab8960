"""Fused consumers in the GEMM epilogues and the attention output (tensor-bound shapes, split-K = 1):
the a5 RoPE + scatter in the QKV GEMM epilogue, the a7/a8 residual add in the O / down GEMM epilogues,
and unsplit attention q-tiles writing their normalised bf16 output directly.  The fused path performs
the same fp32 operations on the same accumulators as the separate kernels (qkv_rope_scatter,
residual_rmsnorm), so the link must be BIT-IDENTICAL to PIC_NO_EPI_FUSE=1 (the separate kernels),
at the tiny D=128 shape and at a cfg4 wave (Llama-3.1-8B width, 2 layers, 8 requests)."""
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


@pytest.mark.parametrize("which", ["tiny", "cfg4"])
def test_fused_epilogues_bit_identical_to_separate_kernels(which, tmp_path):
    script = tmp_path / "run.py"
    script.write_text(SCRIPT % {"root": ROOT})
    outs = []
    for fuse in (True, False):
        env = dict(os.environ)
        env.pop("PIC_NO_EPI_FUSE", None)
        if not fuse:
            env["PIC_NO_EPI_FUSE"] = "1"
        out = tmp_path / f"{which}_{int(fuse)}.npz"
        r = subprocess.run([sys.executable, str(script), which, str(out)], env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(np.load(out))
    a, b = outs
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
