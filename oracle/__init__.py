"""Oracle for the KVLink / LegoLink linked-prefill hot path (arXiv 2410.15332).

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import, call or execute anything in this package.
The product path (``paper_2410_15332_b200``, the C-ABI library ``libpic.so``) never
imports it, and it never imports the product.  The only shared module is
``seedgen`` (seeded synthetic inputs; no arithmetic of the method).

Plain, slow, obviously-correct NumPy float64:
  * ``oracle.model`` — the random-init Llama-family decoder (primitives + layer).
  * ``oracle.pic``   — compile, assemble/plan, link for Naive / FR / LegoLink-k /
    CacheBlend-r, the paged-layout (block allocator / slot map) model.

Pins: tests/test_oracle_pins.py (C1–C13 of SURVEY §8(c).4, plus C14–C19).  LegoLink for
0 < k < n_c and CacheBlend with a non-trivial selection have no closed form in the paper;
they are pinned by independent constructions from HuggingFace Llama's own forward, KV cache
and decoder layers (C18: sequential forwards over a cache of re-based standalone-prefill
chunk KV; C19: layer-wise recomputation under an explicit position mask, the selection rule
restated), so no oracle function is left "parity unpinned".
"""
from . import model, pic  # noqa: F401
