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

Pins: tests/test_oracle_pins.py (C1–C13 of SURVEY §8(c).4).  Functions with no pin
other than their own construction are marked "parity unpinned" below and in
DESIGN.md §3: LegoLink for 0 < k < n_c and CacheBlend with a non-trivial selection
(bracketed by pins C4/C5/C6/C9/C11 but without a closed form).
"""
from . import model, pic  # noqa: F401
