"""Edge cases of the linked-prefill path on the GPU vs the oracle (tcgen05 path, tiny-D128):
query-only prompts, N = 1, length-1 and ragged (non multiple of 16) chunks, k beyond the chunk
length, repeated cache ids, dynamic-first order, many small chunks (many q-tiles / blocks),
CacheBlend with R = 0 and R = 100, a prompt at the engine's max_tokens."""
import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
TOL = 2e-2
CFG = sg.TINY_D128


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def env():
    rng = np.random.default_rng(7)
    chunks = [np.concatenate([[CFG.bos_id], rng.integers(0, CFG.vocab, n - 1)]).astype(np.int32)
              for n in (1, 17, 33, 5, 64, 16, 100)]
    chunks += [np.concatenate([[CFG.bos_id], rng.integers(0, CFG.vocab, 7)]).astype(np.int32) for _ in range(40)]
    eng = B.Engine(CFG, num_blocks=2048, max_rows=2048, max_tokens=1024, max_requests=4, device=0)
    eids = eng.generate_context_cache(chunks)
    store = P.Store(M.Weights(CFG))
    oids = store.compile(chunks)
    yield eng, store, eids, oids, rng
    eng.close()


def run(env, segs, alg):
    eng, store, eids, oids, _ = env
    g = [("cached", eids[v]) if k == "c" else ("tokens", v) for k, v in segs]
    o = [("cached", oids[v]) if k == "c" else ("tokens", v) for k, v in segs]
    out = eng.link(g, alg, keep_linked=True, want_selected=True)
    ref = P.link(store, o, alg)
    assert np.array_equal(out.selected, ref.sel_per_layer[-1])
    assert rel(out.logits, ref.logits) < TOL, rel(out.logits, ref.logits)
    for l in range(CFG.n_layers):
        k, v = eng.linked_export(out.linked, l)
        assert rel(B.bf16_bits_to_f32(k), ref.K[l]) < TOL and rel(B.bf16_bits_to_f32(v), ref.V[l]) < TOL
    eng.release(out.linked)
    return out, ref


def q(env, n):
    return env[4].integers(0, CFG.vocab, n).astype(np.int32)


@pytest.mark.parametrize("alg", ["naive", "legolink:4", "fr", "cacheblend:15"])
def test_query_only_and_single_token(env, alg):
    run(env, [("t", q(env, 16))], alg)
    run(env, [("t", q(env, 1))], alg)


@pytest.mark.parametrize("alg", ["naive", "legolink:4", "legolink:1000", "fr", "cacheblend:0", "cacheblend:100"])
def test_ragged_chunks_and_k_beyond_length(env, alg):
    run(env, [("c", 0), ("c", 1), ("c", 2), ("c", 3), ("t", q(env, 3))], alg)


def test_repeated_ids_and_dynamic_first(env):
    run(env, [("t", q(env, 5)), ("c", 4), ("c", 4), ("t", q(env, 2)), ("c", 1)], "legolink:8")
    run(env, [("c", 6), ("t", q(env, 9)), ("c", 6)], "naive")


def test_many_small_chunks(env):
    segs = [("c", 7 + i) for i in range(40)] + [("t", q(env, 11))]
    run(env, segs, "legolink:2")          # 40 x 8 tokens: 331 rows over many 16-token blocks


def test_prompt_ends_in_cached_chunk(env):
    run(env, [("t", q(env, 4)), ("c", 5), ("c", 2)], "legolink:4")   # last row forced (R8)


def test_max_tokens_capacity(env):
    eng = env[0]
    long_q = q(env, 1024 - 100)
    run(env, [("c", 6), ("t", long_q)], "legolink:4")                # exactly max_tokens
    with pytest.raises(B.PicError) as e:
        eng.link([("cached", eng_id(env, 6)), ("tokens", q(env, 1024 - 99))], "naive")
    assert e.value.name == "PIC_E_CAPACITY"


def eng_id(env, i):
    return env[2][i]
