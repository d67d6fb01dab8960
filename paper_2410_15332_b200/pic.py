"""ctypes binding of libpic.so (include/pic.h).  Argument marshalling only: every step of the
linked-prefill path runs in the library's CUDA kernels.  PyTorch provides the device arena and
the stream.  There is no fallback: if libpic.so is missing or the GPU is absent, calls fail."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("PIC_LIB_NAME", "libpic.so"))  # override: experiment builds only

PIC_SEG_CACHED, PIC_SEG_TOKENS = 0, 1
PIC_NAIVE, PIC_FULL, PIC_LEGOLINK, PIC_CACHEBLEND, PIC_LEGOLINK0 = 0, 1, 2, 3, 4
STATUS = ["PIC_OK", "PIC_E_INVALID_ARG", "PIC_E_CONFIG", "PIC_E_EMPTY_INPUT", "PIC_E_CAPACITY",
          "PIC_E_MISSING_CACHE", "PIC_E_LAYOUT", "PIC_E_VARIANT", "PIC_E_OOM", "PIC_E_CUDA",
          "PIC_E_NO_DEVICE", "PIC_E_TOKEN"]


class PicError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)


class ModelConfigC(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("vocab", C.c_int32), ("max_pos", C.c_int32), ("bos_id", C.c_int32),
                ("rope_theta", C.c_double), ("rms_eps", C.c_double), ("seed", C.c_uint64), ("dtype", C.c_int32)]


class LimitsC(C.Structure):
    _fields_ = [("num_blocks", C.c_int64), ("max_rows", C.c_int32), ("max_tokens", C.c_int32),
                ("max_requests", C.c_int32)]


class SegmentC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_tokens", C.c_int32), ("id", C.c_uint64),
                ("tokens", C.POINTER(C.c_int32))]


class CompileOptionsC(C.Structure):
    _fields_ = [("dummy_prefix", C.c_int32), ("dummy_token", C.c_int32)]


class LinkParamsC(C.Structure):
    _fields_ = [("alg", C.c_int32), ("k", C.c_int32), ("r_percent", C.c_int32), ("check_layer", C.c_int32),
                ("rebase", C.c_int32), ("use_graph", C.c_int32), ("sel_override", C.POINTER(C.c_int32)),
                ("n_sel_override", C.c_int32), ("debug_hidden", C.POINTER(C.c_float)), ("kv_share", C.c_int32)]


class LinkResultC(C.Structure):
    _fields_ = [("logits", C.POINTER(C.c_float)), ("logits_dev", C.c_void_p), ("first_token", C.c_int32),
                ("n_tokens", C.c_int32), ("n_selected", C.c_int32), ("n_selected_layer0", C.c_int32),
                ("selected", C.POINTER(C.c_int32))]


class PlanOutC(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("n_tokens", C.c_int32), ("n_sel", C.c_int32), ("n_chunks", C.c_int32),
                ("n_blocks", C.c_int32), ("sel", C.POINTER(C.c_int32)), ("tok", C.POINTER(C.c_int32)),
                ("src", C.POINTER(C.c_int32)), ("chunks", C.POINTER(C.c_int32)),
                ("block_table", C.POINTER(C.c_int32)), ("slot", C.POINTER(C.c_int32)),
                ("block_delta", C.POINTER(C.c_int32)), ("n_shared", C.c_int32)]


class DecodeResultC(C.Structure):
    _fields_ = [("logits", C.POINTER(C.c_float)), ("logits_dev", C.POINTER(C.c_float)), ("next_token", C.c_int32),
                ("n_tokens", C.c_int32)]


class ServeConfigC(C.Structure):
    _fields_ = [("n_users", C.c_int32), ("user_segs", C.c_void_p), ("user_n_segs", C.POINTER(C.c_int32)),
                ("rate", C.c_double), ("duration_s", C.c_double), ("seed", C.c_uint64), ("max_batch", C.c_int32),
                ("params", LinkParamsC)]


class ServeStatsC(C.Structure):
    _fields_ = [("n_requests", C.c_int64), ("n_completed", C.c_int64), ("n_batches", C.c_int64),
                ("elapsed_s", C.c_double), ("throughput_rps", C.c_double), ("ttft_mean_ms", C.c_double),
                ("ttft_p50_ms", C.c_double), ("ttft_p90_ms", C.c_double), ("ttft_p99_ms", C.c_double),
                ("ttft_max_ms", C.c_double), ("mean_batch", C.c_double), ("ccr", C.c_double),
                ("tokens_per_s", C.c_double)]


class StatsC(C.Structure):
    _fields_ = [("free_blocks", C.c_int64), ("total_blocks", C.c_int64), ("n_cached_chunks", C.c_int64),
                ("kernels_last_call", C.c_int64), ("graphs_cached", C.c_int64),
                ("h2d_bytes_last_call", C.c_int64), ("d2h_bytes_last_call", C.c_int64)]


class KernelStatC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("bytes", C.c_double),
                ("flops", C.c_double)]


# every symbol include/pic.h and include/pic_test.h declare
EXPORTS = ["pic_arena_bytes", "pic_engine_create", "pic_engine_destroy", "pic_generate_context_cache", "pic_link",
           "pic_link_batch", "pic_plan", "pic_linked_export", "pic_linked_info", "pic_linked_sharing", "pic_linked_materialize", "pic_linked_release",
           "pic_cache_export", "pic_cache_info", "pic_expire_cache", "pic_read_weights", "pic_get_stats",
           "pic_last_error", "pic_status_string", "pic_arena_bytes_tp", "pic_engine_create_tp", "pic_tp_ipc_handle",
           "pic_tp_connect", "pic_generate_context_cache_ex", "pic_decode", "pic_serve_poisson", "pic_serve_arrivals", "pic_set_profiling", "pic_get_profile", "pic_test_gemm", "pic_test_attention", "pic_test_attention_v", "pic_test_set_attention_kernel", "pic_test_last_attention_kernel", "pic_test_kv_link", "pic_bench_gemm", "pic_bench_attention", "pic_test_gemm_swiglu"]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2410_15332_b200.build` "
                              "(there is no fallback path)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.pic_last_error.restype = C.c_char_p
        L.pic_status_string.restype = C.c_char_p
        L.pic_arena_bytes.argtypes = [P(ModelConfigC), P(LimitsC), P(C.c_size_t)]
        L.pic_engine_create.argtypes = [P(ModelConfigC), P(LimitsC), C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p,
                                        P(C.c_void_p)]
        L.pic_arena_bytes_tp.argtypes = [P(ModelConfigC), P(LimitsC), C.c_int32, P(C.c_size_t)]
        L.pic_engine_create_tp.argtypes = [P(ModelConfigC), P(LimitsC), C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p,
                                           C.c_int32, C.c_int32, P(C.c_void_p)]
        L.pic_tp_ipc_handle.argtypes = [C.c_void_p, C.c_void_p, P(C.c_uint64)]
        L.pic_tp_connect.argtypes = [C.c_void_p, C.c_void_p, P(C.c_uint64)]
        L.pic_engine_destroy.argtypes = [C.c_void_p]
        L.pic_engine_destroy.restype = None
        L.pic_generate_context_cache.argtypes = [C.c_void_p, P(P(C.c_int32)), P(C.c_int32), C.c_int32, C.c_void_p,
                                                 P(C.c_uint64), P(C.c_int32)]
        L.pic_generate_context_cache_ex.argtypes = [C.c_void_p, P(P(C.c_int32)), P(C.c_int32), C.c_int32,
                                                    P(CompileOptionsC), C.c_void_p, P(C.c_uint64), P(C.c_int32)]
        L.pic_serve_poisson.argtypes = [C.c_void_p, P(ServeConfigC), C.c_void_p, P(ServeStatsC)]
        L.pic_serve_arrivals.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_uint64, P(C.c_double), P(C.c_int32),
                                         P(C.c_int32)]
        L.pic_decode.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32), C.c_int32, C.c_int32, C.c_void_p,
                                 P(DecodeResultC)]
        L.pic_link.argtypes = [C.c_void_p, P(SegmentC), C.c_int32, P(LinkParamsC), C.c_void_p, P(C.c_void_p),
                               P(LinkResultC)]
        L.pic_link_batch.argtypes = [C.c_void_p, C.c_int32, P(P(SegmentC)), P(C.c_int32), P(LinkParamsC), C.c_void_p,
                                     P(C.c_void_p), P(LinkResultC)]
        L.pic_plan.argtypes = [C.c_void_p, P(SegmentC), C.c_int32, P(LinkParamsC), P(PlanOutC)]
        L.pic_linked_export.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.pic_linked_info.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32), P(C.c_int32)]
        L.pic_linked_sharing.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32), P(C.c_int32)]
        if hasattr(L, "pic_linked_materialize") or "PIC_LIB_NAME" not in os.environ:  # older experiment builds lack it
            L.pic_linked_materialize.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.pic_linked_release.argtypes = [C.c_void_p, C.c_void_p]
        L.pic_cache_export.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p]
        L.pic_cache_info.argtypes = [C.c_void_p, C.c_uint64, P(C.c_int32), P(C.c_int32)]
        L.pic_expire_cache.argtypes = [C.c_void_p, C.c_uint64, P(C.c_int32)]
        L.pic_read_weights.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
        L.pic_get_stats.argtypes = [C.c_void_p, P(StatsC)]
        L.pic_set_profiling.argtypes = [C.c_void_p, C.c_int32]
        L.pic_get_profile.argtypes = [C.c_void_p, P(KernelStatC), C.c_int32, P(C.c_int32), C.c_int32]
        L.pic_test_gemm.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_void_p]
        L.pic_test_attention.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.pic_test_attention_v.argtypes = L.pic_test_attention.argtypes[:11] + [C.c_int32, C.c_int32, C.c_void_p]
        L.pic_test_set_attention_kernel.argtypes = [C.c_int32]
        L.pic_test_last_attention_kernel.argtypes = []
        L.pic_test_last_attention_kernel.restype = C.c_int32
        L.pic_test_kv_link.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32]
        L.pic_bench_gemm.argtypes = [C.c_int32] * 6 + [P(C.c_float)]
        L.pic_test_gemm_swiglu.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int32] * 4 + [C.c_void_p]
        L.pic_bench_attention.argtypes = [C.c_void_p] * 4 + [C.c_int32] * 4 + [C.c_void_p] + [C.c_int32] * 3 + [P(C.c_float)]
        for name in EXPORTS:
            if "PIC_LIB_NAME" not in os.environ or hasattr(L, name):  # experiment builds may predate a call
                getattr(L, name)  # AttributeError if the library lacks a declared entry point
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise PicError(status, lib().pic_last_error().decode(errors="replace"))


def _ptr(a: Optional[np.ndarray], ctype=C.c_int32):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


def config_struct(cfg) -> ModelConfigC:
    return ModelConfigC(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn_dim,
                        cfg.vocab, cfg.max_pos, cfg.bos_id, float(cfg.rope_theta), float(cfg.rms_eps),
                        int(cfg.seed), int(getattr(cfg, "dtype", 0)))


ALGS = {"naive": PIC_NAIVE, "fr": PIC_FULL, "legolink": PIC_LEGOLINK, "cacheblend": PIC_CACHEBLEND,
        "legolink0": PIC_LEGOLINK0}


def parse_alg(alg: str) -> Tuple[int, int, int]:
    """SPEC grammar -> (pic_algorithm, k, r_percent)."""
    if alg == "naive":
        return PIC_NAIVE, 0, 0
    if alg == "fr":
        return PIC_FULL, 0, 0
    if alg == "legolink0":
        return PIC_LEGOLINK0, 0, 0
    name, _, val = alg.partition(":")
    if name == "legolink":
        return PIC_LEGOLINK, int(val), 0
    if name == "cacheblend":
        return PIC_CACHEBLEND, 0, int(val)
    raise ValueError(f"unknown algorithm {alg!r}")


class _Segs:
    """Keeps the ctypes segment array and its token buffers alive for one call."""

    def __init__(self, segments):
        self.keep = []
        self.arr = (SegmentC * max(1, len(segments)))()
        self.n = len(segments)
        for i, (kind, val) in enumerate(segments):
            if kind == "cached":
                self.arr[i] = SegmentC(PIC_SEG_CACHED, 0, int(val), None)
            elif kind == "tokens":
                t = np.ascontiguousarray(val, dtype=np.int32)
                self.keep.append(t)
                self.arr[i] = SegmentC(PIC_SEG_TOKENS, len(t), 0, _ptr(t))
            else:
                raise ValueError(kind)


@dataclass
class LinkOutput:
    logits: Optional[np.ndarray]
    first_token: int
    n_tokens: int
    n_selected: int
    n_selected_layer0: int
    linked: Optional[int] = None          # opaque pic_linked* (release with Engine.release)
    selected: Optional[np.ndarray] = None # linked indices recomputed in the last layer
    hidden: Optional[np.ndarray] = None   # debug hidden [L][N][d]


def serve_arrivals(n_users: int, rate: float, duration_s: float, seed: int = 0x5E12E):
    """The Poisson arrival schedule pic_serve_poisson uses: (times [s], users)."""
    n = C.c_int32(0)
    st = lib().pic_serve_arrivals(n_users, rate, duration_s, seed, None, None, C.byref(n))
    if st not in (0, 4):
        check(st)
    t = np.zeros(max(1, n.value), dtype=np.float64)
    u = np.zeros(max(1, n.value), dtype=np.int32)
    check(lib().pic_serve_arrivals(n_users, rate, duration_s, seed, t.ctypes.data_as(C.POINTER(C.c_double)),
                                   u.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n)))
    return t[:n.value], u[:n.value]


@dataclass
class DecodeOutput:
    logits: Optional[np.ndarray]          # [n][vocab] fp32 (None unless requested)
    next_token: np.ndarray                # argmax per sequence (-1 without host output)
    n_tokens: np.ndarray                  # cache lengths after the step


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float32; float32 arrays (fp32 debug build) pass through."""
    if b.dtype == np.float32:
        return b
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


class Engine:
    """One engine = one model replica on one GPU (or a host-only planner when device=None)."""

    def __init__(self, cfg, num_blocks: int, max_rows: int, max_tokens: int, max_requests: int = 1,
                 device: Optional[int] = 0, stream=None, tp_rank: int = 0, tp_size: int = 1):
        L = lib()
        self.cfg = cfg
        self._cfg = config_struct(cfg)
        self._lim = LimitsC(num_blocks, max_rows, max_tokens, max_requests)
        self.max_tokens = max_tokens
        self.kv_share = 0  # default of pic_link_params.kv_share for this engine's calls: 0 copy, 1 shared-block
        #                    link (f3), 2 V by reference with re-based key copies
        self._h = C.c_void_p()
        self.arena = None
        self.device = device
        if device is None:
            check(L.pic_engine_create(C.byref(self._cfg), C.byref(self._lim), -1, None, 0, None, C.byref(self._h)))
            self.stream = None
            return
        import torch
        nbytes = C.c_size_t()
        self.tp_rank, self.tp_size = tp_rank, tp_size
        check(L.pic_arena_bytes_tp(C.byref(self._cfg), C.byref(self._lim), tp_size, C.byref(nbytes)))
        torch.cuda.set_device(device)
        self.arena = torch.empty(nbytes.value, dtype=torch.uint8, device=f"cuda:{device}")
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        check(L.pic_engine_create_tp(C.byref(self._cfg), C.byref(self._lim), device,
                                     C.c_void_p(self.arena.data_ptr()), nbytes.value,
                                     C.c_void_p(self.stream.cuda_stream), tp_rank, tp_size, C.byref(self._h)))

    def ipc_handle(self) -> Tuple[bytes, int]:
        h = (C.c_char * 64)()
        off = C.c_uint64()
        check(lib().pic_tp_ipc_handle(self._h, h, C.byref(off)))
        return bytes(h), off.value

    def tp_connect(self, handles: Sequence[Tuple[bytes, int]]) -> None:
        """handles: every rank's (ipc_handle, offset) in rank order (e.g. from all_gather_object)."""
        buf = (C.c_char * (64 * len(handles)))()
        for r, (h, _) in enumerate(handles):
            C.memmove(C.addressof(buf) + 64 * r, h, 64)
        offs = (C.c_uint64 * len(handles))(*[o for _, o in handles])
        check(lib().pic_tp_connect(self._h, buf, offs))

    @property
    def _stream(self):
        return None if self.stream is None else C.c_void_p(self.stream.cuda_stream)

    def close(self):
        if self._h:
            lib().pic_engine_destroy(self._h)
            self._h = C.c_void_p()
        if self.arena is not None:
            import torch
            self.arena = None
            torch.cuda.empty_cache()   # hand the arena back to the device, not just to torch's cache

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ compile
    def generate_context_cache(self, chunks: Sequence[np.ndarray], dummy_prefix: int = 0,
                               dummy_token: int = -1) -> List[int]:
        """Compile (a0); dummy_prefix = m > 0 is the LegoLink-0 compile (pic_generate_context_cache_ex)."""
        arrs = [np.ascontiguousarray(c, dtype=np.int32) for c in chunks]
        n = len(arrs)
        ptrs = (C.POINTER(C.c_int32) * max(1, n))(*[_ptr(a) for a in arrs])
        lens = (C.c_int32 * max(1, n))(*[len(a) for a in arrs])
        ids = (C.c_uint64 * max(1, n))()
        err = C.c_int32(-1)
        if dummy_prefix:
            opts = CompileOptionsC(int(dummy_prefix), int(dummy_token))
            st = lib().pic_generate_context_cache_ex(self._h, ptrs, lens, n, C.byref(opts), self._stream, ids,
                                                     C.byref(err))
        else:
            st = lib().pic_generate_context_cache(self._h, ptrs, lens, n, self._stream, ids, C.byref(err))
        if st != 0:
            e = PicError(st, lib().pic_last_error().decode())
            e.err_index = err.value
            raise e
        return [int(ids[i]) for i in range(n)]

    # ------------------------------------------------------------------ link
    def _params(self, alg, check_layer=1, rebase=True, use_graph=True, sel_override=None, debug_hidden=None,
                kv_share=None):
        a, k, r = parse_alg(alg)
        share = self.kv_share if kv_share is None else kv_share
        p = LinkParamsC(a, k, r, check_layer, int(rebase), int(use_graph), None, 0, None, int(share))
        keep = []
        if sel_override is not None:
            so = np.ascontiguousarray(sel_override, dtype=np.int32)
            keep.append(so)
            p.sel_override = _ptr(so)
            p.n_sel_override = len(so)
        if debug_hidden is not None:
            p.debug_hidden = debug_hidden.ctypes.data_as(C.POINTER(C.c_float))
        return p, keep

    def link(self, segments, alg: str, *, check_layer: int = 1, rebase: bool = True, use_graph: bool = True,
             want_logits: bool = True, logits_dev=None, keep_linked: bool = False, sel_override=None,
             debug_hidden: bool = False, want_selected: bool = False, kv_share: Optional[int] = None) -> LinkOutput:
        segs = _Segs(segments)
        hid = None
        N = self.plan(segments, alg)["n_tokens"] if (debug_hidden or want_selected) else 0
        if debug_hidden:
            hid = np.full((self.cfg.n_layers, N, self.cfg.d_model), np.nan, dtype=np.float32)
        p, keep = self._params(alg, check_layer, rebase, use_graph, sel_override, hid, kv_share)
        res = LinkResultC()
        logits = None
        if want_logits:
            logits = np.empty(self.cfg.vocab, dtype=np.float32)
            res.logits = _ptr(logits, C.c_float)
        if logits_dev is not None:
            res.logits_dev = C.c_void_p(logits_dev.data_ptr())
        sel = None
        if want_selected:
            sel = np.full(N, -1, dtype=np.int32)
            res.selected = _ptr(sel)
        linked = C.c_void_p()
        check(lib().pic_link(self._h, segs.arr, segs.n, C.byref(p), self._stream,
                             C.byref(linked) if keep_linked else None, C.byref(res)))
        return LinkOutput(logits, res.first_token, res.n_tokens, res.n_selected, res.n_selected_layer0,
                          linked.value if keep_linked else None, sel[:res.n_selected] if sel is not None else None,
                          hid)

    def link_batch(self, requests, alg: str, *, use_graph: bool = True, want_logits: bool = True,
                   keep_linked: bool = False, kv_share: Optional[int] = None,
                   debug_hidden: bool = False, logits_out: Optional[np.ndarray] = None,
                   logits_dev=None) -> List[LinkOutput]:
        """Batched link (pic_link_batch).  debug_hidden: every output's .hidden is the forward's
        [L][R][d] residual array (R = max(N_0, Σ k'); request r's rows follow those of requests < r,
        in selected order, see pic.h).  logits_out: caller-owned float32 [n][vocab] C-contiguous host array
        to receive the logits (page-locked memory, e.g. a pinned torch tensor's .numpy(), is filled by one
        direct device-to-host copy); the outputs' .logits are views of it.  logits_dev: a device fp32 [n][vocab]
        tensor (or its address) filled on the stream; with want_logits=False the call then does not synchronise
        (first tokens stay on the device), so consecutive calls run back to back."""
        n = len(requests)
        segs = [_Segs(r) for r in requests]
        arrp = (C.POINTER(SegmentC) * n)(*[C.cast(s.arr, C.POINTER(SegmentC)) for s in segs])
        ns = (C.c_int32 * n)(*[s.n for s in segs])
        hid = None
        if debug_hidden:
            plans = [self.plan(r, alg, kv_share=kv_share) for r in requests]
            R = max(plans[0]["n_tokens"], sum(len(q["sel"]) for q in plans))
            hid = np.full((self.cfg.n_layers, R, self.cfg.d_model), np.nan, dtype=np.float32)
        p, keep = self._params(alg, use_graph=use_graph, kv_share=kv_share, debug_hidden=hid)
        res = (LinkResultC * n)()
        logits = None
        if want_logits:
            if logits_out is not None:
                if (logits_out.dtype != np.float32 or logits_out.shape != (n, self.cfg.vocab)
                        or not logits_out.flags["C_CONTIGUOUS"]):
                    raise ValueError("logits_out must be a C-contiguous float32 [n][vocab] array")
                logits = logits_out
            else:
                logits = np.empty((n, self.cfg.vocab), dtype=np.float32)
            for i in range(n):
                res[i].logits = logits[i].ctypes.data_as(C.POINTER(C.c_float))
        if logits_dev is not None:
            base = int(logits_dev.data_ptr()) if hasattr(logits_dev, "data_ptr") else int(logits_dev)
            for i in range(n):
                res[i].logits_dev = C.c_void_p(base + 4 * i * self.cfg.vocab)
        linked = (C.c_void_p * n)()
        check(lib().pic_link_batch(self._h, n, arrp, ns, C.byref(p), self._stream, linked if keep_linked else None,
                                   res))
        return [LinkOutput(None if logits is None else logits[i], res[i].first_token, res[i].n_tokens,
                           res[i].n_selected, res[i].n_selected_layer0, linked[i] if keep_linked else None,
                           hidden=hid)
                for i in range(n)]

    def decode(self, linked: Sequence[int], tokens: Sequence[int], *, use_graph: bool = True,
               want_logits: bool = True, logits_dev=None) -> "DecodeOutput":
        """One decode step over live linked caches (pic_decode): tokens[b] is appended to linked[b].
        logits_dev: optional device pointer (int) of an fp32 [n][vocab] buffer filled on the stream."""
        n = len(linked)
        hs = (C.c_void_p * n)(*[int(h) for h in linked])
        toks = (C.c_int32 * n)(*[int(t) for t in tokens])
        res = (DecodeResultC * n)()
        logits = None
        if want_logits:
            logits = np.empty((n, self.cfg.vocab), dtype=np.float32)
            for i in range(n):
                res[i].logits = logits[i].ctypes.data_as(C.POINTER(C.c_float))
        if logits_dev is not None:
            for i in range(n):
                res[i].logits_dev = C.cast(C.c_void_p(int(logits_dev) + 4 * i * self.cfg.vocab), C.POINTER(C.c_float))
        check(lib().pic_decode(self._h, hs, toks, n, int(use_graph), self._stream, res))
        return DecodeOutput(logits, np.array([res[i].next_token for i in range(n)], dtype=np.int64),
                            np.array([res[i].n_tokens for i in range(n)], dtype=np.int64))

    def serve_poisson(self, requests, alg: str, rate: float, duration_s: float, *, seed: int = 0x5E12E,
                      max_batch: Optional[int] = None, check_layer: int = 1, use_graph: bool = False,
                      kv_share: Optional[int] = None) -> dict:
        """Open-loop Poisson serving (pic_serve_poisson, f4): user u resends requests[u] at rate/len(requests).
        Eager launches by default: batch compositions vary, so per-shape graphs would be captured per call."""
        n = len(requests)
        segs = [_Segs(r) for r in requests]
        arrp = (C.POINTER(SegmentC) * n)(*[C.cast(x.arr, C.POINTER(SegmentC)) for x in segs])
        ns = (C.c_int32 * n)(*[x.n for x in segs])
        p, keep = self._params(alg, check_layer=check_layer, use_graph=use_graph, kv_share=kv_share)
        cfgc = ServeConfigC(n, C.cast(arrp, C.c_void_p), ns, float(rate), float(duration_s), int(seed),
                            int(max_batch or self._lim.max_requests), p)
        out = ServeStatsC()
        check(lib().pic_serve_poisson(self._h, C.byref(cfgc), self._stream, C.byref(out)))
        return {k: getattr(out, k) for k, _ in ServeStatsC._fields_}

    def plan(self, segments, alg: str, kv_share: Optional[int] = None) -> dict:
        segs = _Segs(segments)
        p, _ = self._params(alg, kv_share=kv_share)
        cap = self.max_tokens
        names = ("sel", "tok", "src", "chunks", "block_table", "slot", "block_delta")
        bufs = {k: np.zeros(n * cap, dtype=np.int32) for k, n in
                (("sel", 1), ("tok", 1), ("src", 2), ("chunks", 3), ("block_table", 1), ("slot", 1),
                 ("block_delta", 1))}
        out = PlanOutC(cap, 0, 0, 0, 0, *[_ptr(bufs[k]) for k in names], 0)
        check(lib().pic_plan(self._h, segs.arr, segs.n, C.byref(p), C.byref(out)))
        N, ns, nc, nb = out.n_tokens, out.n_sel, out.n_chunks, out.n_blocks
        return {"n_tokens": N, "sel": bufs["sel"][:ns].copy(), "tok": bufs["tok"][:N].copy(),
                "src": bufs["src"][:2 * N].reshape(N, 2).copy(), "chunks": bufs["chunks"][:3 * nc].reshape(nc, 3).copy(),
                "block_table": bufs["block_table"][:nb].copy(), "slot": bufs["slot"][:ns].copy(),
                "block_delta": bufs["block_delta"][:nb].copy(), "n_shared": out.n_shared}

    # ------------------------------------------------------------------ exports / lifecycle
    @property
    def kv_dtype(self):
        """uint16 (bf16 bits) for the product, float32 for the fp32 debug build."""
        return np.float32 if int(getattr(self.cfg, "dtype", 0)) == 1 else np.uint16

    @property
    def local_kv_heads(self) -> int:
        return self.cfg.n_kv_heads // getattr(self, "tp_size", 1)

    def linked_export(self, linked: int, layer: int) -> Tuple[np.ndarray, np.ndarray]:
        n = C.c_int32()
        check(lib().pic_linked_info(self._h, C.c_void_p(linked), C.byref(n), None))
        shape = (n.value, self.local_kv_heads, self.cfg.head_dim)
        k = np.empty(shape, dtype=self.kv_dtype)
        v = np.empty(shape, dtype=self.kv_dtype)
        check(lib().pic_linked_export(self._h, C.c_void_p(linked), layer, k.ctypes.data, v.ctypes.data))
        return k, v

    def linked_blocks(self, linked: int) -> np.ndarray:
        n = C.c_int32()
        check(lib().pic_linked_info(self._h, C.c_void_p(linked), C.byref(n), None))
        bt = np.zeros((n.value + 15) // 16, dtype=np.int32)
        check(lib().pic_linked_info(self._h, C.c_void_p(linked), C.byref(n), _ptr(bt)))
        return bt

    def linked_sharing(self, linked: int) -> Tuple[int, np.ndarray]:
        """(blocks linked by reference, per-block Δ) of a shared-block link (kv_share, f3)."""
        n = C.c_int32()
        check(lib().pic_linked_info(self._h, C.c_void_p(linked), C.byref(n), None))
        bd = np.zeros((n.value + 15) // 16, dtype=np.int32)
        ns = C.c_int32()
        check(lib().pic_linked_sharing(self._h, C.c_void_p(linked), C.byref(ns), _ptr(bd)))
        return ns.value, bd

    def materialize(self, linked: int) -> None:
        """Copy + re-base the shared chunk-store blocks of a kv_share linked cache into owned blocks."""
        check(lib().pic_linked_materialize(self._h, C.c_void_p(linked), self._stream))

    def release(self, linked: int) -> None:
        check(lib().pic_linked_release(self._h, C.c_void_p(linked)))

    def cache_export(self, cid: int, layer: int) -> Tuple[np.ndarray, np.ndarray]:
        n = C.c_int32()
        check(lib().pic_cache_info(self._h, cid, C.byref(n), None))
        shape = (n.value, self.local_kv_heads, self.cfg.head_dim)
        k = np.empty(shape, dtype=self.kv_dtype)
        v = np.empty(shape, dtype=self.kv_dtype)
        check(lib().pic_cache_export(self._h, cid, layer, k.ctypes.data, v.ctypes.data))
        return k, v

    def cache_blocks(self, cid: int) -> np.ndarray:
        n = C.c_int32()
        check(lib().pic_cache_info(self._h, cid, C.byref(n), None))
        b = np.zeros((n.value + 15) // 16, dtype=np.int32)
        check(lib().pic_cache_info(self._h, cid, C.byref(n), _ptr(b)))
        return b

    def expire(self, cid: int) -> bool:
        w = C.c_int32()
        check(lib().pic_expire_cache(self._h, cid, C.byref(w)))
        return bool(w.value)

    def read_weights(self, which: int, layer: int = 0, row0: int = 0, nrows: int = 1) -> np.ndarray:
        c = self.cfg
        if which >= 9:
            out = np.empty(c.d_model, dtype=np.float32)
        else:
            cols = {0: c.d_model, 1: c.d_model, 2: c.d_model, 3: c.n_heads * c.head_dim, 4: c.d_model,
                    5: c.d_model, 6: c.ffn_dim, 7: c.d_model, 8: c.d_model}[which]
            out = np.empty((nrows, cols), dtype=np.uint16)
        check(lib().pic_read_weights(self._h, which, layer, row0, nrows, out.ctypes.data))
        return out

    def set_profiling(self, on: bool) -> None:
        check(lib().pic_set_profiling(self._h, int(on)))

    def profile(self, reset: bool = True) -> dict:
        arr = (KernelStatC * 64)()
        n = C.c_int32()
        check(lib().pic_get_profile(self._h, arr, 64, C.byref(n), int(reset)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].ms, "bytes": arr[i].bytes,
                                       "flops": arr[i].flops} for i in range(n.value)}

    def stats(self) -> dict:
        s = StatsC()
        check(lib().pic_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in StatsC._fields_}


# ---------------------------------------------------------------------------- kernel test hooks
def test_gemm(A: np.ndarray, B: np.ndarray, bn: int = 128, splits: int = 1) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint16)
    B = np.ascontiguousarray(B, dtype=np.uint16)
    M, K = A.shape
    N = B.shape[0]
    out = np.empty((M, N), dtype=np.float32)
    check(lib().pic_test_gemm(A.ctypes.data, B.ctypes.data, M, N, K, bn, splits, out.ctypes.data))
    return out


def test_gemm_swiglu(A: np.ndarray, B: np.ndarray, bn: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint16)
    B = np.ascontiguousarray(B, dtype=np.uint16)
    M, K = A.shape
    N2 = B.shape[0]
    u = np.empty((M, N2 // 2), dtype=np.uint16)
    check(lib().pic_test_gemm_swiglu(A.ctypes.data, B.ctypes.data, M, N2, K, bn, u.ctypes.data))
    return u


def last_attention_kernel() -> int:
    """Test hook: the attention kernel the last forward launched (see pic_test.h)."""
    return int(lib().pic_test_last_attention_kernel())


def set_attention_kernel(version: int) -> None:
    """0 = engine's choice, 1 = one q-tile per CTA, 2 = ping-pong (tests / A/B only)."""
    check(lib().pic_test_set_attention_kernel(version))


def test_attention(Q, K, V, pos, block_perm, num_blocks, n_splits=1, version=2, grid=0) -> np.ndarray:
    Q = np.ascontiguousarray(Q, dtype=np.uint16)
    K = np.ascontiguousarray(K, dtype=np.uint16)
    V = np.ascontiguousarray(V, dtype=np.uint16)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    bp = np.ascontiguousarray(block_perm, dtype=np.int32)
    M, Hq, D = Q.shape
    n, Hkv, _ = K.shape
    O = np.empty((M, Hq, D), dtype=np.uint16)
    check(lib().pic_test_attention_v(Q.ctypes.data, K.ctypes.data, V.ctypes.data, pos.ctypes.data, M, n, Hq, Hkv,
                                     bp.ctypes.data, num_blocks, n_splits, version, grid, O.ctypes.data))
    return O


def test_kv_link(Kpool, Vpool, src, dst, delta, layer0=0, rebase=True, theta=1e4, max_pos=4096):
    Kpool = np.ascontiguousarray(Kpool, dtype=np.uint16)
    Vpool = np.ascontiguousarray(Vpool, dtype=np.uint16)
    L, NB, Hkv, _, D = Kpool.shape
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    delta = np.ascontiguousarray(delta, dtype=np.int32)
    check(lib().pic_test_kv_link(Kpool.ctypes.data, Vpool.ctypes.data, L, NB, Hkv, D, src.ctypes.data,
                                 dst.ctypes.data, delta.ctypes.data, len(src), layer0, int(rebase), theta, max_pos))
    return Kpool, Vpool


def bench_gemm(M, N, K, bn, splits, iters=50) -> float:
    us = C.c_float()
    check(lib().pic_bench_gemm(M, N, K, bn, splits, iters, C.byref(us)))
    return us.value


def bench_attention(Q, K, V, pos, block_perm, num_blocks, n_splits=1, iters=20) -> float:
    Q = np.ascontiguousarray(Q, dtype=np.uint16)
    K = np.ascontiguousarray(K, dtype=np.uint16)
    V = np.ascontiguousarray(V, dtype=np.uint16)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    bp = np.ascontiguousarray(block_perm, dtype=np.int32)
    M, Hq, D = Q.shape
    n, Hkv, _ = K.shape
    us = C.c_float()
    check(lib().pic_bench_attention(Q.ctypes.data, K.ctypes.data, V.ctypes.data, pos.ctypes.data, M, n, Hq, Hkv,
                                    bp.ctypes.data, num_blocks, n_splits, iters, C.byref(us)))
    return us.value
