"""B200-native Pre^3 constrained-decoding hot path (arxiv 2506.03887).

Python host mirror of the reference matcher's runtime API
(`gmask::Engine`, /root/reference/proj/include/gmask/runtime.hpp:92-166) over
the C ABI in include/pre3_gmask.h, implemented by the in-tree CUDA library
``libpre3gmask.so`` (sm_100a).  There is no CPU fallback: if the library is
missing, importing the binding raises.

The batched device API (`DeviceEngine`, `Batch`) is the product; the
single-sequence `Engine`-named helpers (`InitialConfig`, `Step`,
`ComputeMask`) exist so parity tests read like the reference's own
(tests/test_runtime.cpp) — each call runs the CUDA kernels on a batch of one.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRE3_GMASK_LIB") or os.path.join(_HERE, "libpre3gmask.so")  # override: experiments only

GM_OK = 0
GM_ERR_GRAMMAR = 2
GM_ERR_BUILD = 3
GM_ERR_CORRUPT_INPUT = 4
GM_ERR_CUDA = 5
GM_ERR_STACK_OVERFLOW = 6
GM_ERR_VOCAB_EMPTY = 7
GM_ERR_VOCAB_DUPLICATE = 8
GM_ERR_SNAPSHOT_MISMATCH = 9
GM_ERR_USAGE = 64

ALIVE, DEAD, ACCEPTED, OVERFLOW = 0, 1, 2, 3
END_MARKER = 256  # grammar.hpp:28 kEndMarker


class GmError(RuntimeError):
    """Maps a gm_status_code to the reference's exception kinds."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class GrammarError(GmError):
    pass


class BuildError(GmError):
    pass


class SerializeError(GmError):
    pass


class VocabError(GmError):
    """runtime.hpp:29-37; .kind is 'empty' or 'duplicate'."""

    @property
    def kind(self) -> str:
        return "empty" if self.code == GM_ERR_VOCAB_EMPTY else "duplicate"


class CudaError(GmError):
    pass


class StackOverflowError(GmError):
    pass


class SnapshotMismatchError(GmError):
    """A context snapshot taken for another automaton / vocabulary / K, R, slots."""


_ERRORS = {
    GM_ERR_GRAMMAR: GrammarError,
    GM_ERR_BUILD: BuildError,
    GM_ERR_CORRUPT_INPUT: SerializeError,
    GM_ERR_CUDA: CudaError,
    GM_ERR_STACK_OVERFLOW: StackOverflowError,
    GM_ERR_VOCAB_EMPTY: VocabError,
    GM_ERR_VOCAB_DUPLICATE: VocabError,
    GM_ERR_SNAPSHOT_MISMATCH: SnapshotMismatchError,
}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libpre3gmask.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; run __graft_entry__.build() "
                "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, U64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
        PP = ctypes.POINTER(ctypes.c_void_p)
        sigs = {
            "gm_last_error": ([], ctypes.c_char_p),
            "gm_abi_version": ([], ctypes.c_int),
            "gm_automaton_load": ([P, SZ, PP], ctypes.c_int),
            "gm_automaton_compile": ([ctypes.c_char_p, ctypes.c_int, ctypes.c_int, PP], ctypes.c_int),
            "gm_automaton_save": ([P, P, SZ, ctypes.POINTER(SZ)], ctypes.c_int),
            "gm_automaton_destroy": ([P], ctypes.c_int),
            "gm_automaton_info": ([P, P], ctypes.c_int),
            "gm_automaton_compile_stats": ([P, P], ctypes.c_int),
            "gm_automaton_save_gmaskdp1": ([P, P, SZ, ctypes.POINTER(SZ)], ctypes.c_int),
            "gm_vocab_load_json": ([P, SZ, P, I64, P, I32, ctypes.POINTER(I32), ctypes.POINTER(I64)], ctypes.c_int),
            "gm_engine_create": ([P, P, P, I32, P, ctypes.c_int, PP], ctypes.c_int),
            "gm_engine_destroy": ([P], ctypes.c_int),
            "gm_engine_info": ([P, P], ctypes.c_int),
            "gm_engine_set_structural": ([P, P], ctypes.c_int),
            "gm_engine_prewarm": ([P, I32, I32, U64, I32, P], ctypes.c_int),
            "gm_engine_snapshot_save": ([P, P, U64, ctypes.POINTER(U64)], ctypes.c_int),
            "gm_engine_evict": ([P, P], ctypes.c_int),
            "gm_engine_cache_stats": ([P, P], ctypes.c_int),
            "gm_engine_snapshot_load": ([P, P, U64], ctypes.c_int),
            "gm_batch_create": ([P, I32, I32, PP], ctypes.c_int),
            "gm_batch_destroy": ([P], ctypes.c_int),
            "gm_batch_reset": ([P, P], ctypes.c_int),
            "gm_batch_download": ([P, I32, P, P, P, I32, P], ctypes.c_int),
            "gm_batch_upload": ([P, I32, I32, P, I32], ctypes.c_int),
            "gm_batch_check": ([P, P], ctypes.c_int),
            "gm_batch_split_step_launches": ([P], ctypes.c_int),
            "gm_batch_counters": ([P, P], ctypes.c_int),
            "gm_batch_fill_stats": ([P, P], ctypes.c_int),
            "gm_batch_set_stats": ([P, I32], ctypes.c_int),
            "gm_batch_set_trace": ([P, P, I32], ctypes.c_int),
            "gm_fill_next_token_bitmask": ([P, P, I64, P], ctypes.c_int),
            "gm_fill_and_mask_logits": ([P, P, I64, P, I64, P, P], ctypes.c_int),
            "gm_accept_tokens": ([P, P, P, I32, P], ctypes.c_int),
            "gm_allowed_terminals": ([P, P, P], ctypes.c_int),
            "gm_sample_stream_and_accept": ([P, P, I64, P, U64, P, P], ctypes.c_int),
            "gm_sample_stream": ([P, P, I64, P, U64, P, P], ctypes.c_int),
            "gm_decode_step_stream": ([P, P, I64, P, I64, U64, P, P], ctypes.c_int),
            "gm_decode_step_stream_split": ([P, P, I64, P, I64, P, U64, P, P], ctypes.c_int),
            "gm_batch_time_next_fill": ([P, P, P], ctypes.c_int),
            "gm_decode_step_greedy": ([P, P, I64, P, I64, P, P], ctypes.c_int),
            "gm_decode_graph_create": ([P, I32, I32, P, I64, P, I64, P, U64, P, PP], ctypes.c_int),
            "gm_graph_launch": ([P, P], ctypes.c_int),
            "gm_graph_destroy": ([P], ctypes.c_int),
            "gm_sample_tokens": ([P, P, I64, P, I64, ctypes.c_float, I32, ctypes.c_float, U64, P, I32, P],
                                 ctypes.c_int),
            "gm_decode_step_sample": ([P, P, I64, P, I64, ctypes.c_float, I32, ctypes.c_float, U64, P, P],
                                      ctypes.c_int),
            "gmw_synth_vocab": ([I32, I32, P, I64, P], I64),
            "gmw_structural_words": ([P, P, I32, P], I32),
            "gmw_synth_logits": ([P, I64, I32, I32, I32, I32, U64, P], I32),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != GM_OK:
        msg = lib().gm_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, GmError)(rc, msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------- vocab
def synth_vocab(num_tokens: int, flavor: int = 0) -> List[bytes]:
    """Synthetic sorted vocabulary (acceptance_main.cpp:341-359, extended)."""
    L = lib()
    n = L.gmw_synth_vocab(num_tokens, flavor, None, 0, None)
    if n < 0:
        raise ValueError("bad vocabulary size")
    buf = np.zeros(max(n, 1), np.uint8)
    offs = np.zeros(num_tokens + 1, np.int64)
    L.gmw_synth_vocab(num_tokens, flavor, _ptr(buf), n, _ptr(offs))
    raw = buf.tobytes()
    return [raw[offs[i]:offs[i + 1]] for i in range(num_tokens)]


def synth_logits(dst, k: int, seed: int, row0: int = 0, stream=None) -> None:
    """Fills a bf16 CUDA tensor [rows, >=cols] with config 5's synthetic
    logits of rotating buffer k (gmw_synth_logits; the CPU reference arm
    generates the same values, oracle/gmask_port.c gp_synth_logit)."""
    rows, cols = dst.shape
    if lib().gmw_synth_logits(dst.data_ptr(), dst.stride(0), rows, cols, k, row0, seed & (2**64 - 1),
                              _stream(stream)) != 0:
        raise GmError(GM_ERR_USAGE, "gmw_synth_logits failed")


def pack_vocab(tokens: Sequence[bytes]):
    """(bytes uint8[], offsets int64[V+1]) host arrays."""
    offs = np.zeros(len(tokens) + 1, np.int64)
    np.cumsum([len(t) for t in tokens], out=offs[1:])
    data = np.frombuffer(b"".join(tokens), np.uint8).copy() if tokens else np.zeros(1, np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    return data, offs


def load_vocabulary(data: bytes) -> List[bytes]:
    """LoadVocabulary (serialize.cpp:348-364): JSON array of strings with
    `\\xNN` / `\\\\` unescaping (raises SerializeError like the reference)."""
    L = lib()
    n, total = ctypes.c_int32(), ctypes.c_int64()
    src = ctypes.create_string_buffer(data, len(data))
    _check(L.gm_vocab_load_json(src, len(data), None, 0, None, 0, ctypes.byref(n), ctypes.byref(total)))
    buf = np.zeros(max(1, total.value), np.uint8)
    offs = np.zeros(n.value + 1, np.int64)
    _check(L.gm_vocab_load_json(src, len(data), _ptr(buf), total.value, _ptr(offs), n.value, ctypes.byref(n),
                                ctypes.byref(total)))
    raw = buf.tobytes()
    return [raw[offs[i]:offs[i + 1]] for i in range(n.value)]


def escape_token(tok: bytes) -> str:
    """EscapeToken (serialize.cpp:298-313): backslash and every byte outside
    printable ASCII as \\xNN; inverse of the vocabulary unescape."""
    out = []
    for b in tok:
        if b == 0x5C:
            out.append("\\\\")
        elif 0x20 <= b <= 0x7E:
            out.append(chr(b))
        else:
            out.append("\\x%02x" % b)
    return "".join(out)


def structural_words(tokens: Sequence[bytes]) -> np.ndarray:
    data, offs = pack_vocab(tokens)
    words = np.zeros((len(tokens) + 1 + 31) // 32, np.uint32)
    lib().gmw_structural_words(_ptr(data), _ptr(offs), len(tokens), _ptr(words))
    return words


# --------------------------------------------------------------------- automaton
class Automaton:
    """A compiled DPDA (gmask::Dpda, dpda.hpp:97-124) held by the library."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @classmethod
    def load(cls, data: bytes) -> "Automaton":
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(data, len(data))
        _check(lib().gm_automaton_load(buf, len(data), ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def load_file(cls, path: str) -> "Automaton":
        with open(path, "rb") as f:
            return cls.load(f.read())

    @classmethod
    def compile(cls, grammar_text: str, aggregate: bool = True, merge: bool = True) -> "Automaton":
        h = ctypes.c_void_p()
        _check(lib().gm_automaton_compile(grammar_text.encode(), int(aggregate), int(merge), ctypes.byref(h)))
        return cls(h.value)

    def save(self) -> bytes:
        n = ctypes.c_size_t()
        _check(lib().gm_automaton_save(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().gm_automaton_save(self._h, buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    def info(self) -> dict:
        out = np.zeros(8, np.int64)
        _check(lib().gm_automaton_info(self._h, _ptr(out)))
        keys = ["num_states", "num_edges", "initial_state", "accept_state", "max_match_pop",
                "max_push", "dynamic_edges", "grammar_hash"]
        return dict(zip(keys, (int(x) for x in out)))

    def save_gmaskdp1(self) -> bytes:
        """SerializeDpda (serialize.cpp:148-196): the reference's GMASKDP1 bytes."""
        n = ctypes.c_size_t()
        _check(lib().gm_automaton_save_gmaskdp1(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().gm_automaton_save_gmaskdp1(self._h, buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    def compile_stats(self) -> dict:
        out = np.zeros(4, np.int64)
        _check(lib().gm_automaton_compile_stats(self._h, _ptr(out)))
        return {"composites": int(out[0]), "cycles": int(out[1])}

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.gm_automaton_destroy(self._h)
            self._h = ctypes.c_void_p()


class _EngineOptions(ctypes.Structure):
    _fields_ = [("context_depth", ctypes.c_int32), ("context_slots", ctypes.c_int32),
                ("parent_depth", ctypes.c_int64), ("segment_words", ctypes.c_int32),
                ("num_columns", ctypes.c_int32), ("eos_column", ctypes.c_int32),
                ("disabled", ctypes.c_void_p), ("auto_evict_free", ctypes.c_int32)]


@dataclass
class RuntimeConfig:
    """runtime.hpp:23-27 (state, status, stack bottom-first)."""
    state: int
    status: int
    stack: List[int] = field(default_factory=list)


class DeviceEngine:
    """Engine::Engine + TokenTrie::Build on one CUDA device (runtime.cpp:18-113)."""

    def __init__(self, automaton: Automaton, tokens: Sequence[bytes], device: int = 0,
                 context_depth: int = 8, context_slots: int = 8192, parent_depth: int = 0,
                 num_columns: int = 0, eos_column: int = 0, disabled: Optional[Sequence[int]] = None,
                 auto_evict_free: int = 0):
        """num_columns / eos_column / disabled: the model's logit layout
        (gm_engine_options; tokenizer.TokenizerVocab.engine_options() fills
        them from a tokenizer.json): logit rows have num_columns columns, EOS
        is column eos_column, other columns >= V are specials (-inf), and the
        ids in `disabled` (< V) are never allowed."""
        self.automaton = automaton
        self.tokens = list(tokens)
        self.V = len(self.tokens)
        self.W = (self.V + 1 + 31) // 32
        self.device = device
        self.num_columns = num_columns if num_columns > 0 else self.V + 1
        self.eos_column = eos_column if num_columns > 0 else self.V
        self.disabled_words = np.zeros(self.W, np.uint32)
        for i in disabled or ():
            if not 0 <= i < self.V:
                raise ValueError(f"disabled id {i} out of range")
            self.disabled_words[i >> 5] |= np.uint32(1 << (i & 31))
        data, offs = pack_vocab(self.tokens)
        opts = _EngineOptions(context_depth, context_slots, parent_depth, 256, num_columns, eos_column,
                              self.disabled_words.ctypes.data if disabled else None, auto_evict_free)
        h = ctypes.c_void_p()
        _check(lib().gm_engine_create(automaton._h, _ptr(data), _ptr(offs), self.V, ctypes.byref(opts),
                                      device, ctypes.byref(h)))
        self._h = h
        self.structural = structural_words(self.tokens) & ~self.disabled_words
        _check(lib().gm_engine_set_structural(self._h, _ptr(self.structural)))
        self._single: Optional[Batch] = None

    def set_structural(self, words: np.ndarray) -> None:
        """Replaces the sampler's structural token set (W uint32 words; the EOS
        bit is ignored); contexts built so far get their counts recomputed."""
        w = np.ascontiguousarray(words, dtype=np.uint32)
        if w.shape != (self.W,):
            raise ValueError(f"structural words must have shape ({self.W},)")
        _check(lib().gm_engine_set_structural(self._h, _ptr(w)))
        self.structural = w.copy()
        self.structural[self.V >> 5] &= np.uint32(~(1 << (self.V & 31)) & 0xFFFFFFFF)

    def info(self) -> dict:
        out = np.zeros(8, np.int64)
        _check(lib().gm_engine_info(self._h, _ptr(out)))
        keys = ["V", "W", "num_segments", "context_slots_used", "segment_builds", "private_builds",
                "parent_builds", "device"]
        return dict(zip(keys, (int(x) for x in out)))

    def prewarm(self, batch: int = 1024, steps: int = 200, seed: int = 0x5EED, stack_capacity: int = 1024,
                 stream=None) -> None:
        """Populates the context cache with synthetic decode streams (preprocessing)
        over sequences of the given stack capacity (overflow restarts them)."""
        _check(lib().gm_engine_prewarm(self._h, batch, steps, seed, stack_capacity, _stream(stream)))

    def evict(self, stream=None) -> None:
        """gm_engine_evict: frees context rows not referenced since the last
        eviction (every batch of the engine must be idle)."""
        _check(lib().gm_engine_evict(self._h, _stream(stream)))

    def cache_stats(self) -> dict:
        out = np.zeros(8, np.int64)
        _check(lib().gm_engine_cache_stats(self._h, _ptr(out)))
        keys = ["rows", "rows_in_use", "rows_free", "index_positions", "evictions", "rows_evicted",
                "private_builds", "segment_builds"]
        return dict(zip(keys, (int(x) for x in out)))

    def save_contexts(self, path: Optional[str] = None):
        """gm_engine_snapshot_save: the built context table ("P3GMCTX1") into
        `path` (written through a memory map), or returned as bytes."""
        size = ctypes.c_uint64()
        _check(lib().gm_engine_snapshot_save(self._h, None, 0, ctypes.byref(size)))
        if path is None:
            buf = np.empty(size.value, np.uint8)
        else:
            buf = np.memmap(path, np.uint8, "w+", shape=(max(size.value, 1),))
        _check(lib().gm_engine_snapshot_save(self._h, _ptr(buf), size.value, ctypes.byref(size)))
        if path is None:
            return buf.tobytes()
        buf.flush()
        del buf
        return size.value

    def load_contexts(self, source) -> None:
        """gm_engine_snapshot_load from a path or bytes (instead of a prewarm;
        the table must still be empty)."""
        if isinstance(source, (bytes, bytearray)):
            buf = np.frombuffer(source, np.uint8)
        else:
            buf = np.memmap(source, np.uint8, "r")
        _check(lib().gm_engine_snapshot_load(self._h, _ptr(buf) if buf.size else None, buf.size))

    def batch(self, size: int, stack_capacity: int = 1024) -> "Batch":
        return Batch(self, size, stack_capacity)

    # ---- reference-named single-sequence helpers (parity tests) ----
    def _one(self) -> "Batch":
        if self._single is None:
            self._single = Batch(self, 1, 4096)
        return self._single

    def InitialConfig(self) -> RuntimeConfig:
        s = self.automaton.info()["initial_state"]
        return RuntimeConfig(s, ALIVE, [s])

    def ComputeMask(self, cfg: RuntimeConfig) -> np.ndarray:
        """Engine::ComputeMask (runtime.cpp:280-287) via the CUDA fill kernel."""
        import torch
        b = self._one()
        b.set(0, cfg)
        out = torch.zeros((1, self.W), dtype=torch.int32, device=f"cuda:{self.device}")
        b.fill(out)
        b.check()
        return out.cpu().numpy().view(np.uint32)[0].copy()

    def AllowedTerminals(self, cfg: RuntimeConfig):
        """Engine::AllowedTerminals (runtime.cpp:188-208) -> (byte set as int, end_marker)."""
        import torch
        b = self._one()
        b.set(0, cfg)
        out = torch.zeros((1, 9), dtype=torch.int32, device=f"cuda:{self.device}")
        b.allowed_terminals(out)
        w = out.cpu().numpy().view(np.uint32)[0]
        byteset = 0
        for i in range(8):
            byteset |= int(w[i]) << (32 * i)
        return byteset, bool(w[8] & 1)

    def AcceptToken(self, cfg: RuntimeConfig, token: int) -> RuntimeConfig:
        """Engine::Step over the token's bytes (EOS = id V) via the accept kernel."""
        import torch
        b = self._one()
        b.set(0, cfg)
        toks = torch.tensor([token], dtype=torch.int32, device=f"cuda:{self.device}")
        b.accept(toks)
        b.check()
        return b.get(0)

    def __del__(self):
        self._single = None
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.gm_engine_destroy(self._h)
            self._h = ctypes.c_void_p()


def _dptr(t) -> Optional[int]:
    return t.data_ptr() if t is not None else None


_DTYPES = {"i32": ("int32",), "bf16": ("bfloat16",), "i32|u32": ("int32", "uint32")}


def _check_tensor(t, kind: str, what: str, rows: int, cols: int, device: int) -> None:
    """The kernels take raw pointers and leading dimensions: a tensor of the
    wrong dtype, device, row count or inner layout would be silently
    misread (or written out of bounds), so reject it here."""
    if t is None:
        return
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what}: expected a torch.Tensor")
    if not t.is_cuda or t.device.index != device:
        raise ValueError(f"{what}: must live on cuda:{device} (got {t.device})")
    if str(t.dtype).replace("torch.", "") not in _DTYPES[kind]:
        raise TypeError(f"{what}: dtype must be {'/'.join(_DTYPES[kind])} (got {t.dtype})")
    if t.dim() == 1:
        if cols > 1 or t.shape[0] < rows:
            raise ValueError(f"{what}: expected at least {rows} entries")
        if t.stride(0) != 1:
            raise ValueError(f"{what}: must be contiguous")
        return
    if t.dim() != 2 or t.shape[0] < rows or t.shape[1] < cols:
        raise ValueError(f"{what}: expected shape [>= {rows}, >= {cols}] (got {tuple(t.shape)})")
    if t.stride(1) != 1 or t.stride(0) < cols:
        raise ValueError(f"{what}: rows must be contiguous with a leading dimension >= {cols}")


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream


class StepGraph:
    """A captured CUDA graph of decode steps (gm_graph); launch() replays them."""

    def __init__(self, handle, batch, keep):
        self._h = handle
        self.batch = batch
        self._keep = keep  # the baked-in buffers must outlive the graph

    def launch(self, stream=None) -> None:
        _check(lib().gm_graph_launch(self._h, _stream(stream)))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.gm_graph_destroy(self._h)
            self._h = ctypes.c_void_p()


class Batch:
    """B in-flight sequences on the device (gm_batch)."""

    def __init__(self, engine: DeviceEngine, size: int, stack_capacity: int = 1024):
        self.engine = engine
        self.B = size
        self.cap = stack_capacity
        h = ctypes.c_void_p()
        _check(lib().gm_batch_create(engine._h, size, stack_capacity, ctypes.byref(h)))
        self._h = h
        self.nseg = engine.info()["num_segments"]

    def reset(self, stream=None):
        _check(lib().gm_batch_reset(self._h, _stream(stream)))

    def set(self, i: int, cfg: RuntimeConfig):
        st = np.asarray(cfg.stack, np.int32)
        _check(lib().gm_batch_upload(self._h, i, int(cfg.status), _ptr(st), len(st)))

    def get(self, i: int) -> RuntimeConfig:
        buf = np.zeros(self.cap, np.int32)
        state, status, depth = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().gm_batch_download(self._h, i, ctypes.byref(state), ctypes.byref(status), _ptr(buf),
                                       self.cap, ctypes.byref(depth)))
        return RuntimeConfig(state.value, status.value, buf[: depth.value].tolist())

    def _chk(self, bitmask=None, logits=None, seg_counts=None, tokens=None, out9=None):
        d = self.engine.device
        _check_tensor(bitmask, "i32|u32", "bitmask", self.B, self.engine.W, d)
        _check_tensor(logits, "bf16", "logits", self.B, self.engine.num_columns, d)
        _check_tensor(seg_counts, "i32", "seg_counts", self.B, 2 * self.nseg, d)
        _check_tensor(tokens, "i32", "tokens", self.B, 1, d)
        _check_tensor(out9, "i32|u32", "out", self.B, 9, d)

    def fill(self, bitmask, logits=None, seg_counts=None, stream=None):
        """bitmask: int32 CUDA tensor [B, >=W] (or None); logits: bf16 [B, >=V+1]."""
        self._chk(bitmask, logits, seg_counts)
        bm = bitmask.data_ptr() if bitmask is not None else None
        ldw = bitmask.stride(0) if bitmask is not None else 0
        lg = logits.data_ptr() if logits is not None else None
        ld = logits.stride(0) if logits is not None else 0
        sc = seg_counts.data_ptr() if seg_counts is not None else None
        _check(lib().gm_fill_and_mask_logits(self._h, bm, ldw, lg, ld, sc, _stream(stream)))

    def allowed_terminals(self, out, stream=None):
        """Engine::AllowedTerminals per sequence into out: int32 CUDA tensor [B, 9]."""
        self._chk(out9=out)
        _check(lib().gm_allowed_terminals(self._h, out.data_ptr(), _stream(stream)))

    def accept(self, tokens, status_out=None, restart: bool = False, stream=None):
        self._chk(tokens=tokens)
        self._chk(tokens=status_out)
        so = status_out.data_ptr() if status_out is not None else None
        _check(lib().gm_accept_tokens(self._h, tokens.data_ptr(), so, int(restart), _stream(stream)))

    def sample_stream_and_accept(self, bitmask, seg_counts, seed: int, tokens_out=None, stream=None):
        self._chk(bitmask, None, seg_counts, tokens_out)
        to = tokens_out.data_ptr() if tokens_out is not None else None
        _check(lib().gm_sample_stream_and_accept(self._h, bitmask.data_ptr(), bitmask.stride(0),
                                                 seg_counts.data_ptr(), seed, to, _stream(stream)))

    def sample_stream(self, bitmask, seg_counts, seed: int, tokens_out, stream=None):
        self._chk(bitmask, None, seg_counts, tokens_out)
        _check(lib().gm_sample_stream(self._h, bitmask.data_ptr(), bitmask.stride(0), seg_counts.data_ptr(), seed,
                                      tokens_out.data_ptr(), _stream(stream)))

    def decode_step_stream(self, seed: int, bitmask=None, logits=None, tokens_out=None, stream=None):
        """Fused fill + -inf logits + stream sample + accept (one launch)."""
        self._chk(bitmask, logits, None, tokens_out)
        bm = bitmask.data_ptr() if bitmask is not None else None
        ldw = bitmask.stride(0) if bitmask is not None else 0
        lg = logits.data_ptr() if logits is not None else None
        ld = logits.stride(0) if logits is not None else 0
        to = tokens_out.data_ptr() if tokens_out is not None else None
        _check(lib().gm_decode_step_stream(self._h, bm, ldw, lg, ld, seed, to, _stream(stream)))

    def decode_step_stream_split(self, seed: int, bitmask=None, logits=None, seg_counts=None, tokens_out=None,
                                 stream=None):
        """The same step as two overlapping kernels (gm_decode_step_stream_split)."""
        self._chk(bitmask, logits, seg_counts, tokens_out)
        bm = bitmask.data_ptr() if bitmask is not None else None
        ldw = bitmask.stride(0) if bitmask is not None else 0
        lg = logits.data_ptr() if logits is not None else None
        ld = logits.stride(0) if logits is not None else 0
        sc = seg_counts.data_ptr() if seg_counts is not None else None
        to = tokens_out.data_ptr() if tokens_out is not None else None
        _check(lib().gm_decode_step_stream_split(self._h, bm, ldw, lg, ld, sc, seed, to, _stream(stream)))

    def time_next_fill(self, start, end) -> None:
        """Brackets the next fill kernel (whatever call launches it) with two
        torch.cuda.Events (gm_batch_time_next_fill; created ones: record once first)."""
        _check(lib().gm_batch_time_next_fill(self._h, start.cuda_event, end.cuda_event))

    def decode_step_greedy(self, logits, tokens_out=None, bitmask=None, stream=None):
        self._chk(bitmask, logits, None, tokens_out)
        to = tokens_out.data_ptr() if tokens_out is not None else None
        bm = bitmask.data_ptr() if bitmask is not None else None
        ldw = bitmask.stride(0) if bitmask is not None else 0
        _check(lib().gm_decode_step_greedy(self._h, logits.data_ptr(), logits.stride(0), bm, ldw, to,
                                           _stream(stream)))

    def sample(self, logits, bitmask, temperature: float = 1.0, top_k: int = 0, top_p: float = 1.0, seed: int = 0,
               tokens_out=None, accept: bool = True, stream=None):
        """gm_sample_tokens: temperature / top-k / top-p over the allowed tokens (+ accept)."""
        self._chk(bitmask, logits, None, tokens_out)
        _check(lib().gm_sample_tokens(self._h, _dptr(logits), logits.stride(0), _dptr(bitmask), bitmask.stride(0),
                                      float(temperature), int(top_k), float(top_p), seed & (2**64 - 1),
                                      _dptr(tokens_out), int(accept), _stream(stream)))

    def decode_step_sample(self, logits, temperature: float = 1.0, top_k: int = 0, top_p: float = 1.0,
                           seed: int = 0, tokens_out=None, bitmask=None, stream=None):
        """gm_decode_step_sample: fill + sample + accept, no host round trip."""
        self._chk(bitmask, logits, None, tokens_out)
        _check(lib().gm_decode_step_sample(self._h, _dptr(logits), logits.stride(0), _dptr(bitmask),
                                           bitmask.stride(0) if bitmask is not None else 0, float(temperature),
                                           int(top_k), float(top_p), seed & (2**64 - 1), _dptr(tokens_out),
                                           _stream(stream)))

    def capture_steps(self, steps: int, greedy: bool = False, seed: int = 0, bitmask=None, logits=None,
                      seg_counts=None, tokens_out=None) -> "StepGraph":
        """gm_decode_graph_create: a CUDA graph of `steps` (multiple of 6)
        decode steps.  Each of bitmask / logits / seg_counts / tokens_out is
        None, one tensor (every step) or a list of `steps` tensors."""
        def ptrs(x, kind, what, cols):
            if x is None:
                return None, 0
            xs = list(x) if isinstance(x, (list, tuple)) else [x] * steps
            if len(xs) != steps:
                raise ValueError(f"{what}: expected {steps} tensors")
            for t in xs:
                _check_tensor(t, kind, what, self.B, cols, self.engine.device)
            arr = (ctypes.c_void_p * steps)(*[t.data_ptr() for t in xs])
            return arr, (xs[0].stride(0) if xs[0].dim() == 2 else 0)
        bm, ldw = ptrs(bitmask, "i32|u32", "bitmask", self.engine.W)
        lg, ld = ptrs(logits, "bf16", "logits", self.engine.num_columns)
        sc, _ = ptrs(seg_counts, "i32", "seg_counts", 2 * self.nseg)
        to, _ = ptrs(tokens_out, "i32", "tokens_out", 1)
        h = ctypes.c_void_p()
        _check(lib().gm_decode_graph_create(self._h, int(greedy), steps, bm, ldw, lg, ld, sc, seed & (2**64 - 1), to,
                                            ctypes.byref(h)))
        return StepGraph(h, self, (bm, lg, sc, to, bitmask, logits, seg_counts, tokens_out))

    def check(self, stream=None):
        _check(lib().gm_batch_check(self._h, _stream(stream)))

    @property
    def split_step_launches(self) -> int:
        """Kernels one decode_step_stream_split launches (1: the accepts run
        as CTAs of the fill's grid; 2: fill + accept kernel)."""
        return int(lib().gm_batch_split_step_launches(self._h))

    def counters(self) -> dict:
        out = np.zeros(4, np.int64)
        _check(lib().gm_batch_counters(self._h, _ptr(out)))
        return dict(zip(["restarts", "draws", "fills", "accepts"], (int(x) for x in out)))

    def set_trace(self, buf=None):
        """Diagnostics: per-item timing records into a torch uint64/int64
        device tensor of 4 * (capacity + 1) entries (None turns it off)."""
        if buf is None:
            _check(lib().gm_batch_set_trace(self._h, None, 0))
        else:
            _check(lib().gm_batch_set_trace(self._h, ctypes.c_void_p(buf.data_ptr()), buf.numel() // 4 - 1))

    def set_stats(self, enable: bool):
        _check(lib().gm_batch_set_stats(self._h, int(enable)))

    def fill_stats(self) -> dict:
        out = np.zeros(6, np.int64)
        _check(lib().gm_batch_fill_stats(self._h, _ptr(out)))
        return dict(zip(["logit_bytes_read", "logit_bytes_written", "cd_walks", "build_items",
                         "private_fills", "build_wait_timeouts"], (int(x) for x in out)))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.gm_batch_destroy(self._h)
            self._h = ctypes.c_void_p()
