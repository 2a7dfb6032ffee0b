"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes bindings to the two CPU checkers built by oracle/Makefile:

* ``Ref``  — oracle/_ref/libgmask_ref.so: the UNMODIFIED reference matcher
  (gmask, /root/reference/proj) compiled from its own sources plus this repo's
  extern "C" shim (oracle/ref_shim.cpp).
* ``Port`` — oracle/_ref/libgmask_port.so: the plain-C restatement of the
  reference runtime (oracle/gmask_port.c), pinned against ``Ref`` and the
  golden vectors in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgmask_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libgmask_port.so")

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def pack(tokens: Sequence[bytes]) -> Tuple[np.ndarray, np.ndarray]:
    offs = np.zeros(len(tokens) + 1, np.int64)
    if tokens:
        np.cumsum([len(t) for t in tokens], out=offs[1:])
    data = np.frombuffer(b"".join(tokens) or b"\0", np.uint8).copy()
    return data, offs


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


class Ref:
    """The reference gmask::Engine behind oracle/ref_shim.cpp."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(REF_SO)
            sigs = {
                "ref_compile": ([ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P), ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
                "ref_dpda_free": ([P], None),
                "ref_dpda_flat": ([P, P, I64], I64),
                "ref_dpda_stats": ([P, P], None),
                "ref_engine_from_dpda": ([P], P),
                "ref_engine_from_flat": ([P, I64, ctypes.c_char_p, ctypes.c_int], P),
                "ref_engine_free": ([P], None),
                "ref_trie_new": ([P, P, I32, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int], P),
                "ref_trie_free": ([P], None),
                "ref_trie_nodes": ([P], I32),
                "ref_cfg_new": ([P], P),
                "ref_cfg_clone": ([P], P),
                "ref_cfg_free": ([P], None),
                "ref_cfg_get": ([P, P, P, P, I32], I32),
                "ref_cfg_set": ([P, I32, P, I32], None),
                "ref_step": ([P, P, I32], ctypes.c_int),
                "ref_allowed": ([P, P, P, P], None),
                "ref_mask": ([P, P, P, P], None),
                "ref_mask_naive": ([P, P, P, P, I32, P], None),
                "ref_decode_run": ([P, P, P, I32, I32, I32, U64, I32, I32, I32, P, P, P, I32, U64, I32], ctypes.c_int),
                "ref_sample_sentence": ([ctypes.c_char_p, U64, I32, ctypes.c_char_p, I32], I32),
            }
            opt = {  # present when the reference's serialize.cpp was built (json.hpp found)
                "ref_dpda_serialize": ([P, P, I64], I64),
                "ref_dpda_deserialize": ([P, I64, ctypes.POINTER(P), ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
                "ref_load_vocabulary": ([P, I64, P, I64, P, I32, ctypes.c_char_p, ctypes.c_int], I32),
            }
            for n, (a, r) in list(sigs.items()) + [kv for kv in opt.items() if hasattr(L, kv[0])]:
                f = getattr(L, n)
                f.argtypes = a
                f.restype = r
            cls._lib = L
        return cls._lib

    @classmethod
    def serialize_available(cls) -> bool:
        return ref_available() and hasattr(cls.lib(), "ref_dpda_serialize")

    @classmethod
    def compile_gmaskdp1(cls, grammar_text: str, aggregate: bool = True, merge: bool = True) -> Tuple[int, bytes]:
        """BuildDpda + SerializeDpda (serialize.cpp:148-196) -> (rc, GMASKDP1 bytes or error)."""
        L = cls.lib()
        d = P()
        err = ctypes.create_string_buffer(4096)
        rc = L.ref_compile(grammar_text.encode(), int(aggregate), int(merge), ctypes.byref(d), err, 4096)
        if rc != 0:
            return rc, err.value
        n = L.ref_dpda_serialize(d, None, 0)
        buf = ctypes.create_string_buffer(n)
        L.ref_dpda_serialize(d, buf, n)
        L.ref_dpda_free(d)
        return 0, buf.raw[:n]

    @classmethod
    def roundtrip_gmaskdp1(cls, data: bytes) -> Tuple[int, bytes]:
        """DeserializeDpda then SerializeDpda -> (rc, bytes or error message)."""
        L = cls.lib()
        d = P()
        err = ctypes.create_string_buffer(4096)
        src = ctypes.create_string_buffer(data, len(data))
        rc = L.ref_dpda_deserialize(src, len(data), ctypes.byref(d), err, 4096)
        if rc != 0:
            return rc, err.value
        n = L.ref_dpda_serialize(d, None, 0)
        buf = ctypes.create_string_buffer(n)
        L.ref_dpda_serialize(d, buf, n)
        L.ref_dpda_free(d)
        return 0, buf.raw[:n]

    @classmethod
    def load_vocabulary(cls, data: bytes):
        """LoadVocabulary (serialize.cpp:348-364) -> list of bytes, or raises ValueError(message)."""
        L = cls.lib()
        err = ctypes.create_string_buffer(4096)
        src = ctypes.create_string_buffer(data, len(data))
        n = L.ref_load_vocabulary(src, len(data), None, 0, None, 0, err, 4096)
        if n < 0:
            raise ValueError(err.value.decode())
        offs = np.zeros(n + 1, np.int64)
        L.ref_load_vocabulary(src, len(data), None, 0, _ptr(offs), n, err, 4096)
        buf = np.zeros(max(1, int(offs[n])), np.uint8)
        L.ref_load_vocabulary(src, len(data), _ptr(buf), int(offs[n]), _ptr(offs), n, err, 4096)
        raw = buf.tobytes()
        return [raw[offs[i]:offs[i + 1]] for i in range(n)]

    # ---- automaton
    @classmethod
    def compile_flat(cls, grammar_text: str, aggregate: bool = True, merge: bool = True) -> Tuple[int, bytes, dict]:
        """BuildDpda (dpda_builder.cpp:478-522) → (rc, P3DPDA bytes, stats)."""
        L = cls.lib()
        d = P()
        err = ctypes.create_string_buffer(4096)
        rc = L.ref_compile(grammar_text.encode(), int(aggregate), int(merge), ctypes.byref(d), err, 4096)
        if rc != 0:
            return rc, err.value, {}
        n = L.ref_dpda_flat(d, None, 0)
        buf = np.zeros(n, np.uint8)
        L.ref_dpda_flat(d, _ptr(buf), n)
        st = np.zeros(8, np.int64)
        L.ref_dpda_stats(d, _ptr(st))
        L.ref_dpda_free(d)
        keys = ["states", "edges", "composites", "cycles", "dynamic", "max_match_pop", "max_push",
                "edges_before_aggregation"]
        return 0, buf.tobytes(), dict(zip(keys, (int(x) for x in st)))

    @classmethod
    def sample_sentence(cls, grammar_text: str, seed: int, soft_limit: int = 24) -> bytes:
        L = cls.lib()
        buf = ctypes.create_string_buffer(1 << 16)
        n = L.ref_sample_sentence(grammar_text.encode(), seed, soft_limit, buf, 1 << 16)
        if n < 0:
            raise ValueError("sample failed")
        return buf.raw[:n]

    def __init__(self, flat: bytes, tokens: Optional[Sequence[bytes]] = None):
        L = self.lib()
        self._buf = np.frombuffer(flat, np.uint8).copy()
        err = ctypes.create_string_buffer(1024)
        self.h = L.ref_engine_from_flat(_ptr(self._buf), len(flat), err, 1024)
        if not self.h:
            raise ValueError(err.value.decode())
        self.trie = None
        self.tokens = None
        if tokens is not None:
            self.set_vocab(tokens)

    def set_vocab(self, tokens: Sequence[bytes]):
        L = self.lib()
        self.tokens = list(tokens)
        self._data, self._offs = pack(self.tokens)
        kind = ctypes.c_int()
        err = ctypes.create_string_buffer(1024)
        t = L.ref_trie_new(_ptr(self._data), _ptr(self._offs), len(self.tokens), ctypes.byref(kind), err, 1024)
        if not t:
            raise ValueError((kind.value, err.value.decode()))
        if self.trie:
            L.ref_trie_free(self.trie)
        self.trie = t

    @property
    def V(self) -> int:
        return len(self.tokens)

    @property
    def W(self) -> int:
        return (self.V + 1 + 31) // 32

    def initial(self) -> int:
        return self.lib().ref_cfg_new(self.h)

    def free_cfg(self, c):
        self.lib().ref_cfg_free(c)

    def clone(self, c):
        return self.lib().ref_cfg_clone(c)

    def get(self, c) -> Tuple[int, int, List[int]]:
        L = self.lib()
        st, status = I32(), I32()
        n = L.ref_cfg_get(c, ctypes.byref(st), ctypes.byref(status), None, 0)
        buf = np.zeros(max(n, 1), np.int32)
        L.ref_cfg_get(c, ctypes.byref(st), ctypes.byref(status), _ptr(buf), n)
        return st.value, status.value, buf[:n].tolist()

    def set(self, c, status: int, stack: Sequence[int]):
        st = np.asarray(stack, np.int32)
        self.lib().ref_cfg_set(c, status, _ptr(st), len(st))

    def step(self, c, terminal: int) -> bool:
        return bool(self.lib().ref_step(self.h, c, terminal))

    def accept_token(self, c, token: int) -> bool:
        """Step over token bytes (EOS = id V)."""
        if token == self.V:
            return self.step(c, 256)
        for b in self.tokens[token]:
            if not self.step(c, b):
                return False
        return True

    def allowed(self, c) -> Tuple[int, bool]:
        w = np.zeros(4, np.uint64)
        d = I32()
        self.lib().ref_allowed(self.h, c, _ptr(w), ctypes.byref(d))
        return int(w[0]) | int(w[1]) << 64 | int(w[2]) << 128 | int(w[3]) << 192, bool(d.value)

    def mask(self, c) -> np.ndarray:
        out = np.zeros(self.W, np.uint32)
        self.lib().ref_mask(self.h, c, self.trie, _ptr(out))
        return out

    def mask_naive(self, c) -> np.ndarray:
        out = np.zeros(self.W, np.uint32)
        self.lib().ref_mask_naive(self.h, c, _ptr(self._data), _ptr(self._offs), len(self.tokens), _ptr(out))
        return out

    def decode_run(self, structural: np.ndarray, batch: int, steps: int, seed: int, threads: int,
                   stack_cap: int = 1024, logits_row: int = 1, want_tokens: bool = False,
                   want_stacks: bool = False, warmup: int = 0, rows: int = 1, logit_seed: int = 0,
                   digest_seqs: int = 32):
        """stats[0] = seconds of the `steps` timed steps (after `warmup`);
        [5]/[6] = token digest / mask popcount (EOS excluded) of sequences
        < digest_seqs over the timed steps.  logits_row: 0 mask only, 1 +
        bf16 -inf row (stream sampler), 2 greedy argmax over synthetic bf16
        rows (config 5; buffer step % rows, gp_synth_logit)."""
        stats = np.zeros(8, np.float64)
        toks = np.zeros((batch, warmup + steps), np.int32) if want_tokens else None
        stk = np.zeros((batch, stack_cap + 2), np.int32) if want_stacks else None
        self.lib().ref_decode_run(self.h, self.trie, _ptr(structural), batch, warmup, steps, seed, threads, stack_cap,
                                  int(logits_row), _ptr(stats), _ptr(toks) if toks is not None else None,
                                  _ptr(stk) if stk is not None else None, rows, logit_seed & (2**64 - 1),
                                  digest_seqs)
        return stats, toks, stk

    def __del__(self):
        L = self._lib
        if L is not None:
            if getattr(self, "trie", None):
                L.ref_trie_free(self.trie)
            if getattr(self, "h", None):
                L.ref_engine_free(self.h)


class _RunOpts(ctypes.Structure):
    _fields_ = [("mode", I32), ("rows", I32), ("logit_seed", U64), ("warmup", I32), ("digest_seqs", I32),
                ("mask_hash", ctypes.c_void_p)]


def _port_lib():
    return Port.lib()


def synth_vocab(num_tokens: int, flavor: int = 0) -> List[bytes]:
    """The bench vocabulary restated in the C port (gp_synth_vocab:
    WriteBenchVocab, acceptance_main.cpp:341-359, continued) — the CPU arm's
    own input, independent of the product library."""
    L = _port_lib()
    n = L.gp_synth_vocab(num_tokens, flavor, None, 0, None)
    if n < 0:
        raise ValueError("bad vocabulary size")
    buf = np.zeros(max(n, 1), np.uint8)
    offs = np.zeros(num_tokens + 1, np.int64)
    L.gp_synth_vocab(num_tokens, flavor, _ptr(buf), n, _ptr(offs))
    raw = buf.tobytes()
    return [raw[offs[i]:offs[i + 1]] for i in range(num_tokens)]


def structural_words(tokens: Sequence[bytes]) -> np.ndarray:
    data, offs = pack(tokens)
    words = np.zeros((len(tokens) + 1 + 31) // 32, np.uint32)
    _port_lib().gp_structural_words(_ptr(data), _ptr(offs), len(tokens), _ptr(words))
    return words


def synth_logit_row(seed: int, k: int, b: int, n: int) -> np.ndarray:
    """gp_synth_logit row (config 5's synthetic bf16 logits), uint16 bits."""
    row = np.zeros(n, np.uint16)
    _port_lib().gp_synth_logit_row(seed & (2**64 - 1), k, b, n, _ptr(row))
    return row


_HASH_POW = {}


def mask_hashes(masks: np.ndarray) -> np.ndarray:
    """gp_mask_hash of every row of a [..., nw] uint32 mask array (numpy,
    wrapping uint64 arithmetic)."""
    m = np.ascontiguousarray(masks).view(np.uint32)
    nw = m.shape[-1]
    pw = _HASH_POW.get(nw)
    if pw is None:
        pw = np.zeros(nw, np.uint64)
        M = np.uint64(0x9E3779B97F4A7C15)
        p = M
        with np.errstate(over="ignore"):
            for i in range(nw):
                pw[i] = p
                p = p * M
        _HASH_POW[nw] = pw
    with np.errstate(over="ignore"):
        return (m.astype(np.uint64) * pw).sum(axis=-1, dtype=np.uint64)


class _Cfg(ctypes.Structure):
    _fields_ = [("state", I32), ("status", I32), ("depth", I32), ("cap", I32),
                ("stack", ctypes.POINTER(I32))]


class Port:
    """The C restatement (oracle/gmask_port.c) over a P3DPDA automaton."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(PORT_SO)
            CP = ctypes.POINTER(_Cfg)
            sigs = {
                "gp_automaton_load": ([P, I64], P),
                "gp_automaton_free": ([P], None),
                "gp_trie_build": ([P, P, I32, ctypes.POINTER(ctypes.c_int)], P),
                "gp_trie_free": ([P], None),
                "gp_trie_nodes": ([P], I32),
                "gp_config_init": ([P, CP], None),
                "gp_config_copy": ([CP, CP], None),
                "gp_config_free": ([CP], None),
                "gp_step": ([P, CP, I32], ctypes.c_int),
                "gp_allowed": ([P, CP, P, ctypes.POINTER(ctypes.c_int)], None),
                "gp_mask": ([P, CP, P, P], None),
                "gp_mask_naive": ([P, CP, P, P, I32, P], None),
                "gp_stream_draw": ([U64, U64, U64], U64),
                "gp_stream_pick": ([P, P, I32, U64], I32),
                "gp_greedy_pick": ([P, P, I32], I32),
                "gp_sample_pick": ([P, P, I32, ctypes.c_float, I32, ctypes.c_uint32, U64], I32),
                "gp_sample_weight": ([ctypes.c_uint32, ctypes.c_float, ctypes.c_float], U64),
                "gp_decode_run": ([P, P, P, P, P, I32, I32, U64, I32, P, P, P, P], ctypes.c_int),
                "gp_synth_vocab": ([I32, I32, P, I64, P], I64),
                "gp_structural_words": ([P, P, I32, P], I32),
                "gp_synth_logit_row": ([U64, I32, I32, I32, P], None),
                "gp_mask_hash": ([P, I32], U64),
            }
            for n, (a, r) in sigs.items():
                f = getattr(L, n)
                f.argtypes = a
                f.restype = r
            cls._lib = L
        return cls._lib

    def __init__(self, flat: bytes, tokens: Sequence[bytes]):
        L = self.lib()
        self._buf = np.frombuffer(flat, np.uint8).copy()
        self.a = L.gp_automaton_load(_ptr(self._buf), len(flat))
        if not self.a:
            raise ValueError("bad automaton")
        self.tokens = list(tokens)
        self._data, self._offs = pack(self.tokens)
        kind = ctypes.c_int()
        self.trie = L.gp_trie_build(_ptr(self._data), _ptr(self._offs), len(self.tokens), ctypes.byref(kind))
        if not self.trie:
            raise ValueError(("vocab", kind.value))

    @property
    def V(self) -> int:
        return len(self.tokens)

    @property
    def W(self) -> int:
        return (self.V + 1 + 31) // 32

    def initial(self) -> _Cfg:
        c = _Cfg()
        self.lib().gp_config_init(self.a, ctypes.byref(c))
        return c

    def config(self, status: int, stack: Sequence[int]) -> _Cfg:
        c = self.initial()
        src = _Cfg()
        arr = (I32 * len(stack))(*stack)
        src.state = stack[-1]
        src.status = status
        src.depth = len(stack)
        src.cap = len(stack)
        src.stack = ctypes.cast(arr, ctypes.POINTER(I32))
        self.lib().gp_config_copy(ctypes.byref(c), ctypes.byref(src))
        return c

    @staticmethod
    def get(c: _Cfg) -> Tuple[int, int, List[int]]:
        return c.state, c.status, [c.stack[i] for i in range(c.depth)]

    def free(self, c: _Cfg):
        self.lib().gp_config_free(ctypes.byref(c))

    def step(self, c: _Cfg, terminal: int) -> bool:
        return bool(self.lib().gp_step(self.a, ctypes.byref(c), terminal))

    def accept_token(self, c: _Cfg, token: int) -> bool:
        if token == self.V:
            return self.step(c, 256)
        for b in self.tokens[token]:
            if not self.step(c, b):
                return False
        return True

    def allowed(self, c: _Cfg) -> Tuple[int, bool]:
        w = np.zeros(4, np.uint64)
        d = ctypes.c_int()
        self.lib().gp_allowed(self.a, ctypes.byref(c), _ptr(w), ctypes.byref(d))
        return int(w[0]) | int(w[1]) << 64 | int(w[2]) << 128 | int(w[3]) << 192, bool(d.value)

    def mask(self, c: _Cfg) -> np.ndarray:
        out = np.zeros(self.W, np.uint32)
        self.lib().gp_mask(self.a, ctypes.byref(c), self.trie, _ptr(out))
        return out

    def mask_naive(self, c: _Cfg) -> np.ndarray:
        out = np.zeros(self.W, np.uint32)
        self.lib().gp_mask_naive(self.a, ctypes.byref(c), _ptr(self._data), _ptr(self._offs), len(self.tokens),
                                 _ptr(out))
        return out

    def stream_pick(self, mask: np.ndarray, structural: np.ndarray, u: int) -> int:
        return self.lib().gp_stream_pick(_ptr(mask), _ptr(structural), self.V, u)

    @classmethod
    def stream_draw(cls, seed: int, seq: int, draw: int) -> int:
        return cls.lib().gp_stream_draw(seed, seq, draw)

    def sample_pick(self, mask: np.ndarray, logits_bf16: np.ndarray, temperature: float, top_k: int, top_p: float,
                    u: int) -> int:
        """Temperature / top-k / top-p pick (the SampleKernel rule)."""
        p24 = (1 << 24) if top_p >= 1.0 else max(1, int(np.floor(np.float64(np.float32(top_p)) * 16777216.0)))
        return int(self.lib().gp_sample_pick(_ptr(np.ascontiguousarray(mask, np.uint32)),
                                             _ptr(np.ascontiguousarray(logits_bf16, np.uint16)), self.V,
                                             float(temperature), int(top_k), p24, u & (2**64 - 1)))

    def greedy_pick(self, mask: np.ndarray, logits_bf16: np.ndarray) -> int:
        return self.lib().gp_greedy_pick(_ptr(mask), _ptr(logits_bf16), self.V)

    def decode_run(self, structural: np.ndarray, batch: int, steps: int, seed: int, stack_cap: int = 1024,
                   want_tokens: bool = False, want_stacks: bool = False, want_mask_hashes: bool = False,
                   greedy_rows: int = 0, logit_seed: int = 0, warmup: int = 0, digest_seqs: int = 0):
        """The C port's decode loop.  greedy_rows > 0: greedy over
        gp_synth_logit rows (buffer step % greedy_rows) instead of the stream
        sampler.  want_mask_hashes: [batch][steps] gp_mask_hash of every
        mask (compare with mask_hashes() of device bitmasks)."""
        stats = np.zeros(8, np.float64)
        toks = np.zeros((batch, steps), np.int32) if want_tokens else None
        stk = np.zeros((batch, stack_cap + 2), np.int32) if want_stacks else None
        mh = np.zeros((batch, steps), np.uint64) if want_mask_hashes else None
        opts = _RunOpts(1 if greedy_rows > 0 else 0, max(1, greedy_rows), logit_seed & (2**64 - 1), warmup,
                        digest_seqs, mh.ctypes.data if mh is not None else None)
        self.lib().gp_decode_run(self.a, self.trie, _ptr(self._data), _ptr(self._offs), _ptr(structural), batch,
                                 steps, seed, stack_cap, _ptr(stats), _ptr(toks) if toks is not None else None,
                                 _ptr(stk) if stk is not None else None, ctypes.byref(opts))
        if want_mask_hashes:
            return stats, toks, stk, mh
        return stats, toks, stk

    def __del__(self):
        L = self._lib
        if L is not None:
            if getattr(self, "trie", None):
                L.gp_trie_free(self.trie)
            if getattr(self, "a", None):
                L.gp_automaton_free(self.a)


def build(ref: bool = True) -> None:
    """make -C oracle (port always; ref when /root/reference is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def read_flat(flat: bytes) -> dict:
    """Parses P3DPDA v1 into plain Python structures."""
    import struct
    assert flat[:8] == b"P3DPDA01"
    o = 8
    S, init, acc, ghash, tl = struct.unpack_from("<iiiQi", flat, o)
    o += 24
    text = flat[o:o + tl].decode("latin-1")
    o += tl
    shift = np.frombuffer(flat, np.int32, S * 256, o).copy()
    o += S * 256 * 4
    (E,) = struct.unpack_from("<i", flat, o)
    o += 4
    begin = np.frombuffer(flat, np.int32, S + 1, o).copy()
    o += (S + 1) * 4
    edges = []
    for _ in range(E):
        src, w0, w1, w2, w3, dollar, origin, dyn, _pad, target, cl, pl = struct.unpack_from("<iQQQQBBBBiii", flat, o)
        o += 4 + 32 + 4 + 12
        cond = list(struct.unpack_from(f"<{cl}i", flat, o))
        o += 4 * cl
        push = list(struct.unpack_from(f"<{pl}i", flat, o))
        o += 4 * pl
        edges.append({"source": src, "accepted": w0 | w1 << 64 | w2 << 128 | w3 << 192, "dollar": bool(dollar),
                      "origin": origin, "dynamic": bool(dyn), "target": target, "match_pop": cond, "push": push})
    assert o == len(flat)
    return {"num_states": S, "initial": init, "accept": acc, "grammar_hash": ghash, "grammar_text": text,
            "shift": shift, "edge_begin": begin, "edges": edges}
