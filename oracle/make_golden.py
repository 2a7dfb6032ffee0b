"""oracle/make_golden.py — TEST INFRASTRUCTURE ONLY.

Regenerates tests/golden/ from the UNMODIFIED reference matcher
(oracle/_ref/libgmask_ref.so, built from /root/reference/proj by
oracle/Makefile).  Run here (the reference does not exist on the GPU box):

    make -C oracle && python oracle/make_golden.py

Outputs
  tests/golden/<fixture>.p3dpda   BuildDpda(default options) of every fixture
                                  grammar (grammars/*.bnf of the reference),
                                  exported to the flat P3DPDA v1 format;
                                  digits_noagg.p3dpda = aggregate off.
  tests/golden/vectors.json       known-answer tests (see keys below).
  tests/golden/acceptance_masks.json
                                  acceptance criterion 3 at the reference's own
                                  scale and seeds (acceptance_main.cpp:202-219,
                                  through oracle/_ref/libgmask_acc.so): per
                                  fixture the 1,000-token SampleVocab, the 200
                                  SampleConfigs and their reference masks.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import Ref, read_flat  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402  (cross-check of the product's vocab generator only)

GRAMMARS = os.environ.get("GMASK_GRAMMAR_DIR", "/root/reference/proj/grammars")
OUT = os.path.join(ROOT, "tests", "golden")
FIXTURES = ["paren", "list_left", "list_right", "digits", "expr", "json"]


def sha(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, np.uint32).tobytes()).hexdigest()[:32]


def mask_hex(w: np.ndarray, V: int) -> str:
    """TokenMask::ToHex (runtime.cpp:73-86)."""
    n = V + 1
    out = []
    for i in range((n + 3) // 4):
        nib = 0
        for j in range(4):
            bit = i * 4 + j
            if bit < n and (int(w[bit >> 5]) >> (bit & 31)) & 1:
                nib |= 1 << j
        out.append("0123456789abcdef"[nib])
    return "".join(out)


def sample_vocab(grammar_text: str, terminals: bytes, count: int, rng: random.Random):
    """Like acceptance_main.cpp:98-115 SampleVocab: grammar bytes + noise."""
    alphabet = sorted(set(terminals)) + [0x00, 0xFF, 0x5A, 0x20]
    seen, vocab = set(), []
    while len(vocab) < count:
        n = 1 + rng.randrange(8)
        tok = bytes(alphabet[rng.randrange(len(alphabet))] for _ in range(n))
        if tok not in seen:
            seen.add(tok)
            vocab.append(tok)
    return vocab


def sample_configs(ref: Ref, count: int, max_prefix: int, rng: random.Random):
    """Like acceptance_main.cpp:74-95 SampleConfigs: random walks over allowed bytes."""
    out = []
    c = ref.initial()
    depth = 0
    while len(out) < count:
        out.append(ref.get(c))
        allowed, _ = ref.allowed(c)
        bytes_ = [b for b in range(256) if (allowed >> b) & 1]
        depth += 1
        if not bytes_ or depth > max_prefix:
            ref.free_cfg(c)
            c = ref.initial()
            depth = 0
            continue
        ref.step(c, bytes_[rng.randrange(len(bytes_))])
    ref.free_cfg(c)
    return out


def _acc_lib():
    import ctypes
    L = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libgmask_acc.so"))
    L.acc_write_bench_vocab.argtypes = [ctypes.c_char_p]
    P, I64 = ctypes.c_void_p, ctypes.c_int64
    L.acc_mask_agreement_inputs.argtypes = [ctypes.c_char_p, P, I64, ctypes.POINTER(I64), P, I64,
                                            ctypes.POINTER(I64)]
    return L


def reference_bench_vocab():
    """WriteBenchVocab (acceptance_main.cpp:341-359) run from the reference's
    own source: the 32,000-token bench vocabulary as the reference writes it."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "vocab32k.json")
        assert _acc_lib().acc_write_bench_vocab(path.encode()) == 0
        return [t.encode("latin-1") for t in json.load(open(path, encoding="utf-8"))]


def acceptance_masks(flats) -> None:
    """Acceptance criterion 3 at the reference's scale: per fixture, the
    reference's own SampleVocab(1000) and SampleConfigs(200, 40) with the
    MaskAgreement seeds (0xba5e + std::hash(name)); masks from the reference
    engine over our fixture automata (asserted == ComputeMaskNaive)."""
    import ctypes
    L = _acc_lib()
    out = {"source": "acceptance_main.cpp:202-219 via oracle/_ref/libgmask_acc.so", "fixtures": {}}
    total = 0
    for name in FIXTURES:
        vn, cn = ctypes.c_int64(), ctypes.c_int64()
        assert L.acc_mask_agreement_inputs(name.encode(), None, 0, ctypes.byref(vn), None, 0, ctypes.byref(cn)) == 0
        vb, cb = ctypes.create_string_buffer(vn.value), ctypes.create_string_buffer(cn.value)
        assert L.acc_mask_agreement_inputs(name.encode(), vb, vn.value, ctypes.byref(vn), cb, cn.value,
                                           ctypes.byref(cn)) == 0
        vocab_hex = json.loads(vb.raw[: vn.value].decode())
        vocab = [bytes.fromhex(h) for h in vocab_hex]
        ref = Ref(flats[name], vocab)
        cases = []
        for line in cb.raw[: cn.value].decode().splitlines():
            f = [int(x) for x in line.split()]
            status, depth, stack = f[0], f[1], f[2:]
            assert len(stack) == depth
            c = ref.initial()
            ref.set(c, status, stack)
            m = ref.mask(c)
            assert np.array_equal(m, ref.mask_naive(c)), name
            ref.free_cfg(c)
            cases.append({"status": status, "stack": stack, "hex": mask_hex(m, len(vocab))})
        assert len(cases) == 200 and len(vocab) == 1000
        total += len(cases)
        out["fixtures"][name] = {"vocab_hex": vocab_hex, "cases": cases}
    with open(os.path.join(OUT, "acceptance_masks.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=True)
    print("acceptance masks:", total)


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    vectors: dict = {"source": "reference gmask (oracle/_ref/libgmask_ref.so) via oracle/make_golden.py"}
    flats = {}
    stats = {}
    for name in FIXTURES:
        text = open(os.path.join(GRAMMARS, name + ".bnf")).read()
        rc, flat, st = Ref.compile_flat(text)
        assert rc == 0, (name, flat)
        flats[name] = flat
        stats[name] = st
        with open(os.path.join(OUT, name + ".p3dpda"), "wb") as f:
            f.write(flat)
    text = open(os.path.join(GRAMMARS, "digits.bnf")).read()
    rc, flat, st = Ref.compile_flat(text, aggregate=False)
    with open(os.path.join(OUT, "digits_noagg.p3dpda"), "wb") as f:
        f.write(flat)
    stats["digits_noagg"] = st
    rc, err, _ = Ref.compile_flat(open(os.path.join(GRAMMARS, "ambiguous.bnf")).read())
    vectors["ambiguous_rc"] = rc
    vectors["ambiguous_err"] = err.decode(errors="replace")
    vectors["automaton_stats"] = stats

    # 1. The worked seven-token paren vocabulary (test_runtime.cpp:184-206,
    #    test_cli.cpp:113-132): masks after "", "(a", "a", "(a)".
    vocab7 = [b"a", b"(", b")", b"((", b"a)", b"(a)", b")))"]
    r = Ref(flats["paren"], vocab7)
    paren = {}
    for prefix in ["", "(a", "a", "(a)", "((", "(((a"]:
        c = r.initial()
        for ch in prefix.encode():
            assert r.step(c, ch)
        m = r.mask(c)
        paren[prefix] = {"hex": mask_hex(m, 7), "config": r.get(c)}
        r.free_cfg(c)
    assert paren[""]["hex"] == "b2" and paren["(a"]["hex"] == "40"
    vectors["paren7"] = {"vocab": [t.decode() for t in vocab7], "masks": paren}

    # 2. Trie walk == naive replay on sampled configs (acceptance criterion 3,
    #    acceptance_main.cpp:202-219), 300-token sampled vocabularies.
    agreement = {}
    for name in FIXTURES:
        rng = random.Random(0xBA5E + FIXTURES.index(name))
        ref = Ref(flats[name])
        # terminal alphabet = every byte some edge accepts
        acc = 0
        for e in read_flat(flats[name])["edges"]:
            acc |= e["accepted"]
        terms = bytes(b for b in range(256) if (acc >> b) & 1)
        vocab = sample_vocab("", terms, 300, rng)
        ref.set_vocab(vocab)
        cases = []
        for (state, status, stack) in sample_configs(ref, 40, 40, rng):
            c = ref.initial()
            ref.set(c, status, stack)
            m = ref.mask(c)
            assert np.array_equal(m, ref.mask_naive(c)), name
            cases.append({"stack": stack, "status": status, "hex": mask_hex(m, len(vocab))})
            ref.free_cfg(c)
        agreement[name] = {"vocab_hex": [t.hex() for t in vocab], "cases": cases}
    vectors["mask_agreement"] = agreement

    # 3. Config 1: JSON + the acceptance bench vocabulary (32,000 tokens,
    #    acceptance_main.cpp:341-359), token-level stream replay,
    #    4 sequences x 120 steps: per-step mask digests, tokens, post-accept
    #    states and stacks.
    vocab32 = oracle.synth_vocab(32000)
    assert vocab32 == reference_bench_vocab(), "gp_synth_vocab != WriteBenchVocab"
    assert vocab32 == pk.synth_vocab(32000), "product generator != WriteBenchVocab"
    structural = oracle.structural_words(vocab32)
    ref = Ref(flats["json"], vocab32)
    seed = 1
    steps, batch = 120, 4
    stats_, toks, stacks = ref.decode_run(structural, batch, steps, seed, threads=1, stack_cap=1024,
                                          want_tokens=True, want_stacks=True)
    # Step-by-step replay through the plain reference API to pin every mask.
    from oracle import Port  # sampler restatement (identical rule)
    port = Port(flats["json"], vocab32)
    trace = []
    for b in range(batch):
        c = ref.initial()
        seq = []
        for s in range(steps):
            m = ref.mask(c)
            u = Port.stream_draw(seed, b, s)
            tok = port.stream_pick(m, structural, u)
            assert tok == toks[b, s], (b, s, tok, toks[b, s])
            if tok >= 0:
                ref.accept_token(c, tok)
            st, status, stack = ref.get(c)
            seq.append({"mask": sha(m), "pop": int(sum(bin(int(x)).count("1") for x in m)), "token": int(tok),
                        "state": st, "status": status, "depth": len(stack),
                        "stack": hashlib.sha256(np.asarray(stack, np.int32).tobytes()).hexdigest()[:16]})
            if tok < 0 or status != 0 or len(stack) > 1024:
                ref.free_cfg(c)
                c = ref.initial()
        ref.free_cfg(c)
        trace.append(seq)
    vectors["json32k_stream"] = {
        "vocab_sha": hashlib.sha256(b"\0".join(vocab32)).hexdigest(),
        "seed": seed, "batch": batch, "steps": steps,
        "digest": int(stats_[3]), "restarts": int(stats_[2]), "popcount_sum": int(stats_[4]),
        "tokens": toks.tolist(),
        "final": [{"depth": int(row[0]), "status": int(row[1]), "stack": row[2:2 + row[0]].tolist()} for row in stacks],
        "trace": trace,
    }
    with open(os.path.join(OUT, "vectors.json"), "w") as f:
        json.dump(vectors, f, indent=0, sort_keys=True)
    acceptance_masks(flats)
    print("wrote", OUT, {k: os.path.getsize(os.path.join(OUT, k)) for k in os.listdir(OUT)})


if __name__ == "__main__":
    main()
