"""Pins the oracle: the C restatement (oracle/gmask_port.c) against the golden
vectors generated from the reference (tests/golden/, oracle/make_golden.py)
and, when /root/reference is present, against the reference itself.

Mirrors the reference's own runtime tests (tests/test_runtime.cpp) and the
acceptance gate's mask criterion (tests/acceptance/acceptance_main.cpp:202-219).
"""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import oracle
from oracle import Port, Ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = ["paren", "list_left", "list_right", "digits", "expr", "json"]


def flat(name):
    with open(os.path.join(GOLDEN, name + ".p3dpda"), "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def vectors():
    with open(os.path.join(GOLDEN, "vectors.json")) as f:
        return json.load(f)


def mask_hex(w, V):
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


def test_paren_seven_token_masks(vectors):
    """test_runtime.cpp:184-206 / test_cli.cpp:113-132: b2, 40, eos-only."""
    vocab = [t.encode() for t in vectors["paren7"]["vocab"]]
    p = Port(flat("paren"), vocab)
    want = {"": "b2", "(a": "40", "a": "08", "(a)": "08"}
    for prefix, g in vectors["paren7"]["masks"].items():
        c = p.initial()
        for ch in prefix.encode():
            assert p.step(c, ch)
        m = p.mask(c)
        assert mask_hex(m, 7) == g["hex"]
        if prefix in want:
            assert g["hex"] == want[prefix]
        assert list(p.get(c)) == g["config"]
        assert np.array_equal(m, p.mask_naive(c))
        p.free(c)


@pytest.mark.parametrize("name", FIXTURES)
def test_mask_agreement_cases(vectors, name):
    """Trie walk == golden (reference) masks == naive replay on sampled configs."""
    case = vectors["mask_agreement"][name]
    vocab = [bytes.fromhex(h) for h in case["vocab_hex"]]
    p = Port(flat(name), vocab)
    for c in case["cases"]:
        cfg = p.config(c["status"], c["stack"])
        m = p.mask(cfg)
        assert mask_hex(m, len(vocab)) == c["hex"]
        assert np.array_equal(m, p.mask_naive(cfg))
        p.free(cfg)


def test_json32k_stream_replay(vectors):
    """Config 1: JSON + 32k acceptance-bench vocabulary, token-level streams:
    every mask digest, token, post-accept state/stack matches the reference."""
    import paper_2506_03887_b200 as pk
    g = vectors["json32k_stream"]
    vocab = pk.synth_vocab(32000)
    assert hashlib.sha256(b"\0".join(vocab)).hexdigest() == g["vocab_sha"]
    structural = pk.structural_words(vocab)
    p = Port(flat("json"), vocab)
    for b in range(g["batch"]):
        c = p.initial()
        for s in range(g["steps"]):
            want = g["trace"][b][s]
            m = p.mask(c)
            assert hashlib.sha256(m.tobytes()).hexdigest()[:32] == want["mask"], (b, s)
            tok = p.stream_pick(m, structural, Port.stream_draw(g["seed"], b, s))
            assert tok == want["token"] == g["tokens"][b][s]
            if tok >= 0:
                p.accept_token(c, tok)
            st, status, stack = p.get(c)
            assert (st, status, len(stack)) == (want["state"], want["status"], want["depth"])
            assert hashlib.sha256(np.asarray(stack, np.int32).tobytes()).hexdigest()[:16] == want["stack"]
            if tok < 0 or status != 0 or len(stack) > 1024:
                p.free(c)
                c = p.initial()
        fin = g["final"][b]
        st, status, stack = p.get(c)
        assert stack == fin["stack"] and status == fin["status"]
        p.free(c)
    # The port's batched decode loop reproduces the reference loop's digest.
    stats, toks, _ = p.decode_run(structural, g["batch"], g["steps"], g["seed"], want_tokens=True)
    assert toks.tolist() == g["tokens"]
    assert int(stats[3]) == g["digest"] and int(stats[2]) == g["restarts"] and int(stats[4]) == g["popcount_sum"]


def test_statuses_and_invariants():
    """test_runtime.cpp:88-114: terminal statuses, stack top mirrors state."""
    p = Port(flat("paren"), [b"a"])
    c = p.initial()
    assert p.step(c, ord("a")) and p.step(c, 256)
    assert c.status == 2 and not p.step(c, ord("a")) and c.status == 2
    d = p.initial()
    assert not p.step(d, ord(")")) and d.status == 1
    assert not p.step(d, ord("a")) and d.status == 1
    assert p.allowed(d)[0] == 0 and p.mask(d).sum() == 0
    e = Port(flat("expr"), [b"n"])
    c = e.initial()
    for ch in b"n+n*(n+n)":
        assert e.step(c, ch)
        st, _, stack = e.get(c)
        assert stack[-1] == st and stack[0] == 0


def test_cycle_collapse_constant_depth():
    """test_runtime.cpp:279-291: list_right depth(x^4) == depth(x^64)."""
    p = Port(flat("list_right"), [b"x"])

    def depth(n):
        c = p.initial()
        for _ in range(n):
            assert p.step(c, ord("x"))
        return len(p.get(c)[2])

    assert depth(4) == depth(64) == depth(512)


def test_trie_rejects():
    """test_runtime.cpp:139-158: empty and duplicate tokens."""
    with pytest.raises(ValueError) as e:
        Port(flat("paren"), [b"x", b""])
    assert e.value.args[0] == ("vocab", 1)
    with pytest.raises(ValueError) as e:
        Port(flat("paren"), [b"ab", b"cd", b"ab"])
    assert e.value.args[0] == ("vocab", 2)


def test_stream_sampler_rule():
    """EOS-only → EOS, empty → -1, picks are allowed tokens."""
    p = Port(flat("paren"), [b"a", b"(", b")"])
    s = np.zeros(1, np.uint32)
    assert p.stream_pick(np.array([0], np.uint32), s, 0) == -1
    assert p.stream_pick(np.array([1 << 3], np.uint32), s, 0) == 3
    rng = random.Random(3)
    for _ in range(200):
        m = np.array([rng.randrange(16)], np.uint32)
        t = p.stream_pick(m, s, rng.getrandbits(64))
        if m[0] == 0:
            assert t == -1
        else:
            assert (int(m[0]) >> t) & 1


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("name", FIXTURES)
def test_port_matches_reference_engine(name):
    """Port vs the reference Engine on random configs and random vocabularies:
    masks, allowed terminals, step outcomes (kernels.cpp semantics incl. -1
    padding and union over all matching edges)."""
    rng = random.Random(hash(name) & 0xFFFF)
    f = flat(name)
    info = oracle.read_flat(f)
    acc = 0
    for e in info["edges"]:
        acc |= e["accepted"]
    alphabet = [b for b in range(256) if (acc >> b) & 1] + [0, 0x5A, 0xFF]
    vocab = sorted({bytes(rng.choice(alphabet) for _ in range(1 + rng.randrange(6))) for _ in range(400)})
    r = Ref(f, vocab)
    p = Port(f, vocab)
    for _ in range(30):
        rc, pc = r.initial(), p.initial()
        for _ in range(rng.randrange(30)):
            allowed, _ = r.allowed(rc)
            assert (allowed, _) == p.allowed(pc)
            bs = [b for b in range(256) if (allowed >> b) & 1]
            if not bs:
                break
            b = rng.choice(bs)
            assert r.step(rc, b) == p.step(pc, b)
        assert r.get(rc) == p.get(pc)
        assert np.array_equal(r.mask(rc), p.mask(pc))
        junk = rng.randrange(257)
        assert r.step(rc, junk) == p.step(pc, junk)
        assert r.get(rc) == p.get(pc)
        r.free_cfg(rc)
        p.free(pc)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
def test_port_decode_loop_matches_reference_128k():
    """Config 2 shape (JSON, 128,255-token vocab): the two CPU decode loops
    (reference Engine vs C port) produce identical token streams/stacks."""
    import paper_2506_03887_b200 as pk
    vocab = pk.synth_vocab(128255)
    structural = pk.structural_words(vocab)
    f = flat("json")
    r = Ref(f, vocab)
    p = Port(f, vocab)
    sr, tr, kr = r.decode_run(structural, 3, 6, 11, threads=3, want_tokens=True, want_stacks=True)
    sp, tp, kp = p.decode_run(structural, 3, 6, 11, want_tokens=True, want_stacks=True)
    assert np.array_equal(tr, tp) and np.array_equal(kr, kp)
    assert sr[3] == sp[3] and sr[4] == sp[4]


@pytest.fixture(scope="module")
def acceptance():
    with open(os.path.join(GOLDEN, "acceptance_masks.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", FIXTURES)
def test_acceptance_criterion3_reference_scale(acceptance, name):
    """Acceptance criterion 3 at the reference's own scale and seeds
    (acceptance_main.cpp:202-219: 200 SampleConfigs x a 1,000-token
    SampleVocab per fixture, generated by the reference's own helpers): the
    port's trie mask and its naive replay equal the reference's masks."""
    case = acceptance["fixtures"][name]
    vocab = [bytes.fromhex(h) for h in case["vocab_hex"]]
    assert len(vocab) == 1000 and len(case["cases"]) == 200
    p = Port(flat(name), vocab)
    for c in case["cases"]:
        cfg = p.config(c["status"], c["stack"])
        m = p.mask(cfg)
        assert mask_hex(m, len(vocab)) == c["hex"]
        if c is case["cases"][0] or random.Random(len(c["stack"])).random() < 0.1:
            assert np.array_equal(m, p.mask_naive(cfg))
        p.free(cfg)


def test_oracle_workload_generators_match_product():
    """The CPU arm's own inputs (gp_synth_vocab / gp_structural_words, C
    restatements in the oracle) equal the product's generator byte for byte,
    for every flavour the bench uses."""
    import paper_2506_03887_b200 as pk
    for n, flavor in [(32000, 0), (128255, 0), (128255, 1)]:
        a = oracle.synth_vocab(n, flavor)
        assert a == pk.synth_vocab(n, flavor)
        assert np.array_equal(oracle.structural_words(a), pk.structural_words(a))


def test_bench_vocab_is_the_references(vectors):
    """gp_synth_vocab(32000) == WriteBenchVocab (acceptance_main.cpp:341-359):
    the sha256 recorded by make_golden.py after asserting equality with the
    reference's own function (oracle/_ref/libgmask_acc.so)."""
    import hashlib as h
    v = oracle.synth_vocab(32000)
    assert h.sha256(b"\0".join(v)).hexdigest() == vectors["json32k_stream"]["vocab_sha"]
    acc = os.path.join(os.path.dirname(oracle.__file__), "_ref", "libgmask_acc.so")
    if os.path.exists(acc) and os.path.isdir("/root/reference/proj"):
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "make_golden", os.path.join(os.path.dirname(oracle.__file__), "make_golden.py"))
        mg = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mg)
        assert mg.reference_bench_vocab() == v


def test_mask_hash_numpy_matches_c():
    rng = np.random.default_rng(1)
    m = rng.integers(0, 2**32, size=(5, 4008), dtype=np.uint64).astype(np.uint32)
    got = oracle.mask_hashes(m)
    L = oracle.Port.lib()
    for i in range(5):
        assert int(got[i]) == int(L.gp_mask_hash(m[i].ctypes.data, 4008))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("greedy", [False, True])
def test_window_digests_reference_vs_port(greedy):
    """The in-run evidence both bench arms print (token digest and mask
    popcounts of sequences < 32 over the timed steps): the reference decode
    loop and the port agree, stream and greedy (synthetic logits rows)."""
    vocab = oracle.synth_vocab(32000)
    structural = oracle.structural_words(vocab)
    f = flat("json")
    r = Ref(f, vocab)
    p = Port(f, vocab)
    B, W_, K = 36, 5, 12
    kw = dict(greedy_rows=3, logit_seed=99) if greedy else {}
    sr, tr, _ = r.decode_run(structural, B, K, 4, threads=4, warmup=W_, want_tokens=True,
                             logits_row=2 if greedy else 1, rows=3, logit_seed=99, digest_seqs=32)
    sp, tp, _ = p.decode_run(structural, B, W_ + K, 4, want_tokens=True, warmup=W_, digest_seqs=32, **kw)
    assert np.array_equal(tr, tp)
    assert sr[5] == sp[5] and sr[6] == sp[6]
    assert sr[6] > 0
