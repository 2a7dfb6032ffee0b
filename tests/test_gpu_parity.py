"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Bit-exact for everything: bitmasks, -inf positions of the masked bf16
logits, sampled tokens, post-accept DPDA states/statuses/stacks.  Mirrors the
reference's runtime tests (tests/test_runtime.cpp:160-291) and acceptance
criterion 3 (acceptance_main.cpp:202-219).
"""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import paper_2506_03887_b200 as pk
from oracle import Port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = ["paren", "list_left", "list_right", "digits", "expr", "json"]
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def flat(name):
    with open(os.path.join(GOLDEN, name + ".p3dpda"), "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def vectors():
    with open(os.path.join(GOLDEN, "vectors.json")) as f:
        return json.load(f)


def mask_hex(w, V):
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


def fill_batch(eng, cfgs, logits=False, cap=1024):
    """Uploads configs, runs the fused fill, returns (masks, logits or None)."""
    b = eng.batch(len(cfgs), cap)
    for i, c in enumerate(cfgs):
        b.set(i, c)
    bm = torch.zeros((len(cfgs), eng.W), dtype=torch.int32, device=DEV)
    lg = None
    if logits:
        lg = torch.randn((len(cfgs), eng.V + 1), dtype=torch.bfloat16, device=DEV)
    b.fill(bm, lg)
    b.check()
    return bm.cpu().numpy().view(np.uint32), lg


def test_paren_seven_token_masks(vectors):
    vocab = [t.encode() for t in vectors["paren7"]["vocab"]]
    eng = pk.DeviceEngine(pk.Automaton.load(flat("paren")), vocab)
    for prefix, g in vectors["paren7"]["masks"].items():
        st, status, stack = g["config"]
        m = eng.ComputeMask(pk.RuntimeConfig(st, status, stack))
        assert mask_hex(m, 7) == g["hex"], prefix
    assert mask_hex(eng.ComputeMask(eng.InitialConfig()), 7) == "b2"


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("K", [1, 4, 16])
def test_mask_agreement_cases(vectors, name, K):
    """Golden reference masks for sampled configs, at several context depths
    (K=1 forces many context-dependent tokens), twice (build then hit)."""
    case = vectors["mask_agreement"][name]
    vocab = [bytes.fromhex(h) for h in case["vocab_hex"]]
    eng = pk.DeviceEngine(pk.Automaton.load(flat(name)), vocab, context_depth=K)
    cfgs = [pk.RuntimeConfig(c["stack"][-1], c["status"], c["stack"]) for c in case["cases"]]
    for _ in range(2):
        masks, _ = fill_batch(eng, cfgs)
        for m, c in zip(masks, case["cases"]):
            assert mask_hex(m, len(vocab)) == c["hex"]


def test_dead_and_accepted_rows_are_empty():
    """runtime.cpp:282: non-alive configs get all-zero masks (and all -inf)."""
    eng = pk.DeviceEngine(pk.Automaton.load(flat("paren")), [b"a", b"("])
    cfgs = [pk.RuntimeConfig(0, pk.DEAD, [0]), pk.RuntimeConfig(0, pk.ACCEPTED, [0]),
            pk.RuntimeConfig(0, pk.ALIVE, [0])]
    masks, lg = fill_batch(eng, cfgs, logits=True)
    assert masks[0].sum() == 0 and masks[1].sum() == 0 and masks[2].sum() != 0
    lgf = lg.float().cpu().numpy()
    assert np.all(np.isneginf(lgf[0])) and np.all(np.isneginf(lgf[1]))


def host_seg_counts(eng, m, nseg):
    """Per (sequence, segment) {allowed regular tokens, allowed structural
    tokens} of bitmask rows m (EOS bit excluded): the fill's seg_counts."""
    bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, : eng.V + 1].astype(np.int64)
    bits[:, eng.V] = 0
    sbits = np.unpackbits(eng.structural.view(np.uint8), bitorder="little")[: eng.V + 1].astype(np.int64)
    out = np.zeros((m.shape[0], nseg * 2), dtype=np.int64)
    for s in range(nseg):
        lo, hi = s * 8192, min(eng.V + 1, (s + 1) * 8192)
        out[:, 2 * s] = bits[:, lo:hi].sum(1)
        out[:, 2 * s + 1] = (bits[:, lo:hi] * sbits[lo:hi]).sum(1)
    return out


def run_stream(eng, B, steps, seed, cap=1024, check_logits=False, fused=False):
    """Device decode loop: fill (+logits) then stream-sample + accept, as two
    API calls, (fused=True) one gm_decode_step_stream launch or
    (fused="split") gm_decode_step_stream_split."""
    batch = eng.batch(B, cap)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=DEV)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    lg = torch.randn((B, eng.V + 1), dtype=torch.bfloat16, device=DEV) if check_logits else None
    masks, tokens = [], []
    for _ in range(steps):
        if lg is not None:
            lg.normal_()
            before = lg.clone()
        if fused == "split":
            batch.decode_step_stream_split(seed, bitmask=bm, logits=lg, seg_counts=counts, tokens_out=toks)
        elif fused:
            batch.decode_step_stream(seed, bitmask=bm, logits=lg, tokens_out=toks)
        else:
            batch.fill(bm, lg, counts)
            batch.sample_stream_and_accept(bm, counts, seed, toks)
        batch.check()
        m = bm.cpu().numpy().view(np.uint32).copy()
        if fused in (False, "split"):
            assert np.array_equal(counts.cpu().numpy(), host_seg_counts(eng, m, batch.nseg))
        masks.append(m)
        tokens.append(toks.cpu().numpy().copy())
        if lg is not None:
            bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, : eng.V + 1].astype(bool)
            after = lg.float().cpu().numpy()
            assert np.array_equal(np.isneginf(after), ~bits | np.isneginf(before.float().cpu().numpy()))
            assert np.array_equal(after[bits], before.float().cpu().numpy()[bits])
    return batch, np.stack(masks, 1), np.stack(tokens, 1)


@pytest.mark.parametrize("fused", [False, True, "split"])
def test_json32k_stream_matches_golden(vectors, fused):
    """Config 1 replayed on the GPU: every mask digest, token and the final
    stacks equal the reference's (golden)."""
    g = vectors["json32k_stream"]
    vocab = pk.synth_vocab(32000)
    eng = pk.DeviceEngine(pk.Automaton.load(flat("json")), vocab)
    batch, masks, tokens = run_stream(eng, g["batch"], g["steps"], g["seed"], check_logits=True, fused=fused)
    assert tokens.tolist() == g["tokens"]
    for b in range(g["batch"]):
        for s in range(g["steps"]):
            assert hashlib.sha256(masks[b, s].tobytes()).hexdigest()[:32] == g["trace"][b][s]["mask"], (b, s)
        fin = g["final"][b]
        got = batch.get(b)
        assert got.stack == fin["stack"] and got.status == fin["status"]


@pytest.mark.parametrize("K,fused", [(2, False), (8, False), (12, True), (16, True), (16, False), (2, "split"),
                                     (12, "split"), (16, "split")])
def test_json128k_stream_matches_port(K, fused):
    """Config 2 shape (JSON, 128,255 tokens): GPU decode loop == C port loop
    (tokens every step, final stacks) for 24 sequences x 16 steps."""
    vocab = pk.synth_vocab(128255)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
    port = Port(f, vocab)
    B, steps, seed = 24, 16, 5
    batch, masks, tokens = run_stream(eng, B, steps, seed, fused=fused)
    _, ptoks, pstacks = port.decode_run(eng.structural, B, steps, seed, want_tokens=True, want_stacks=True)
    assert np.array_equal(tokens, ptoks)
    for b in range(B):
        d = pstacks[b, 0]
        got = batch.get(b)
        assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1]


def test_cache_pressure_paths():
    """Tiny context tables force the private (uncached) path; results must
    not change."""
    vocab = pk.synth_vocab(40000)
    f = flat("json")
    port = Port(f, vocab)
    B, steps, seed = 16, 10, 9
    _, ptoks, _ = port.decode_run(pk.structural_words(vocab), B, steps, seed, want_tokens=True)
    for slots in [1, 4, 1024]:
        eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=3, context_slots=slots)
        _, _, tokens = run_stream(eng, B, steps, seed)
        assert np.array_equal(tokens, ptoks), slots
        _, _, tokens = run_stream(eng, B, steps, seed, fused=True)  # warm cache, second batch
        assert np.array_equal(tokens, ptoks), slots
        _, _, tokens = run_stream(eng, B, steps, seed, fused="split")
        assert np.array_equal(tokens, ptoks), slots
        if slots <= 4:
            assert eng.info()["private_builds"] > 0


@pytest.mark.parametrize("name", ["expr", "json", "digits"])
def test_accept_tokens_matches_port(name):
    """Engine::Step over token bytes, batched: random (often invalid) tokens,
    EOS, skips (-1); statuses and stacks after every step equal the port's."""
    rng = random.Random(17)
    f = flat(name)
    import oracle
    acc = 0
    for e in oracle.read_flat(f)["edges"]:
        acc |= e["accepted"]
    alphabet = [b for b in range(256) if (acc >> b) & 1]
    vocab = sorted({bytes(rng.choice(alphabet) for _ in range(1 + rng.randrange(4))) for _ in range(300)})
    V = len(vocab)
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab)
    port = Port(f, vocab)
    B = 64
    batch = eng.batch(B, 512)
    cfgs = [port.initial() for _ in range(B)]
    toks_d = torch.zeros(B, dtype=torch.int32, device=DEV)
    status_d = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(40):
        toks = []
        for b in range(B):
            m = port.mask(cfgs[b])
            allowed = [t for t in range(V + 1) if (int(m[t >> 5]) >> (t & 31)) & 1]
            r = rng.random()
            if allowed and r < 0.8:
                t = rng.choice(allowed)
            elif r < 0.9:
                t = rng.randrange(V + 1)
            else:
                t = -1
            toks.append(t)
        toks_d.copy_(torch.tensor(toks, dtype=torch.int32))
        batch.accept(toks_d, status_d)
        batch.check()
        st = status_d.cpu().numpy()
        for b in range(B):
            if toks[b] >= 0:
                port.accept_token(cfgs[b], toks[b])
            want = port.get(cfgs[b])
            got = batch.get(b)
            assert got.status == want[1] == st[b]
            assert got.stack == want[2]
            if want[1] != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
                batch.set(b, pk.RuntimeConfig(cfgs[b].state, 0, [cfgs[b].stack[0]]))


def test_greedy_decode_matches_port():
    """Config 5 rule: argmax over allowed bf16 logits (ties -> lowest id)."""
    vocab = pk.synth_vocab(32000)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab)
    port = Port(f, vocab)
    B = 16
    batch = eng.batch(B)
    cfgs = [port.initial() for _ in range(B)]
    g = torch.Generator(device=DEV).manual_seed(0)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    for s in range(12):
        lg = torch.randn((B, eng.V + 1), generator=g, device=DEV).to(torch.bfloat16)
        if s % 3 == 0:
            lg[:, ::7] = 3.0  # ties
        batch.decode_step_greedy(lg, toks, bm)
        batch.check()
        host = lg.view(torch.int16).cpu().numpy().view(np.uint16)
        tk = toks.cpu().numpy()
        for b in range(B):
            m = port.mask(cfgs[b])
            t = port.greedy_pick(m, np.ascontiguousarray(host[b]))
            assert t == tk[b], (s, b)
            if t >= 0:
                port.accept_token(cfgs[b], t)
            if t < 0 or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            assert batch.get(b).stack == port.get(cfgs[b])[2]


@pytest.mark.parametrize("kind", ["zeros", "few_values", "specials"])
def test_greedy_ties_and_special_values(kind):
    """The packed 16-bit-key argmax (PairKeys): all-equal rows (lowest
    allowed id wins), few distinct values, and rows holding +-inf, -0.0 and
    NaNs (0xFFFF keys like a masked token) — equal to the port's 32-bit keys."""
    vocab = pk.synth_vocab(40000)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=8)
    port = Port(f, vocab)
    B = 24
    batch = eng.batch(B)
    cfgs = [port.initial() for _ in range(B)]
    rng = np.random.default_rng({"zeros": 1, "few_values": 2, "specials": 3}[kind])
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    for s in range(10):
        if kind == "zeros":
            host = np.zeros((B, eng.V + 1), np.uint16)
        elif kind == "few_values":
            host = rng.choice(np.array([0xBF80, 0x0000, 0x3F80, 0x4000], np.uint16), size=(B, eng.V + 1))
        else:
            host = rng.choice(np.array([0xFFFF, 0x7FC0, 0x7F80, 0xFF80, 0x8000, 0x0000, 0xC000], np.uint16),
                              size=(B, eng.V + 1), p=[0.3, 0.1, 0.02, 0.2, 0.18, 0.1, 0.1])
            host[: B // 3] = 0xFFFF  # rows of NaN 0xFFFF only
        lg = torch.from_numpy(host.view(np.int16)).to(DEV).view(torch.bfloat16)
        batch.decode_step_greedy(lg, toks)
        batch.check()
        tk = toks.cpu().numpy()
        for b in range(B):
            t = port.greedy_pick(port.mask(cfgs[b]), np.ascontiguousarray(host[b]))
            assert t == tk[b], (kind, s, b)
            if t >= 0:
                port.accept_token(cfgs[b], t)
            if t < 0 or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()


def test_stack_overflow_status():
    """A stack beyond the batch capacity yields GM_OVERFLOW, never a write
    past the end."""
    vocab = [b"[", b"]", b"1"]
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab)
    batch = eng.batch(1, 12)
    t = torch.zeros(1, dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    for _ in range(8):
        batch.accept(t, st)
    batch.check()
    assert int(st.item()) == pk.OVERFLOW


@pytest.mark.parametrize("name,flavor", [("schema", 0), ("sql", 1)])
def test_workload_grammar_stream_matches_port(name, flavor):
    """Configs 3/4: the repo-authored grammars, compiled by our own compiler
    (byte-identical to the reference builder, test_compiler.py), drive the
    GPU decode loop at 128k tokens; tokens every step and final stacks equal
    the C port's."""
    text = open(os.path.join(ROOT, "paper_2506_03887_b200", "grammars", name + ".bnf")).read()
    f = pk.Automaton.compile(text).save()
    vocab = pk.synth_vocab(128255, flavor)
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=12)
    port = Port(f, vocab)
    B, steps, seed = 16, 12, 9
    for fused in (False, True, "split"):
        batch, masks, tokens = run_stream(eng, B, steps, seed, fused=fused)
        _, ptoks, pstacks = port.decode_run(eng.structural, B, steps, seed, want_tokens=True, want_stacks=True)
        assert np.array_equal(tokens, ptoks), fused
        for b in range(B):
            d = pstacks[b, 0]
            got = batch.get(b)
            assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1]


@pytest.mark.parametrize("K,R", [(12, -1), (12, 1), (12, 3), (12, 8), (16, 4), (6, 5)])
def test_parent_based_context_builds(K, R):
    """New contexts built from their parent context (same stack top keyed R
    deep; only the parent's context-dependent tokens re-walked) give the same
    decode loop as full builds: tokens every step and final stacks equal the
    C port's."""
    vocab = pk.synth_vocab(128255)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K, parent_depth=R)
    port = Port(f, vocab)
    B, steps, seed = 24, 20, 11
    batch, masks, tokens = run_stream(eng, B, steps, seed, fused=True)
    _, ptoks, pstacks = port.decode_run(eng.structural, B, steps, seed, want_tokens=True, want_stacks=True)
    assert np.array_equal(tokens, ptoks)
    for b in range(B):
        d = pstacks[b, 0]
        got = batch.get(b)
        assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1]
    info = eng.info()
    assert (info["parent_builds"] > 0) == (R > 0)


def test_tokenizer_json_vocabulary_on_device():
    """A byte-level BPE vocabulary ingested from a tokenizer.json
    (paper_2506_03887_b200/tokenizer.py) drives the device loop exactly like
    the C port (tokens every step, final stacks)."""
    tokenizers = pytest.importorskip("tokenizers")
    from tokenizers import Tokenizer, decoders, models, pre_tokenizers, trainers
    from paper_2506_03887_b200 import tokenizer as tk
    corpus = ['{"name": "ada", "tags": ["x", "y"], "n": [1, 2, 30], "ok": true, "z": null}',
              '[{"a": {"b": []}}, "s p a c e", -12]'] * 50
    tok = Tokenizer(models.BPE())
    tok.pre_tokenizer = pre_tokenizers.ByteLevel(add_prefix_space=False)
    tok.decoder = decoders.ByteLevel()
    tok.train_from_iterator(corpus, trainers.BpeTrainer(vocab_size=1500, show_progress=False,
                                                        initial_alphabet=pre_tokenizers.ByteLevel.alphabet()))
    tok.add_special_tokens(["<|endoftext|>"])
    tv = tk.from_tokenizer_json(tok.to_str())
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), tv.tokens, context_depth=12)
    port = Port(f, tv.tokens)
    B, steps, seed = 16, 24, 3
    batch, masks, tokens = run_stream(eng, B, steps, seed, fused=True)
    _, ptoks, pstacks = port.decode_run(eng.structural, B, steps, seed, want_tokens=True, want_stacks=True)
    assert np.array_equal(tokens, ptoks)
    for b in range(B):
        d = pstacks[b, 0]
        got = batch.get(b)
        assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1]


@pytest.mark.parametrize("T,k,p,ties", [(1.0, 0, 1.0, False), (0.7, 50, 1.0, False), (1.3, 0, 0.9, False),
                                        (0.5, 20, 0.8, False), (2.0, 3, 0.5, True), (1.0, 0, 0.95, True),
                                        (0.05, 0, 1.0, False), (1.0, 1, 1.0, True), (1.0, 0, 1.0, "wide"),
                                        (40.0, 200, 0.9, "wide")])
def test_sample_decode_step_matches_port(T, k, p, ties):
    """gm_decode_step_sample (fill + temperature/top-k/top-p sampler + accept,
    one host call, no round trip) == the C port's rule step by step: masks,
    sampled tokens, stacks.  `ties` quantizes the logits to few values so the
    tie rules (thresholds keep ties, draws walk ties in id order) are hit;
    "wide" spreads them over 2^-40..2^40 (more than 24 sign+exponent bytes:
    the sampler's two-pass histogram path instead of one-pass key counts)."""
    vocab = pk.synth_vocab(128255)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=12)
    port = Port(f, vocab)
    B, steps, seed = 12, 10, 77
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    cfgs = [port.initial() for _ in range(B)]
    g = torch.Generator(device=DEV).manual_seed(5)
    for s in range(steps):
        lg = torch.randn((B, eng.V + 1), dtype=torch.float32, device=DEV, generator=g)
        if ties == "wide":
            lg = torch.sign(lg) * torch.exp2(torch.rand((B, eng.V + 1), device=DEV, generator=g) * 80 - 40)
        elif ties:
            lg = torch.round(lg * 2) / 2
        lg = lg.to(torch.bfloat16)
        batch.decode_step_sample(lg, temperature=T, top_k=k, top_p=p, seed=seed, tokens_out=toks, bitmask=bm)
        batch.check()
        got = bm.cpu().numpy().view(np.uint32)
        rows = lg.view(torch.int16).cpu().numpy().view(np.uint16)
        tk = toks.cpu().numpy()
        for b in range(B):
            want = port.mask(cfgs[b])
            assert np.array_equal(got[b], want), (b, s)
            tok = port.sample_pick(want, rows[b], T, k, p, Port.stream_draw(seed, b, s))
            assert tok == tk[b], (b, s, tok, tk[b])
            if tok >= 0:
                port.accept_token(cfgs[b], tok)
            if tok < 0 or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            assert batch.get(b).stack == port.get(cfgs[b])[2], (b, s)


@pytest.mark.parametrize("name", FIXTURES)
def test_allowed_terminals_matches_port(vectors, name):
    """Engine::AllowedTerminals on the device (gm_allowed_terminals) == the C
    port's on every sampled configuration (test_runtime.cpp:116-137 pins the
    reference's own against viability)."""
    case = vectors["mask_agreement"][name]
    vocab = [bytes.fromhex(h) for h in case["vocab_hex"]]
    f = flat(name)
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab)
    port = Port(f, vocab)
    for c in case["cases"]:
        cfg = pk.RuntimeConfig(c["stack"][-1], c["status"], c["stack"])
        got = eng.AllowedTerminals(cfg)
        pc = port.config(c["status"], c["stack"])
        want = port.allowed(pc) if c["status"] == 0 else (0, False)
        port.free(pc)
        assert got == want, (c["stack"], got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("grammar,flavor,K,B,two", [("json", 0, 16, 1024, False), ("schema", 0, 16, 1024, False),
                                                   ("json", 0, 16, 1536, False), ("json", 0, 16, 1536, True)])
def test_split_step_large_batch(grammar, flavor, K, B, two, monkeypatch):
    """gm_decode_step_stream_split at a batch that fills several waves (the
    accepts overlap the fill and pure-CI sequences sample from the context
    cache; accept CTAs inside the fill's grid, or — PRE3_SPLIT_TWO_KERNELS —
    the separate accept kernel): tokens, masks and stacks equal the two-call
    loop's, and the first 48 sequences' tokens equal the C port's."""
    if two:
        monkeypatch.setenv("PRE3_SPLIT_TWO_KERNELS", "1")
    if grammar == "json":
        f = flat("json")
    else:
        text = open(os.path.join(ROOT, "paper_2506_03887_b200", "grammars", grammar + ".bnf")).read()
        f = pk.Automaton.compile(text).save()
    vocab = pk.synth_vocab(128255, flavor)
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
    eng.prewarm(512, 200, seed=0xC0FFEE)
    steps, seed = 8, 13
    assert eng.batch(B).split_step_launches == (2 if two else 1)
    b1, m1, t1 = run_stream(eng, B, steps, seed, fused="split", check_logits=True)
    b2, m2, t2 = run_stream(eng, B, steps, seed)
    assert np.array_equal(t1, t2)
    assert np.array_equal(m1, m2)
    for b in range(0, B, 37):
        assert b1.get(b).stack == b2.get(b).stack
    port = Port(f, vocab)
    _, ptoks, _ = port.decode_run(eng.structural, 48, steps, seed, want_tokens=True)
    assert np.array_equal(t1[:48], ptoks)


def test_structural_change_recounts_built_contexts():
    """Changing the structural token set after contexts were built recounts
    their per-segment counts (the split step samples pure-CI sequences from
    them): the decode loop still equals the C port's under the new set."""
    vocab = pk.synth_vocab(128255)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=12)
    eng.prewarm(256, 100, seed=3)
    rng = np.random.default_rng(5)
    words = rng.integers(0, 2**32, size=eng.W, dtype=np.uint64).astype(np.uint32) & eng.structural
    eng.set_structural(words)
    port = Port(f, vocab)
    B, steps, seed = 32, 12, 21
    _, _, tokens = run_stream(eng, B, steps, seed, fused="split")
    _, ptoks, _ = port.decode_run(eng.structural, B, steps, seed, want_tokens=True)
    assert np.array_equal(tokens, ptoks)


def _random_grammar(rng):
    """Same generator as test_compiler.py's differential fuzzing: small
    grammars over the terminals a b c ( ) , with epsilon rules, recursion
    and conflicts (the ones that do not compile are skipped)."""
    names = ["A", "B", "C", "D", "E"][: rng.randint(1, 5)]
    lines = []
    for n in names:
        alts = []
        for _ in range(rng.randint(1, 3)):
            syms = []
            for _ in range(rng.randint(0, 4)):
                if rng.random() < 0.45:
                    syms.append(rng.choice(names))
                else:
                    syms.append('"' + rng.choice("abc(),") + '"')
            alts.append(" ".join(syms))
        lines.append(n + " -> " + " | ".join(alts))
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", range(6))
def test_random_grammars_decode_matches_port(seed):
    """Random grammars compiled by our compiler, a vocabulary of every string
    of 1-3 characters over the grammar's alphabet (258 tokens): the device
    decode loop in all three step forms, with context keys 1 and 3 deep (so
    context-dependent walks are common), equals the C port's — tokens every
    step, final stacks and statuses."""
    import itertools
    rng = random.Random(7000 + seed)
    alphabet = [bytes([c]) for c in b"abc(),"]
    vocab = [b"".join(p) for n in (1, 2, 3) for p in itertools.product(alphabet, repeat=n)]
    done = 0
    while done < 12:
        text = _random_grammar(rng)
        try:
            a = pk.Automaton.compile(text)
        except pk.GmError:
            continue
        f = a.save()
        port = Port(f, vocab)
        B, steps, s = 8, 12, rng.randrange(1 << 30)
        for K in (1, 3):
            eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
            _, ptoks, pstacks = port.decode_run(eng.structural, B, steps, s, want_tokens=True, want_stacks=True)
            for mode in (False, True, "split"):
                batch, _, tokens = run_stream(eng, B, steps, s, fused=mode, check_logits=True)
                assert np.array_equal(tokens, ptoks), (text, K, mode)
                for b in range(B):
                    d = pstacks[b, 0]
                    got = batch.get(b)
                    assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1], (text, K, mode)
        done += 1


@pytest.mark.parametrize("grammar,flavor,K,B", [("json", 0, 16, 1024), ("sql", 1, 20, 2048)])
def test_split_step_soak_matches_two_call_loop(grammar, flavor, K, B):
    """Race check of the overlapped split step (the accept kernel runs under
    the fill; pure-CI sequences sample from the context cache while the fill
    writes their bitmask rows): 400 steps of B sequences give the same token
    every step as the serial two-call loop on the same engine."""
    if grammar == "json":
        f = flat("json")
    else:
        text = open(os.path.join(ROOT, "paper_2506_03887_b200", "grammars", grammar + ".bnf")).read()
        f = pk.Automaton.compile(text).save()
    vocab = pk.synth_vocab(128255, flavor)
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K, context_slots=1 << 17)
    steps, seed = 400, 77
    runs = []
    for split in (True, False):
        batch = eng.batch(B, 1024)
        bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
        counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=DEV)
        lg = torch.randn((B, eng.V + 1), dtype=torch.bfloat16, device=DEV)
        toks = torch.zeros((steps, B), dtype=torch.int32, device=DEV)
        for s in range(steps):
            if split:
                batch.decode_step_stream_split(seed, bitmask=bm, logits=lg, seg_counts=counts, tokens_out=toks[s])
            else:
                batch.fill(bm, lg, counts)
                batch.sample_stream_and_accept(bm, counts, seed, toks[s])
        batch.check()
        runs.append(toks.cpu().numpy())
    assert np.array_equal(runs[0], runs[1])


def test_cpp_device_engine_known_answers(vectors, tmp_path):
    """The reference-side C++ binding (include/pre3/device_engine.hpp:
    InitialConfig / AcceptToken / ComputeMask / AllowedTerminals on the GPU)
    reproduces the reference's paren known answers (test_runtime.cpp:184-206:
    masks b2, 40, eos-only) and the C port's stacks, built with g++ against
    the C ABI."""
    import subprocess
    lib_dir = os.path.join(ROOT, "paper_2506_03887_b200")
    exe = tmp_path / "engine_cli"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "engine_cli.cpp"), "-o", str(exe), "-L", lib_dir,
                    "-lpre3gmask", f"-Wl,-rpath,{lib_dir}", "-L/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    vocab = vectors["paren7"]["vocab"]
    prefixes = [""] + sorted(vectors["paren7"]["masks"])
    lines = [" ".join(str(vocab.index(c)) for c in p) for p in prefixes]
    path = tmp_path / "paren.p3dpda"
    path.write_bytes(flat("paren"))
    env = dict(os.environ, PRE3_CLI_SNAPSHOT="1")
    out = subprocess.run([str(exe), str(path)] + vocab, input="\n".join(lines) + "\n", capture_output=True,
                         text=True, check=True, env=env).stdout.splitlines()
    assert out[-1].startswith("snapshot ok") and int(out[-1].split()[2]) > 0, out[-1]
    out = out[:-1]
    assert len(out) == len(prefixes)
    port = Port(flat("paren"), [t.encode() for t in vocab])
    for p, row in zip(prefixes, out):
        f = row.split()
        words = np.array([int(x, 16) for x in f[1:f.index("eos")]], dtype=np.uint32)
        want = "b2" if p == "" else vectors["paren7"]["masks"][p]["hex"]
        assert mask_hex(words, 7) == want, p
        assert int(f[f.index("eos") + 1]) == int(words[0] >> 7 & 1), p
        c = port.initial()
        for ch in p:
            port.accept_token(c, vocab.index(ch))
        _, status, stack = port.get(c)
        assert int(f[f.index("status") + 1]) == status, p
        assert [int(x) for x in f[f.index("stack") + 1:]] == stack, p


def test_time_next_fill_brackets_one_fill():
    """gm_batch_time_next_fill: the next fill kernel (here inside the split
    step) is bracketed by the two events; the hook is one-shot."""
    vocab = pk.synth_vocab(32000)
    eng = pk.DeviceEngine(pk.Automaton.load(flat("json")), vocab)
    B = 64
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e1.record()
    torch.cuda.synchronize()
    batch.time_next_fill(e0, e1)
    batch.decode_step_stream_split(3, bitmask=bm, tokens_out=toks)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    assert 0.0 < t < 50.0
    batch.decode_step_stream_split(3, bitmask=bm, tokens_out=toks)  # not timed: the events stay put
    torch.cuda.synchronize()
    assert e0.elapsed_time(e1) == t


def test_dead_end_restarts_like_the_port():
    """A grammar whose non-productive rules lead to configurations with no
    allowed token and no EOS (found by scripts/gpu_fuzz.py): the sampled token
    is -1 and the sequence restarts from InitialConfig in every step form,
    as in the C port's decode loop."""
    import itertools
    text = 'A -> "a" "c" ")" | D D "b" | "(" B B\nB -> D "a"\nC ->  | \nD -> D "c" D A\n'
    alphabet = [bytes([c]) for c in b"abc(),"]
    vocab = [b"".join(p) for n in (1, 2, 3) for p in itertools.product(alphabet, repeat=n)]
    f = pk.Automaton.compile(text).save()
    port = Port(f, vocab)
    for K in (1, 8):
        eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
        _, ptoks, _ = port.decode_run(eng.structural, 16, 16, 1000, want_tokens=True, want_stacks=True)
        assert (ptoks < 0).any()  # the dead end is reached
        for mode in (False, True, "split"):
            _, _, tokens = run_stream(eng, 16, 16, 1000, fused=mode)
            assert np.array_equal(tokens, ptoks), (K, mode)


def test_wide_random_grammar_fuzz_sample():
    """A 12-grammar sample of scripts/gpu_fuzz2.py (multi-byte literals,
    random vocabularies, small stack capacities; stream/greedy/temperature
    steps, AllowedTerminals, tiny context tables, a 1,024-sequence
    split-vs-two-call check) — the full sweeps are recorded in profiles/."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gpu_fuzz2", os.path.join(ROOT, "scripts", "gpu_fuzz2.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    done, _, runs = m.run(12, 31337)
    assert done == 12 and runs > 100


@pytest.mark.parametrize("B", [1, 3, 33])
def test_split_step_odd_batches(B):
    """Batch sizes that leave partial CTAs (accept: 4 warps per CTA; fill: 8
    items per CTA): the split step still equals the C port."""
    vocab = pk.synth_vocab(40000)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=8)
    port = Port(f, vocab)
    _, ptoks, pstacks = port.decode_run(eng.structural, B, 14, 23, want_tokens=True, want_stacks=True)
    batch, _, tokens = run_stream(eng, B, 14, 23, fused="split", check_logits=True)
    assert np.array_equal(tokens, ptoks)
    for b in range(B):
        d = pstacks[b, 0]
        assert batch.get(b).stack == pstacks[b, 2:2 + d].tolist()


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("K", [1, 8])
def test_acceptance_criterion3_on_device(name, K):
    """Acceptance criterion 3 at the reference's own scale and seeds
    (acceptance_main.cpp:202-219; tests/golden/acceptance_masks.json from the
    reference's SampleVocab/SampleConfigs): all 200 configurations x 1,000
    tokens per fixture, device masks == the reference's, at context depths 1
    (most tokens context-dependent) and 8."""
    with open(os.path.join(GOLDEN, "acceptance_masks.json")) as f:
        case = json.load(f)["fixtures"][name]
    vocab = [bytes.fromhex(h) for h in case["vocab_hex"]]
    eng = pk.DeviceEngine(pk.Automaton.load(flat(name)), vocab, context_depth=K)
    cfgs = [pk.RuntimeConfig(c["stack"][-1], c["status"], c["stack"]) for c in case["cases"]]
    masks, _ = fill_batch(eng, cfgs, logits=True)
    for m, c in zip(masks, case["cases"]):
        assert mask_hex(m, len(vocab)) == c["hex"], c["stack"]


def test_python_binding_rejects_bad_tensors():
    """The binding checks dtype, device, row count and inner layout before a
    raw pointer reaches a kernel (a float32 logits row would otherwise be
    read as bf16, a short tensor written out of bounds)."""
    eng = pk.DeviceEngine(pk.Automaton.load(flat("paren")), [b"a", b"("])
    b = eng.batch(4)
    bm = torch.zeros((4, eng.W), dtype=torch.int32, device=DEV)
    with pytest.raises(TypeError):
        b.fill(bm, torch.zeros((4, 3), dtype=torch.float32, device=DEV))
    with pytest.raises(ValueError):
        b.fill(torch.zeros((3, eng.W), dtype=torch.int32, device=DEV))
    with pytest.raises(ValueError):
        b.fill(bm.cpu())
    with pytest.raises(ValueError):
        b.accept(torch.zeros(2, dtype=torch.int32, device=DEV))
    b.fill(bm, torch.zeros((4, 3), dtype=torch.bfloat16, device=DEV))
    b.check()


def test_token_id_beyond_vocabulary_kills_the_sequence():
    """an id > V (a model special the caller did not remap) makes
    the sequence dead instead of reading past the token tables."""
    eng = pk.DeviceEngine(pk.Automaton.load(flat("paren")), [b"a", b"(", b")"])
    b = eng.batch(2)
    st = torch.zeros(2, dtype=torch.int32, device=DEV)
    b.accept(torch.tensor([4, 1 << 30], dtype=torch.int32, device=DEV), st)
    b.check()
    assert st.cpu().tolist() == [pk.DEAD, pk.DEAD]


@pytest.mark.parametrize("greedy", [False, True])
def test_captured_graph_steps_match_eager_and_port(greedy):
    """gm_decode_graph_create / gm_graph_launch: 12 captured steps replayed
    twice (24 steps) give, step for step, the eager loop's tokens and the C
    port's; a replay from a state the graph was not captured at is refused."""
    vocab = pk.synth_vocab(40000)
    f = flat("json")
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=12)
    port = Port(f, vocab)
    B, G, seed = 48, 12, 31
    V1 = eng.V + 1
    logits = [torch.empty((B, V1), dtype=torch.bfloat16, device=DEV) for _ in range(3)]
    for k, t in enumerate(logits):
        pk.synth_logits(t, k, 77)
    kw = dict(greedy_rows=3, logit_seed=77) if greedy else {}
    _, ptoks, pstacks = port.decode_run(eng.structural, B, 2 * G, seed, want_tokens=True, want_stacks=True, **kw)
    batch = eng.batch(B)
    bms = [torch.zeros((B, eng.W), dtype=torch.int32, device=DEV) for _ in range(G)]
    cnt = [torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV) for _ in range(G)]
    tks = [torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(G)]
    graph = batch.capture_steps(G, greedy=greedy, seed=seed, bitmask=bms, logits=[logits[i % 3] for i in range(G)],
                                seg_counts=None if greedy else cnt, tokens_out=tks)
    got = []
    for rep in range(2):
        graph.launch()
        batch.check()
        got.append(torch.stack(tks, 1).cpu().numpy())
        for i in (0, G - 1):
            m = bms[i].cpu().numpy().view(np.uint32)
            assert np.array_equal(oracle_mask_hashes(m), port_hashes(port, eng, B, 2 * G, seed, kw)[:, rep * G + i])
    assert np.array_equal(np.concatenate(got, 1), ptoks)
    for b in range(B):
        d = pstacks[b, 0]
        assert batch.get(b).stack == pstacks[b, 2:2 + d].tolist()
    # one eager step moves the batch off the graph's start state
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    if greedy:
        batch.decode_step_greedy(logits[0], tokens_out=toks)
    else:
        batch.decode_step_stream_split(seed, tokens_out=toks)
    with pytest.raises(pk.GmError):
        graph.launch()


_PORT_HASHES = {}


def port_hashes(port, eng, B, steps, seed, kw):
    key = (id(port), B, steps, seed, tuple(sorted(kw.items())))
    if key not in _PORT_HASHES:
        _PORT_HASHES[key] = port.decode_run(eng.structural, B, steps, seed, want_mask_hashes=True, **kw)[3]
    return _PORT_HASHES[key]


def oracle_mask_hashes(m):
    import oracle
    return oracle.mask_hashes(m)
