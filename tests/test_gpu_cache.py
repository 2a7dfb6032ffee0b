"""The context cache's robustness:

* context-table snapshots ("P3GMCTX1", gm_engine_snapshot_save/load): a
  loaded table reproduces the saved one byte for byte and the masks of a
  decode loop on it equal the C port's; other automata / vocabularies /
  options are refused, altered or truncated data is rejected;
* builds queued by a batch that stops stepping are built by whichever batch
  needs them (no fill gives up waiting and walks a whole segment);
* tokens whose walk pushes up to the 256-entry walk overlay (60 opening
  brackets) give the port's masks; past it, a shared slot marks the token
  context-dependent (never a cached reject) and the full-stack walk raises
  GM_ERR_STACK_OVERFLOW — loudly, not a wrong mask.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2506_03887_b200 as pk
from oracle import Port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def flat(name):
    with open(os.path.join(os.path.dirname(__file__), "golden", f"{name}.p3dpda"), "rb") as f:
        return f.read()


def engine(vocab, K=8, slots=4096, R=0, f=None):
    return pk.DeviceEngine(pk.Automaton.load(f or flat("json")), vocab, context_depth=K, context_slots=slots,
                           parent_depth=R)


def split_loop(eng, B, steps, seed, stats=False):
    """gm_decode_step_stream_split steps; per-step mask hashes and tokens."""
    batch = eng.batch(B)
    if stats:
        batch.set_stats(True)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    hashes, toks = [], []
    for _ in range(steps):
        batch.decode_step_stream_split(seed, bitmask=bm, seg_counts=cnt, tokens_out=tk)
        batch.check()
        hashes.append(oracle.mask_hashes(bm.cpu().numpy().view(np.uint32)))
        toks.append(tk.cpu().numpy().copy())
    return batch, np.stack(hashes, 1), np.stack(toks, 1)


def port_run(vocab, structural, B, steps, seed, f=None):
    port = Port(f or flat("json"), vocab)
    _, toks, stk, hashes = port.decode_run(structural, B, steps, seed, want_tokens=True, want_stacks=True,
                                           want_mask_hashes=True)
    return toks, stk, hashes


@pytest.fixture(scope="module")
def vocab():
    return pk.synth_vocab(30000)


def test_snapshot_roundtrip_reproduces_table_and_masks(vocab, tmp_path):
    a = engine(vocab)
    a.prewarm(256, 120, seed=0xC0FFEE)
    used = a.info()["context_slots_used"]
    assert used > 50
    path = str(tmp_path / "ctx.p3gmctx")
    size = a.save_contexts(path)
    blob = a.save_contexts()
    assert size == len(blob) and open(path, "rb").read() == blob and blob[:8] == b"P3GMCTX1"
    b = engine(vocab)
    b.load_contexts(path)
    assert b.info()["context_slots_used"] == used
    assert b.save_contexts() == blob  # the loaded table is the saved one
    B, steps, seed = 48, 24, 17
    batch, hashes, toks = split_loop(b, B, steps, seed, stats=True)
    ptoks, pstk, phashes = port_run(vocab, b.structural, B, steps, seed)
    assert np.array_equal(hashes, phashes) and np.array_equal(toks, ptoks)
    for i in range(B):
        assert batch.get(i).stack == pstk[i, 2:2 + pstk[i, 0]].tolist()


def test_snapshot_refuses_other_engines_and_bad_data(vocab):
    a = engine(vocab)
    a.prewarm(128, 40)
    blob = a.save_contexts()
    for other in (dict(K=12), dict(slots=8192), dict(R=-1)):
        with pytest.raises(pk.SnapshotMismatchError):
            engine(vocab, **other).load_contexts(blob)
    with pytest.raises(pk.SnapshotMismatchError):
        engine(vocab[:-1] + [b"\x01zz"]).load_contexts(blob)  # another vocabulary
    with pytest.raises(pk.SnapshotMismatchError):
        engine(vocab, f=flat("expr")).load_contexts(blob)  # another automaton
    bad = bytearray(blob)
    bad[len(bad) // 2] ^= 0x40
    with pytest.raises(pk.SerializeError):
        engine(vocab).load_contexts(bytes(bad))
    with pytest.raises(pk.SerializeError):
        engine(vocab).load_contexts(blob[:-4])
    with pytest.raises(pk.SerializeError):
        engine(vocab).load_contexts(b"P3GMCTX0" + blob[8:])
    full = engine(vocab)
    full.prewarm(16, 4)
    with pytest.raises(pk.GmError):
        full.load_contexts(blob)  # the table is not empty


def test_builds_queued_by_an_idle_batch_are_built_by_others(vocab):
    """Batch A steps 3 times and stops: its last lookups queued builds of the
    contexts its sequences reach next.  Batch B replays the same streams on
    the same engine: it meets those contexts, builds them itself, and never
    falls back to walking a whole segment (which the 2 ms wait used to cause)."""
    eng = engine(vocab, slots=4096)
    B, seed = 64, 23
    idle, _, _ = split_loop(eng, B, 3, seed)
    batch, hashes, toks = split_loop(eng, B, 14, seed, stats=True)
    st = batch.fill_stats()
    assert st["build_wait_timeouts"] == 0, st
    ptoks, _, phashes = port_run(vocab, eng.structural, B, 14, seed)
    assert np.array_equal(hashes, phashes) and np.array_equal(toks, ptoks)
    del idle


def deep_vocab(base, n):
    """The JSON test vocabulary plus tokens of n opening brackets (each '['
    pushes 2 entries: n = 60 passes the old 64-entry walk overlay)."""
    extra = [b"[" * k for k in range(2, n + 1)] + [b"[" * k + b"1" for k in (n // 2, n)]
    return [t for t in base if t not in set(extra)] + extra


@pytest.mark.parametrize("K", [4, 12])
def test_long_pushing_tokens_match_the_port(vocab, K):
    voc = deep_vocab(vocab[:8000], 60)
    eng = engine(voc, K=K, slots=1024)
    B, steps, seed = 32, 20, 5
    batch, hashes, toks = split_loop(eng, B, steps, seed)
    ptoks, pstk, phashes = port_run(voc, eng.structural, B, steps, seed)
    assert np.array_equal(hashes, phashes) and np.array_equal(toks, ptoks)
    # the long tokens were allowed on the way (the mask really exercised them)
    port = Port(flat("json"), voc)
    m = port.mask(port.initial())
    t40 = voc.index(b"[" * 60)
    assert (int(m[t40 >> 5]) >> (t40 & 31)) & 1
    dev = eng.ComputeMask(eng.InitialConfig())
    assert np.array_equal(dev, m)


def test_walk_past_the_overlay_fails_loudly(vocab):
    """A token pushing more than 256 entries (400 '[') cannot be walked: the
    fill raises GM_ERR_STACK_OVERFLOW instead of returning a wrong mask."""
    voc = vocab[:2000] + [b"[" * 400]
    eng = engine(voc, K=4, slots=256)
    with pytest.raises(pk.StackOverflowError):
        eng.ComputeMask(eng.InitialConfig())


# ---------------------------------------------------------------- eviction
def test_auto_eviction_keeps_every_mask_exact(vocab):
    """A 64-row table that keeps evicting (CLOCK: rows not referenced since
    the previous eviction, never those a fill is about to read or a pending
    build needs): every step's masks and tokens equal the port's."""
    eng = pk.DeviceEngine(pk.Automaton.load(flat("json")), vocab, context_depth=8, context_slots=64,
                          auto_evict_free=24)
    B, steps, seed = 40, 48, 29
    batch, hashes, toks = split_loop(eng, B, steps, seed)
    ptoks, pstk, phashes = port_run(vocab, eng.structural, B, steps, seed)
    assert np.array_equal(hashes, phashes) and np.array_equal(toks, ptoks)
    for i in range(B):
        assert batch.get(i).stack == pstk[i, 2:2 + pstk[i, 0]].tolist()
    st = eng.cache_stats()
    assert st["evictions"] > 0 and st["rows_evicted"] > 0, st
    assert st["rows_in_use"] + st["rows_free"] == st["rows"] == 64, st


def test_explicit_eviction_between_steps_and_graph_replays(vocab):
    """gm_engine_evict between eager steps and between replays of a captured
    graph (rows never move, so the graph's baked-in state stays valid)."""
    eng = engine(vocab, K=8, slots=256)
    B, G, seed = 32, 6, 41
    batch = eng.batch(B)
    tks = [torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(G)]
    graph = batch.capture_steps(G, seed=seed, tokens_out=tks)
    got = []
    for rep in range(4):
        graph.launch()
        batch.check()
        got.append(torch.stack(tks, 1).cpu().numpy())
        used = eng.cache_stats()["rows_in_use"]
        eng.evict()
        torch.cuda.synchronize()
        st = eng.cache_stats()
        assert st["rows_in_use"] <= used and st["rows_in_use"] + st["rows_free"] == 256
    ptoks, pstk, _ = port_run(vocab, eng.structural, B, 4 * G, seed)
    assert np.array_equal(np.concatenate(got, 1), ptoks)
    for i in range(B):
        assert batch.get(i).stack == pstk[i, 2:2 + pstk[i, 0]].tolist()
    # two evictions in a row with nothing referenced in between: the second
    # frees what the first kept only for its reference bit
    eng.evict()
    eng.evict()
    torch.cuda.synchronize()
    assert eng.cache_stats()["rows_in_use"] <= 2 * B  # next-fill rows and their parents


def test_table_full_at_128k_matches_the_port():
    """Configs' vocabulary size with an 8-row table and no eviction: most
    sequences fall back to private rows (built from their whole stack every
    step) and the masks stay exact."""
    voc = pk.synth_vocab(128255)
    eng = pk.DeviceEngine(pk.Automaton.load(flat("json")), voc, context_depth=8, context_slots=8)
    B, steps, seed = 16, 10, 3
    batch, hashes, toks = split_loop(eng, B, steps, seed, stats=True)
    assert batch.fill_stats()["private_fills"] > 0
    ptoks, _, phashes = port_run(voc, eng.structural, B, steps, seed)
    assert np.array_equal(hashes, phashes) and np.array_equal(toks, ptoks)
