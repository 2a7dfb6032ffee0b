"""Call sequences a decode loop does not take, on the device path (-m gpu):

* the mask filled again and again on unchanged sequences (ComputeMask twice,
  `runtime.cpp:280-287`, has no side effects) — past the 6-fill period of the
  heavy-list tags, so a fill can never read context rows or heavy-list
  entries a lookup wrote for an older fill;
* a sample without accept, then a fill;
* a CUDA graph captured right after such fills;
* two batches of one engine stepping concurrently on two CUDA streams.

Every mask is compared with the C port's on the sequences' current stacks.
Context depth 2 leaves many context-dependent tokens, so the fills schedule
heavy segments (the heavy-list path these sequences exercise).
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


def flat():
    with open(os.path.join(os.path.dirname(__file__), "golden", "json.p3dpda"), "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def setup():
    vocab = pk.synth_vocab(20000)
    eng = pk.DeviceEngine(pk.Automaton.load(flat()), vocab, context_depth=2, context_slots=4096)
    return vocab, eng, Port(flat(), vocab)


def port_masks(port, batch, B):
    rows = []
    for b in range(B):
        c = batch.get(b)
        cfg = port.config(c.status, c.stack)
        rows.append(port.mask(cfg))
        port.free(cfg)
    return np.stack(rows)


def test_repeated_fills_and_sample_without_accept(setup):
    vocab, eng, port = setup
    B = 48
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(7):  # varied stacks; a fill number that is not 0 mod 6
        batch.decode_step_stream_split(5, bitmask=bm, seg_counts=cnt, tokens_out=tk)
    batch.check()
    want = port_masks(port, batch, B)
    assert len({r.tobytes() for r in want}) > 4
    for i in range(14):  # two and a half tag periods of fills on the same stacks
        bm.zero_()
        batch.fill(bm, None, cnt)
        batch.check()
        assert np.array_equal(bm.cpu().numpy().view(np.uint32), want), f"repeated fill {i}"
    # Sample (no accept), fill, then the two-call step: still the same stacks.
    batch.sample_stream(bm, cnt, 5, tk)
    bm.zero_()
    batch.fill(bm, None, cnt)
    batch.check()
    assert np.array_equal(bm.cpu().numpy().view(np.uint32), want)
    batch.sample_stream_and_accept(bm, cnt, 5, tk)
    batch.check()
    bm.zero_()
    batch.fill(bm, None, cnt)
    batch.check()
    assert np.array_equal(bm.cpu().numpy().view(np.uint32), port_masks(port, batch, B))


def test_graph_captured_after_repeated_fills(setup):
    """Fresh sequences, fills only, then a 6-step graph: the graph's steps are
    the port's decode loop from InitialConfig (draws 0..5)."""
    vocab, eng, port = setup
    B, seed, steps = 40, 11, 6
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    for _ in range(13):
        batch.fill(bm, None, cnt)
    batch.check()
    bms = [torch.zeros((B, eng.W), dtype=torch.int32, device=DEV) for _ in range(steps)]
    cns = [torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV) for _ in range(steps)]
    tks = [torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(steps)]
    g = batch.capture_steps(steps, seed=seed, bitmask=bms, seg_counts=cns, tokens_out=tks)
    g.launch()
    torch.cuda.synchronize()
    batch.check()
    structural = oracle.structural_words(vocab)
    _, toks, _, hashes = port.decode_run(structural, B, steps, seed, want_tokens=True, want_stacks=True,
                                         want_mask_hashes=True)
    got_h = np.stack([oracle.mask_hashes(x.cpu().numpy().view(np.uint32)) for x in bms], 1)
    got_t = np.stack([x.cpu().numpy() for x in tks], 1)
    assert np.array_equal(got_h, hashes)
    assert np.array_equal(got_t, toks)


@pytest.mark.parametrize("slots", [2048, 16])
def test_two_batches_step_concurrently_on_two_streams(slots):
    """Two batches of one engine decode at the same time on two CUDA streams
    (they share the context cache: lookups, inserts, builds and parent links
    race; 16 slots: the table fills and sequences fall back to private rows):
    every step's mask and token equal the port's decode loop."""
    vocab = pk.synth_vocab(20000)
    eng = pk.DeviceEngine(pk.Automaton.load(flat()), vocab, context_depth=6, context_slots=slots, parent_depth=3)
    port = Port(flat(), vocab)
    structural = oracle.structural_words(vocab)
    B, steps = 64, 30
    seeds = (101, 202)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    batches = [eng.batch(B), eng.batch(B)]
    bms = [[torch.zeros((B, eng.W), dtype=torch.int32, device=DEV) for _ in range(steps)] for _ in range(2)]
    cns = [torch.zeros((B, 2 * batches[0].nseg), dtype=torch.int32, device=DEV) for _ in range(2)]
    tks = [[torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(steps)] for _ in range(2)]
    torch.cuda.synchronize()
    for s in range(steps):  # interleaved launches, no synchronization between the streams
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                batches[i].decode_step_stream_split(seeds[i], bitmask=bms[i][s], seg_counts=cns[i], tokens_out=tks[i][s],
                                                    stream=streams[i].cuda_stream)
    torch.cuda.synchronize()
    for i in range(2):
        batches[i].check(stream=streams[i].cuda_stream)
        _, toks, _, hashes = port.decode_run(structural, B, steps, seeds[i], want_tokens=True, want_stacks=True,
                                             want_mask_hashes=True)
        got_h = np.stack([oracle.mask_hashes(x.cpu().numpy().view(np.uint32)) for x in bms[i]], 1)
        got_t = np.stack([x.cpu().numpy() for x in tks[i]], 1)
        assert np.array_equal(got_h, hashes), f"batch {i}: masks"
        assert np.array_equal(got_t, toks), f"batch {i}: tokens"
    assert eng.info()["context_slots_used"] > min(50, slots // 2)
