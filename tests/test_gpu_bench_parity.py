"""GPU parity at the exact settings bench.py measures.

For every BASELINE config the engine is built exactly as bench.py builds it
(grammar, context depth K, table size, parent depth R, the prewarm of the
context cache) and the benchmarked step form runs (the split step for
configs 2-4, the greedy step for config 5).  Every step of >= 64 sequences
x >= 32 steps is compared with the C port (oracle/gmask_port.c, pinned to the
reference): the full bitmask of every sequence (polynomial hash of all W
words, oracle.mask_hashes == gp_mask_hash), the sampled token, the -inf
positions of the masked bf16 logits, and the final stacks and statuses.
"""
import os
import sys

import numpy as np
import pytest

import oracle
import paper_2506_03887_b200 as pk
from oracle import Port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

DEV = "cuda:0"


def bench_engine(config):
    a = bench.parse(["--config", str(config)])
    flat = bench.automaton_bytes(a.grammar)
    vocab = pk.synth_vocab(a.vocab, a.flavor)
    eng = pk.DeviceEngine(pk.Automaton.load(flat), vocab, context_depth=a.context_depth,
                          context_slots=a.context_slots, parent_depth=a.parent_depth)
    eng.prewarm(a.prewarm_batch, a.prewarm_steps, seed=0xC0FFEE, stack_capacity=a.stack_cap)  # bench.py's rank-0 prewarm
    return a, flat, vocab, eng


def device_loop(a, eng, B, steps, seed, check_logits=True):
    """The benchmarked step form, every step's bitmask hashed on the host."""
    batch = eng.batch(B, a.stack_cap)
    V1 = eng.V + 1
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=DEV)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    greedy = a.mode == "greedy"
    R = 3
    if greedy:
        logits = [torch.empty((B, V1), dtype=torch.bfloat16, device=DEV) for _ in range(R)]
        for k, t in enumerate(logits):
            pk.synth_logits(t, k, bench.LOGIT_SEED)
    else:
        lg = torch.empty((B, V1), dtype=torch.bfloat16, device=DEV)
    hashes, tokens = [], []
    for s in range(steps):
        if greedy:
            batch.decode_step_greedy(logits[s % R], tokens_out=toks, bitmask=bm)
        else:
            lg.normal_()
            before = lg.clone() if check_logits else None
            batch.decode_step_stream_split(seed, bitmask=bm, logits=lg, seg_counts=counts, tokens_out=toks)
        batch.check()
        m = bm.cpu().numpy().view(np.uint32)
        hashes.append(oracle.mask_hashes(m))
        tokens.append(toks.cpu().numpy().copy())
        if not greedy and check_logits:
            bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, :V1].astype(bool)
            after = lg.float().cpu().numpy()
            b0 = before.float().cpu().numpy()
            assert np.array_equal(np.isneginf(after), ~bits | np.isneginf(b0)), s
            assert np.array_equal(after[bits], b0[bits]), s
    return batch, np.stack(hashes, 1), np.stack(tokens, 1)


def port_loop(a, flat, vocab, structural, B, steps, seed):
    port = Port(flat, vocab)
    kw = dict(greedy_rows=3, logit_seed=bench.LOGIT_SEED) if a.mode == "greedy" else {}
    _, ptoks, pstacks, phash = port.decode_run(structural, B, steps, seed, stack_cap=a.stack_cap, want_tokens=True,
                                               want_stacks=True, want_mask_hashes=True, **kw)
    return ptoks, pstacks, phash


@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_bench_settings_per_step_masks_match_port(config):
    """Configs 2-5 at bench.py's engine settings (config 2: K=20, 65,536
    slots, 10k-step prewarm; 3: K=16; 4: K=20, R=6, 262,144 slots, 30k-step
    prewarm; 5: greedy, K=12) and bench.py's rank-0 streams: 64 sequences x
    32 steps, every mask, token, -inf position and the final stacks equal the
    port's."""
    a, flat, vocab, eng = bench_engine(config)
    B, steps = 64, 32
    seed = bench.rank_seed(a.seed, 0)
    batch, hashes, tokens = device_loop(a, eng, B, steps, seed)
    ptoks, pstacks, phash = port_loop(a, flat, vocab, eng.structural, B, steps, seed)
    assert np.array_equal(tokens, ptoks)
    bad = np.argwhere(hashes != phash)
    assert bad.size == 0, f"mask mismatches at (seq, step) {bad[:8].tolist()}"
    for b in range(B):
        d = pstacks[b, 0]
        got = batch.get(b)
        assert got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1], b
    info = eng.info()
    assert info["context_slots_used"] > 0


def test_bench_config3_full_batch_matches_port():
    """Config 3 at its full bench batch (1,024 sequences) for 8 steps: every
    sequence's mask and token each step equal the port's (not a sample)."""
    a, flat, vocab, eng = bench_engine(3)
    B, steps = 1024, 8
    seed = bench.rank_seed(a.seed, 0)
    batch, hashes, tokens = device_loop(a, eng, B, steps, seed, check_logits=False)
    ptoks, pstacks, phash = port_loop(a, flat, vocab, eng.structural, B, steps, seed)
    assert np.array_equal(tokens, ptoks)
    assert np.array_equal(hashes, phash)
