"""A small run of every device step form for compute-sanitizer:
two-call fill + sample/accept, the split step, the one-launch step, greedy,
the temperature/top-k/top-p step, prewarm, a 4-slot table (private rows),
parent builds, a captured graph, model logit layouts, overflow restarts.
Tokens and final stacks are checked against the C port where the port has
the same rule.  Usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py [part ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_03887_b200 as pk  # noqa: E402
from oracle import Port  # noqa: E402

DEV = "cuda:0"
FLAT = open(os.path.join(ROOT, "tests", "golden", "json.p3dpda"), "rb").read()
VOCAB = pk.synth_vocab(20000)


def port_tokens(eng, B, steps, seed, **kw):
    port = Port(FLAT, VOCAB)
    _, toks, stk = port.decode_run(eng.structural, B, steps, seed, want_tokens=True, want_stacks=True, **kw)
    return toks, stk


def check_stacks(batch, stk, B):
    for b in range(B):
        d = stk[b, 0]
        assert batch.get(b).stack == stk[b, 2:2 + d].tolist(), b


def stream(kind, slots=1024, parent=0, K=8, B=24, steps=10, seed=5):
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=K, context_slots=slots, parent_depth=parent)
    batch = eng.batch(B)
    if kind == "split":
        print(f"split step: {batch.split_step_launches} launch(es) at B = {B}")
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    lg = torch.randn((B, eng.V + 1), dtype=torch.bfloat16, device=DEV)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    got = []
    for _ in range(steps):
        if kind == "two_call":
            batch.fill(bm, lg, cnt)
            batch.sample_stream_and_accept(bm, cnt, seed, tk)
        elif kind == "split":
            batch.decode_step_stream_split(seed, bitmask=bm, logits=lg, seg_counts=cnt, tokens_out=tk)
        else:
            batch.decode_step_stream(seed, bitmask=bm, logits=lg, tokens_out=tk)
        batch.check()
        got.append(tk.cpu().numpy().copy())
    toks, stk = port_tokens(eng, B, steps, seed)
    assert np.array_equal(np.stack(got, 1), toks), kind
    check_stacks(batch, stk, B)


def greedy(B=16, steps=8):
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=8)
    batch = eng.batch(B)
    rows = [torch.empty((B, eng.V + 1), dtype=torch.bfloat16, device=DEV) for _ in range(3)]
    for k, t in enumerate(rows):
        pk.synth_logits(t, k, 77)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    got = []
    for s in range(steps):
        batch.decode_step_greedy(rows[s % 3], tokens_out=tk)
        batch.check()
        got.append(tk.cpu().numpy().copy())
    toks, stk = port_tokens(eng, B, steps, 0, greedy_rows=3, logit_seed=77)
    assert np.array_equal(np.stack(got, 1), toks)
    check_stacks(batch, stk, B)


def sample(B=8, steps=6):
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=8)
    batch = eng.batch(B)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    g = torch.Generator(device=DEV).manual_seed(1)
    for _ in range(steps):
        lg = torch.randn((B, eng.V + 1), generator=g, device=DEV).to(torch.bfloat16)
        batch.decode_step_sample(lg, temperature=0.8, top_k=40, top_p=0.9, seed=3, tokens_out=tk)
        batch.check()


def prewarm():
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=8, context_slots=256)
    eng.prewarm(batch=64, steps=40)
    stream_on(eng)


def stream_on(eng, B=16, steps=6, seed=9):
    batch = eng.batch(B)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(steps):
        batch.decode_step_stream_split(seed, tokens_out=tk)
        batch.check()


def graph(B=16, G=6, seed=31):
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=8)
    batch = eng.batch(B)
    tks = [torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(G)]
    gr = batch.capture_steps(G, seed=seed, tokens_out=tks)
    got = []
    for _ in range(2):
        gr.launch()
        batch.check()
        got.append(torch.stack(tks, 1).cpu().numpy())
    toks, stk = port_tokens(eng, B, 2 * G, seed)
    assert np.array_equal(np.concatenate(got, 1), toks)


def layout(B=8, steps=6):
    V = len(VOCAB)
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=8, num_columns=V + 256, eos_column=V + 1)
    batch = eng.batch(B)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(steps):
        lg = torch.randn((B, V + 256), device=DEV).to(torch.bfloat16)
        batch.decode_step_stream_split(4, logits=lg, tokens_out=tk)
        batch.check()
        batch.decode_step_greedy(lg, tokens_out=tk)
        batch.check()


def layout_eos_inside(B=16, steps=8):
    """Llama-2-like layout: the EOS column (id 2) among the regular ids,
    K = 2 so EOS is mostly context-dependent (its segment goes heavy)."""
    vocab = [b"", b"", b""] + VOCAB[3:]
    V = len(vocab)
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), vocab, context_depth=2, num_columns=V, eos_column=2,
                          disabled=[0, 1, 2])
    batch = eng.batch(B)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(steps):
        lg = torch.randn((B, V), device=DEV).to(torch.bfloat16)
        batch.decode_step_stream_split(4, logits=lg, tokens_out=tk)
        batch.check()


def two_streams(B=16, steps=8):
    """Two batches of one engine stepping concurrently on two streams."""
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=6, context_slots=64, parent_depth=3)
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    bs = [eng.batch(B), eng.batch(B)]
    tks = [torch.zeros(B, dtype=torch.int32, device=DEV) for _ in range(2)]
    for _ in range(steps):
        for i in range(2):
            with torch.cuda.stream(ss[i]):
                bs[i].decode_step_stream_split(11 + i, tokens_out=tks[i], stream=ss[i].cuda_stream)
    torch.cuda.synchronize()
    for i in range(2):
        bs[i].check(stream=ss[i].cuda_stream)


def overflow(B=8, steps=12):
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=4)
    batch = eng.batch(B, stack_capacity=8)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(steps):
        batch.decode_step_stream_split(2, tokens_out=tk)
        batch.check()


def refill(B=16, K=2):
    """Fills without an accept between (past the 6-fill tag period), a sample
    without accept, then split steps with heavy segments (K = 2 leaves many
    context-dependent tokens): masks equal to the port's on the same stacks."""
    eng = pk.DeviceEngine(pk.Automaton.load(FLAT), VOCAB, context_depth=K, context_slots=1024)
    port = Port(FLAT, VOCAB)
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    tk = torch.zeros(B, dtype=torch.int32, device=DEV)
    for _ in range(5):
        batch.decode_step_stream_split(3, bitmask=bm, seg_counts=cnt, tokens_out=tk)
    want = []
    for b in range(B):
        c = batch.get(b)
        cfg = port.config(c.status, c.stack)
        want.append(port.mask(cfg))
        port.free(cfg)
    want = np.stack(want)
    for _ in range(8):
        batch.fill(bm, None, cnt)
        batch.check()
        assert np.array_equal(bm.cpu().numpy().view(np.uint32), want)
    batch.sample_stream(bm, cnt, 3, tk)
    for _ in range(4):
        batch.decode_step_stream_split(3, bitmask=bm, seg_counts=cnt, tokens_out=tk)
        batch.check()


def split_two_grid(B=64, steps=6):
    """The split step as fill + accept kernel (PRE3_SPLIT_TWO_KERNELS)."""
    os.environ["PRE3_SPLIT_TWO_KERNELS"] = "1"
    try:
        stream("split", B=B, steps=steps)
    finally:
        del os.environ["PRE3_SPLIT_TWO_KERNELS"]


PARTS = {
    "two_call": lambda: stream("two_call"),
    "split": lambda: stream("split"),
    "split_two_grid": split_two_grid,
    "one_launch": lambda: stream("one_launch"),
    "tiny_table": lambda: stream("split", slots=4),
    "parents": lambda: stream("split", parent=3, K=12),
    "greedy": greedy,
    "sample": sample,
    "prewarm": prewarm,
    "graph": graph,
    "layout": layout,
    "overflow": overflow,
    "refill": refill,
    "layout_eos_inside": layout_eos_inside,
    "two_streams": two_streams,
}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(PARTS):
        PARTS[name]()
        torch.cuda.synchronize()
        print("ok", name, flush=True)
