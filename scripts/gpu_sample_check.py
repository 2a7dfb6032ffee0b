"""Temperature / top-k / top-p decode step vs the C port's rule at 128k
tokens (diagnostics; the -m gpu suite runs a smaller sample): masks, tokens
and stacks every step, dense and quantized (tied) logits.

    python scripts/gpu_sample_check.py [batch] [steps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402
from oracle import Port  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
vocab = pk.synth_vocab(128255)
f = bench.automaton_bytes("json")
port = Port(f, vocab)
n = 0
for T, k, p, ties in ((1.0, 0, 1.0, False), (1.0, 0, 1.0, True), (0.7, 0, 0.95, False), (1.3, 40, 1.0, True),
                      (0.8, 50, 0.9, False), (2.0, 0, 0.5, True)):
    eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=16)
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device="cuda")
    toks = torch.zeros(B, dtype=torch.int32, device="cuda")
    cfgs = [port.initial() for _ in range(B)]
    g = torch.Generator(device="cuda").manual_seed(11)
    seed = 1234
    for s in range(steps):
        lg = torch.randn((B, eng.V + 1), dtype=torch.float32, device="cuda", generator=g)
        if ties:
            lg = torch.round(lg * 2) / 2
        lg = lg.to(torch.bfloat16)
        batch.decode_step_sample(lg, temperature=T, top_k=k, top_p=p, seed=seed, tokens_out=toks, bitmask=bm)
        batch.check()
        got = bm.cpu().numpy().view(np.uint32)
        rows = lg.view(torch.int16).cpu().numpy().view(np.uint16)
        tk = toks.cpu().numpy()
        for b in range(B):
            want = port.mask(cfgs[b])
            assert np.array_equal(got[b], want), (T, k, p, ties, b, s)
            tok = port.sample_pick(want, rows[b], T, k, p, Port.stream_draw(seed, b, s))
            assert tok == tk[b], (T, k, p, ties, b, s, tok, tk[b])
            if tok >= 0:
                port.accept_token(cfgs[b], tok)
            if tok < 0 or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            assert batch.get(b).stack == port.get(cfgs[b])[2], (T, k, p, ties, b, s)
            n += 1
print(f"sampler parity at 128k: {n} sequence-steps over 6 (T, top-k, top-p, ties) settings, batch {B}: masks, "
      f"tokens and stacks equal to the C port's")
