"""Step rate of gm_decode_step_sample (fill + temperature/top-k/top-p sampler
+ accept, one host call) on JSON at 128k tokens (diagnostics).

    python scripts/sample_rate.py [batch ...]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402

vocab = pk.synth_vocab(128255)
eng = pk.DeviceEngine(pk.Automaton.load(bench.automaton_bytes("json")), vocab, context_depth=20,
                      context_slots=65536)
eng.prewarm(1024, 10000, seed=0xC0FFEE)
for B in [int(x) for x in sys.argv[1:]] or [256, 1024]:
    batch = eng.batch(B)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device="cuda")
    toks = torch.zeros(B, dtype=torch.int32, device="cuda")
    R = max(2, -(-3 * 126 * 2**20 // (B * (eng.V + 1) * 2)))
    lg = [torch.randn((B, eng.V + 1), dtype=torch.bfloat16, device="cuda") for _ in range(R)]
    for T, k, p in ((1.0, 0, 1.0), (0.8, 50, 0.9)):
        for i in range(20):
            batch.decode_step_sample(lg[i % R], temperature=T, top_k=k, top_p=p, seed=1, tokens_out=toks, bitmask=bm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 200
        e0.record()
        for i in range(K):
            batch.decode_step_sample(lg[i % R], temperature=T, top_k=k, top_p=p, seed=1, tokens_out=toks, bitmask=bm)
        e1.record()
        torch.cuda.synchronize()
        batch.check()
        ms = e0.elapsed_time(e1) / K
        print(f"B={B} T={T} top_k={k} top_p={p}: {ms * 1e3:.1f} us/step, {B / ms * 1e3 / 1e6:.2f} M seq-steps/s")
