"""Diagnose test_gpu_cache.test_long_pushing_tokens_match_the_port: first
(sequence, step) whose device mask differs from the port's, and which tokens."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_03887_b200 as pk  # noqa: E402
from oracle import Port  # noqa: E402
from test_gpu_cache import deep_vocab, flat  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
voc = deep_vocab(pk.synth_vocab(30000)[:8000], N)
f = flat("json")
eng = pk.DeviceEngine(pk.Automaton.load(f), voc, context_depth=K, context_slots=1024)
port = Port(f, voc)
B, steps, seed = 32, 20, 5
batch = eng.batch(B)
bm = torch.zeros((B, eng.W), dtype=torch.int32, device="cuda:0")
cnt = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device="cuda:0")
tk = torch.zeros(B, dtype=torch.int32, device="cuda:0")
cfgs = [port.initial() for _ in range(B)]
long_ids = {i for i, t in enumerate(voc) if len(t) > 8}
for s in range(steps):
    batch.decode_step_stream_split(seed, bitmask=bm, seg_counts=cnt, tokens_out=tk)
    try:
        batch.check()
    except pk.GmError as e:
        print("check error at step", s, e)
    got = bm.cpu().numpy().view(np.uint32)
    toks = tk.cpu().numpy()
    for b in range(B):
        want = port.mask(cfgs[b])
        if not np.array_equal(got[b], want):
            gb = np.unpackbits(got[b].view(np.uint8), bitorder="little")
            wb = np.unpackbits(want.view(np.uint8), bitorder="little")
            d = np.nonzero(gb != wb)[0]
            depth = len(port.get(cfgs[b])[2])
            print(f"step {s} seq {b} depth {depth}: {len(d)} bits differ; first {d[:10].tolist()} "
                  f"dev {gb[d[:10]].tolist()} port {wb[d[:10]].tolist()} long {[int(x) in long_ids for x in d[:10]]} "
                  f"tokens {[voc[int(x)][:12] for x in d[:5] if x < len(voc)]}")
            sys.exit(1)
        t = port.stream_pick(want, eng.structural, Port.stream_draw(seed, b, s))
        if t != toks[b]:
            print(f"step {s} seq {b}: token {toks[b]} vs port {t}")
            sys.exit(1)
        if t >= 0:
            port.accept_token(cfgs[b], t)
        if t < 0 or cfgs[b].status != 0:
            port.free(cfgs[b])
            cfgs[b] = port.initial()
print("all equal")
