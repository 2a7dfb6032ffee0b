"""Random-grammar device parity sweep (diagnostics; the -m gpu suite runs a
small fixed sample): N grammars from the compiler-fuzz generator, a 258-token
vocabulary over their alphabet, context depth 1/3/8, all three step forms,
tokens and final stacks against the C port.

    python scripts/gpu_fuzz.py [N] [seed]
"""
import itertools
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2506_03887_b200 as pk  # noqa: E402
from oracle import Port  # noqa: E402
import test_gpu_parity as T  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 99)
alphabet = [bytes([c]) for c in b"abc(),"]
vocab = [b"".join(p) for n in (1, 2, 3) for p in itertools.product(alphabet, repeat=n)]
done = skipped = runs = 0
while done < N:
    text = T._random_grammar(rng)
    try:
        a = pk.Automaton.compile(text)
    except pk.GmError:
        skipped += 1
        continue
    f = a.save()
    port = Port(f, vocab)
    B, steps, s = 16, 16, rng.randrange(1 << 30)
    # The port's masks along its own token streams (the reference rule).
    eng0 = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=1)
    _, ptoks, pstacks = port.decode_run(eng0.structural, B, steps, s, want_tokens=True, want_stacks=True)
    pmasks = np.zeros((B, steps, eng0.W), dtype=np.uint32)
    for b in range(B):
        c = port.initial()
        for t in range(steps):
            pmasks[b, t] = port.mask(c)
            tok = int(ptoks[b, t])
            if tok >= 0:
                port.accept_token(c, tok)
            if tok < 0 or c.status != 0:
                port.free(c)
                c = port.initial()
        port.free(c)
    for K in (1, 3, 8):
        eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
        for mode in (False, True, "split"):
            batch, masks, tokens = T.run_stream(eng, B, steps, s, fused=mode, check_logits=True)
            ok = np.array_equal(tokens, ptoks) and np.array_equal(masks, pmasks)
            for b in range(B):
                d = pstacks[b, 0]
                got = batch.get(b)
                ok = ok and got.stack == pstacks[b, 2:2 + d].tolist() and got.status == pstacks[b, 1]
            runs += 1
            if not ok:
                print("MISMATCH", K, mode, repr(text))
                sys.exit(1)
    done += 1
print(f"random-grammar parity: {done} grammars ({skipped} rejected by the compiler), {runs} device runs "
      f"(K in 1/3/8 x separate/fused/split, 16 sequences x 16 steps): masks, -inf logits, tokens and final "
      f"stacks all equal to the C port's")
