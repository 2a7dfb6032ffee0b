"""Wider random-grammar device parity sweep (diagnostics): grammars with up
to 8 nonterminals and multi-byte literals over a larger alphabet, random
vocabularies (all single characters + random 2-5 byte strings), small stack
capacities (overflow paths), context depth 1/4/12, the three stream step
forms and the greedy step — masks, -inf logits, tokens and final stacks
against the C port.

    python scripts/gpu_fuzz2.py [N] [seed]
"""
import os
import random
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2506_03887_b200 as pk  # noqa: E402
from oracle import Port  # noqa: E402
import test_gpu_parity as T  # noqa: E402

ALPHA = "ab{}[],: x1"


def grammar(rng):
    names = ["S", "A", "B", "C", "D", "E", "F", "G"][: rng.randint(2, 8)]
    lines = []
    for n in names:
        alts = []
        for _ in range(rng.randint(1, 4)):
            syms = []
            for _ in range(rng.randint(0, 5)):
                if rng.random() < 0.4:
                    syms.append(rng.choice(names))
                else:
                    lit = "".join(rng.choice(ALPHA) for _ in range(rng.randint(1, 3)))
                    syms.append('"' + lit + '"')
            alts.append(" ".join(syms))
        lines.append(n + " -> " + " | ".join(alts))
    return "\n".join(lines) + "\n"


VOCAB_RANGE = (60, 400)  # tokens per random vocabulary (gpu_fuzz2.py N seed [min max])


def vocab_for(rng):
    v = {c.encode() for c in ALPHA}
    want = rng.randint(*VOCAB_RANGE)
    longest = 5 if VOCAB_RANGE[1] <= 400 else 8
    while len(v) < want:
        v.add("".join(rng.choice(ALPHA) for _ in range(rng.randint(2, longest))).encode())
    return sorted(v)


def port_masks(port, vocab, ptoks, B, steps, W, cap):
    """The port's mask at every step of its own streams (gp_decode_run's loop:
    Step per byte, restart on a dead end, a finished sequence or depth > cap)."""
    out = np.zeros((B, steps, W), dtype=np.uint32)
    V = len(vocab)
    for b in range(B):
        c = port.initial()
        for t in range(steps):
            out[b, t] = port.mask(c)
            tok = int(ptoks[b, t])
            overflow = False
            if tok == V:
                port.step(c, 256)
            elif tok >= 0:
                for byte in vocab[tok]:
                    if not port.step(c, byte):
                        break
                    if len(port.get(c)[2]) > cap:
                        overflow = True
                        break
            if tok < 0 or overflow or c.status != 0:
                port.free(c)
                c = port.initial()
        port.free(c)
    return out


def greedy_run(eng, port, vocab_of, B, steps, cap, gseed):
    """Device gm_decode_step_greedy vs the port's argmax rule, step by step."""
    batch = eng.batch(B, cap)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device="cuda")
    toks = torch.zeros(B, dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(gseed)
    cfgs = [port.initial() for _ in range(B)]
    for s in range(steps):
        lg = torch.randn((B, eng.V + 1), dtype=torch.float32, device="cuda", generator=g)
        lg = (torch.round(lg * 2) / 2).to(torch.bfloat16)  # ties
        batch.decode_step_greedy(lg, toks, bm)
        batch.check()
        got = bm.cpu().numpy().view(np.uint32)
        rows = lg.view(torch.int16).cpu().numpy().view(np.uint16)
        tk = toks.cpu().numpy()
        for b in range(B):
            want = port.mask(cfgs[b])
            if not np.array_equal(got[b], want):
                return False
            tok = port.greedy_pick(want, rows[b])
            if tok != tk[b]:
                return False
            overflow = False
            if tok == eng.V:
                port.step(cfgs[b], 256)
            elif tok >= 0:  # Step per byte with the capacity check of gp_decode_run
                for byte in vocab_of[tok]:
                    if not port.step(cfgs[b], byte):
                        break
                    if len(port.get(cfgs[b])[2]) > cap:
                        overflow = True
                        break
            if tok < 0 or overflow or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            if batch.get(b).stack != port.get(cfgs[b])[2]:
                return False
    return True


def sample_run(eng, port, vocab_of, B, steps, cap, gseed, T_, k_, p_):
    """Device gm_decode_step_sample (temperature/top-k/top-p) vs the port's
    rule, step by step, plus AllowedTerminals of every configuration."""
    batch = eng.batch(B, cap)
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device="cuda")
    toks = torch.zeros(B, dtype=torch.int32, device="cuda")
    at = torch.zeros((B, 9), dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(gseed)
    cfgs = [port.initial() for _ in range(B)]
    for s in range(steps):
        batch.allowed_terminals(at)
        atw = at.cpu().numpy().view(np.uint32)
        for b in range(B):
            byteset, eos = port.allowed(cfgs[b])
            got = sum(int(atw[b, i]) << (32 * i) for i in range(8))
            if got != byteset or bool(atw[b, 8] & 1) != eos:
                return False
        lg = torch.randn((B, eng.V + 1), dtype=torch.float32, device="cuda", generator=g)
        lg = (torch.round(lg * 2) / 2).to(torch.bfloat16)
        batch.decode_step_sample(lg, temperature=T_, top_k=k_, top_p=p_, seed=gseed, tokens_out=toks, bitmask=bm)
        batch.check()
        got = bm.cpu().numpy().view(np.uint32)
        rows = lg.view(torch.int16).cpu().numpy().view(np.uint16)
        tk = toks.cpu().numpy()
        for b in range(B):
            want = port.mask(cfgs[b])
            if not np.array_equal(got[b], want):
                return False
            tok = port.sample_pick(want, rows[b], T_, k_, p_, Port.stream_draw(gseed, b, s))
            if tok != tk[b]:
                return False
            overflow = False
            if tok == eng.V:
                port.step(cfgs[b], 256)
            elif tok >= 0:
                for byte in vocab_of[tok]:
                    if not port.step(cfgs[b], byte):
                        break
                    if len(port.get(cfgs[b])[2]) > cap:
                        overflow = True
                        break
            if tok < 0 or overflow or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            if batch.get(b).stack != port.get(cfgs[b])[2]:
                return False
    return True


def run(N, seed):
    """Returns (grammars, rejected, runs); exits on the first mismatch."""
    rng = random.Random(seed)
    done = skipped = runs = 0
    while done < N:
        text = grammar(rng)
        try:
            a = pk.Automaton.compile(text)
        except pk.GmError:
            skipped += 1
            continue
        f = a.save()
        vocab = vocab_for(rng)
        port = Port(f, vocab)
        B, steps, s = 24, 20, rng.randrange(1 << 30)
        cap = rng.choice([6, 12, 1024])
        eng0 = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=1)
        _, ptoks, pstacks = port.decode_run(eng0.structural, B, steps, s, stack_cap=cap, want_tokens=True,
                                            want_stacks=True)
        pm = port_masks(port, vocab, ptoks, B, steps, eng0.W, cap)
        for K in (1, 4, 12):
            eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=K)
            for mode in (False, True, "split"):
                batch, masks, tokens = T.run_stream(eng, B, steps, s, cap=cap, fused=mode, check_logits=True)
                ok = np.array_equal(tokens, ptoks) and np.array_equal(masks, pm)
                for b in range(B):
                    d = pstacks[b, 0]
                    got = batch.get(b)
                    ok = ok and got.stack == pstacks[b, 2:2 + d].tolist()
                runs += 1
                if not ok:
                    print("MISMATCH stream", K, mode, cap, repr(text), len(vocab))
                    dt = np.argwhere(tokens != ptoks)
                    dm = np.argwhere((masks != pm).any(axis=2))
                    print("  first token diff", dt[:1].tolist(), "first mask diff", dm[:1].tolist())
                    if len(dt):
                        bb, ss = [int(x) for x in dt[0]]
                        print("  dev toks", tokens[bb, :ss + 1].tolist(), "port toks", ptoks[bb, :ss + 1].tolist())
                        print("  tokens:", [vocab[t] if 0 <= t < len(vocab) else t for t in ptoks[bb, :ss + 1].tolist()])
                    for b in range(B):
                        d = pstacks[b, 0]
                        if batch.get(b).stack != pstacks[b, 2:2 + d].tolist():
                            print("  stack diff seq", b, batch.get(b).stack, batch.get(b).status, pstacks[b, 2:2 + d].tolist(), pstacks[b, 1])
                            break
                    raise AssertionError("device and C port differ (details above)")
            if K == 4:
                runs += 1
                if not greedy_run(eng, port, vocab, B, 12, cap, s & 0xffff):
                    print("MISMATCH greedy", K, cap, repr(text), len(vocab))
                    raise AssertionError("device and C port differ (details above)")
                runs += 1
                T_, k_, p_ = rng.choice([0.7, 1.0, 1.6]), rng.choice([0, 1, 5]), rng.choice([1.0, 0.9, 0.5])
                if not sample_run(eng, port, vocab, B, 10, cap, s & 0xffff, T_, k_, p_):
                    print("MISMATCH sample/allowed", K, cap, T_, k_, p_, repr(text), len(vocab))
                    raise AssertionError("device and C port differ (details above)")
        # Overlap race check at a multi-wave batch: the split step equals the
        # serial two-call loop token for token (device vs device).
        if done % 10 == 0:
            eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=rng.choice([1, 4, 12]))
            _, _, t_split = T.run_stream(eng, 1024, 40, s, cap=cap, fused="split")
            _, _, t_two = T.run_stream(eng, 1024, 40, s, cap=cap, fused=False)
            runs += 2
            if not np.array_equal(t_split, t_two):
                print("MISMATCH split vs two-call at 1024", cap, repr(text), len(vocab))
                raise AssertionError("device and C port differ (details above)")
        # Context-cache pressure: 4 slots (private rows) and parent depths.
        for slots, R in ((4, 0), (64, 1), (1 << 12, 3), (1 << 12, -1)):
            eng = pk.DeviceEngine(pk.Automaton.load(f), vocab, context_depth=6, context_slots=slots, parent_depth=R)
            batch, masks, tokens = T.run_stream(eng, B, steps, s, cap=cap, fused="split")
            runs += 1
            if not (np.array_equal(tokens, ptoks) and np.array_equal(masks, pm)):
                print("MISMATCH cache", slots, R, cap, repr(text), len(vocab))
                raise AssertionError("device and C port differ (details above)")
        done += 1
    return done, skipped, runs


def report(done, skipped, runs):
    print(f"wide random-grammar parity: {done} grammars ({skipped} rejected by the compiler), {runs} device runs "
          f"(K 1/4/12 x separate/fused/split + greedy + temperature/top-k/top-p with AllowedTerminals, context tables "
          f"of 4/64/4096 slots and parent depths -1/1/3, 1024-sequence split-vs-two-call runs every 10th grammar, "
          f"random {VOCAB_RANGE[0]}-{VOCAB_RANGE[1]}-token vocabularies, stack capacity 6/12/1024): "
          f"masks, -inf logits, tokens, terminal sets and stacks all equal to the C port's")


if __name__ == "__main__":
    if len(sys.argv) > 4:
        VOCAB_RANGE = (int(sys.argv[3]), int(sys.argv[4]))
    report(*run(int(sys.argv[1]) if len(sys.argv) > 1 else 100, int(sys.argv[2]) if len(sys.argv) > 2 else 7))
