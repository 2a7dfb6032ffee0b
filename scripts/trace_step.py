"""Per-item timeline of one decode step (diagnostics; gm_batch_set_trace).

    python scripts/trace_step.py [--batch 256] [--fused] [--grammar json]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=256)
p.add_argument("--fused", action="store_true")
p.add_argument("--split", action="store_true", help="gm_decode_step_stream_split")
p.add_argument("--greedy", action="store_true", help="gm_decode_step_greedy")
p.add_argument("--grammar", default="json")
p.add_argument("--flavor", type=int, default=0)
p.add_argument("--parent", type=int, default=0)
p.add_argument("--steps", type=int, default=3)
p.add_argument("--k", type=int, default=12)
p.add_argument("--slots", type=int, default=8192)
p.add_argument("--no-logits", action="store_true", help="bitmask-only fill (no logits stream)")
p.add_argument("--prewarm", type=int, default=2000)
p.add_argument("--chain", type=int, default=0, help="also trace N back-to-back steps")
p.add_argument("--per-sm", action="store_true", help="per-SM summary of the last traced step")
p.add_argument("--queue", action="store_true", help="spin the GPU first so the host enqueues the whole step before it starts (steady-state launch overlap)")
a = p.parse_args()
flat = bench.automaton_bytes(a.grammar)
vocab = pk.synth_vocab(128255, a.flavor)
eng = pk.DeviceEngine(pk.Automaton.load(flat), vocab, device=0, context_depth=a.k, context_slots=a.slots,
                      parent_depth=a.parent)
eng.prewarm(1024, a.prewarm, seed=0xC0FFEE)
B = a.batch
batch = eng.batch(B, 1024)
dev = torch.device("cuda:0")
bm = torch.zeros((B, eng.W), dtype=torch.int32, device=dev)
counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=dev)
toks = torch.zeros(B, dtype=torch.int32, device=dev)
logits = [torch.randn((B, eng.V + 1), dtype=torch.bfloat16, device=dev) for _ in range(3)]


def step(i):
    if a.greedy:
        batch.decode_step_greedy(logits[i % 3], tokens_out=toks, bitmask=bm)
    elif a.fused:
        batch.decode_step_stream(1, bitmask=bm, logits=logits[i % 3], tokens_out=toks)
    elif a.split:
        batch.decode_step_stream_split(1, bitmask=bm, logits=None if a.no_logits else logits[i % 3],
                                       seg_counts=counts, tokens_out=toks)
    else:
        batch.fill(bm, None if a.no_logits else logits[i % 3], counts)
        batch.sample_stream_and_accept(bm, counts, 1, toks)


for i in range(40):
    step(i)
torch.cuda.synchronize()
cap = 1 << 20
tr = torch.zeros(4 * (cap + 1), dtype=torch.int64, device=dev)
names = {1: "light", 2: "heavy", 3: "tail", 4: "accept", 5: "build", 10: "h:build", 11: "h:wait", 12: "h:cdscan", 13: "h:walks",
         20: "a:step", 21: "a:lookup", 22: "a:publish", 14: "l:head", 15: "l:mixed", 16: "l:bwait"}
for s in range(a.steps):
    tr.zero_()
    batch.set_trace(tr)
    if a.queue:
        torch.cuda._sleep(400000)
    step(100 + s)
    torch.cuda.synchronize()
    batch.set_trace(None)
    t = tr.cpu().numpy().view(np.uint64)
    n = min(int(t[0]), cap)
    rec = t[4:4 * (n + 1)].reshape(n, 4).astype(np.int64)
    kind = rec[:, 0] & 0xff
    t0 = rec[:, 1].min()
    print(f"step {s}: {n} records, span {(rec[:, 2].max() - t0) / 1e3:.1f} us, contexts {eng.info()['context_slots_used']}")
    for k in sorted(set(kind.tolist())):
        r = rec[kind == k]
        st = (r[:, 1] - t0) / 1e3
        du = (r[:, 2] - r[:, 1]) / 1e3
        en = (r[:, 2] - t0) / 1e3
        pct = lambda v: " ".join(f"{x:6.1f}" for x in np.percentile(v, [0, 50, 90, 99, 100]))
        print(f"  {names[int(k)]:7s} n={len(r):6d} start[p0 p50 p90 p99 max] {pct(st)} | dur {pct(du)} | end max {en.max():6.1f}"
              f" | extra sum {int(r[:, 3].sum())}")
    if s == a.steps - 1:
        lo = np.unique(rec[:, 1] % 1024)
        print(f"  globaltimer granularity probe: {len(lo)} distinct values of t mod 1024 ns; min step "
              f"{np.diff(np.unique(rec[:, 1])).min()} ns")

if a.chain:
    # Back-to-back steps (the bench's steady state): light-item start clusters
    # mark the fills; per step, when its fill items start/end and when its
    # accepts end.
    tr.zero_()
    batch.set_trace(tr)
    torch.cuda._sleep(2000000)
    for s in range(a.chain):
        step(200 + s)
    torch.cuda.synchronize()
    batch.set_trace(None)
    t = tr.cpu().numpy().view(np.uint64)
    n = min(int(t[0]), cap)
    rec = t[4:4 * (n + 1)].reshape(n, 4).astype(np.int64)
    kind = rec[:, 0] & 0xff
    t0 = rec[:, 1].min()
    light = np.sort((rec[kind == 1, 1] - t0) / 1e3)
    cuts = [0] + [i + 1 for i in range(len(light) - 1) if light[i + 1] - light[i] > 3.0] + [len(light)]
    acc_end = np.sort((rec[kind == 4, 2] - t0) / 1e3)
    lend = (rec[kind == 1, 2] - t0) / 1e3
    lst = (rec[kind == 1, 1] - t0) / 1e3
    print(f"chain of {a.chain} steps: {len(cuts) - 1} light clusters")
    for k in range(len(cuts) - 1):
        lo, hi = light[cuts[k]], light[cuts[k + 1] - 1]
        sel = (lst >= lo) & (lst <= hi)
        ae = acc_end[(acc_end > lo)]
        print(f"  fill {k}: light start {lo:7.1f}..{hi:7.1f}  light end max {lend[sel].max():7.1f}  "
              f"accepts ended by then: {int((acc_end <= lo).sum())}")
    print("  accept end times (sorted, every 256th):", " ".join(f"{x:.1f}" for x in acc_end[::256]))
    # Per step: accept records come B per step; a fill's items start after
    # the previous step's accepts ended (its grid waits for them).
    acc = rec[kind == 4]
    acc = acc[np.argsort(acc[:, 2])]
    ends = [(acc[(k + 1) * B - 1, 2] - t0) / 1e3 for k in range(len(acc) // B)]
    prev = -1e9
    print("  step: heavy start / light start..end / accept start..end (us); gap = this fill's first item - previous accept end")
    for k, e in enumerate(ends):
        def sel(kd):
            r = rec[kind == kd]
            st = (r[:, 1] - t0) / 1e3
            m = (st > prev) & (st <= e)
            return r[m], st[m]
        hr, hs = sel(2)
        lr, ls = sel(1)
        a_r = acc[k * B:(k + 1) * B]
        first = min(hs.min() if len(hs) else 1e9, ls.min() if len(ls) else 1e9)
        print(f"  {k}: heavy {hs.min() if len(hs) else float('nan'):7.1f} light {ls.min():7.1f}..{((lr[:, 2] - t0) / 1e3).max():7.1f}"
              f"  accept {((a_r[:, 1] - t0) / 1e3).min():7.1f}..{e:7.1f}  gap {first - prev if prev > 0 else float('nan'):5.1f}")
        prev = e

if a.per_sm:
    # Per-SM view of the last traced step's light items (extra = walks |
    # smid << 32 | bytes << 40): items, bytes and last end per SM.
    light = rec[kind == 1]
    sm = (light[:, 3] >> 32) & 0xff
    by = light[:, 3] >> 40
    end = (light[:, 2] - t0) / 1e3
    rows = []
    for k in np.unique(sm):
        sel = sm == k
        rows.append((end[sel].max(), int(sel.sum()), int(by[sel].sum()), int(k)))
    rows.sort()
    arr = np.array(rows)
    print(f"per-SM light: {len(rows)} SMs; items/SM min {arr[:,1].min()} max {arr[:,1].max()}; "
          f"KB/SM min {arr[:,2].min()/1e3:.0f} max {arr[:,2].max()/1e3:.0f}; end min {arr[:,0].min():.1f} max {arr[:,0].max():.1f} us")
    for q in (0, len(rows) // 4, len(rows) // 2, 3 * len(rows) // 4, len(rows) - 1):
        e, n_i, b_, k = rows[q]
        print(f"  SM {k:3d}: end {e:6.1f} us  items {n_i:3d}  {b_/1e3:7.0f} KB  -> {b_/max(e,1e-3)/1e3:6.1f} GB/s")
