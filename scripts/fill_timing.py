"""Where a config-2-shaped step's time goes (diagnostics): the same engine and
streams timed several ways — events between steps, the fill bracketed by
events (split step and two-call step), the fill alone re-run on a frozen
batch state, and a captured graph of steps.

    python scripts/fill_timing.py [--batch 256] [--grammar json] [--k 20] [--slots 65536]
"""
import argparse
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=256)
p.add_argument("--grammar", default="json")
p.add_argument("--flavor", type=int, default=0)
p.add_argument("--k", type=int, default=20)
p.add_argument("--slots", type=int, default=65536)
p.add_argument("--parent", type=int, default=0)
p.add_argument("--prewarm", type=int, default=10000)
p.add_argument("--n", type=int, default=60)
p.add_argument("--graph-first", type=int, default=0, help="replay a graph of N split steps before the measurements")
a = p.parse_args()

flat = bench.automaton_bytes(a.grammar)
vocab = pk.synth_vocab(128255, a.flavor)
eng = pk.DeviceEngine(pk.Automaton.load(flat), vocab, device=0, context_depth=a.k, context_slots=a.slots,
                      parent_depth=a.parent)
eng.prewarm(1024, a.prewarm, seed=0xC0FFEE)
B = a.batch
dev = torch.device("cuda:0")
batch = eng.batch(B, 1024)
W, V1 = eng.W, eng.V + 1
R = bench.logits_buffers(B, V1)
logits = [torch.randn((B, V1), dtype=torch.bfloat16, device=dev) for _ in range(R)]
bm = torch.zeros((B, W), dtype=torch.int32, device=dev)
counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=dev)
toks = torch.zeros(B, dtype=torch.int32, device=dev)
g = [0]


def split():
    batch.decode_step_stream_split(1, bitmask=bm, logits=logits[g[0] % R], seg_counts=counts, tokens_out=toks)
    g[0] += 1


def two_call():
    batch.fill(bm, logits[g[0] % R], counts)
    batch.sample_stream_and_accept(bm, counts, 1, toks)
    g[0] += 1


def stats(xs):
    xs = sorted(xs)
    return f"mean {statistics.mean(xs):7.2f} p50 {xs[len(xs)//2]:7.2f} min {xs[0]:7.2f} max {xs[-1]:7.2f} us"


def ev():
    return torch.cuda.Event(enable_timing=True)


for _ in range(30):
    split()
torch.cuda.synchronize()
n = a.n


def between(fn, label):
    es = [ev() for _ in range(n + 1)]
    es[0].record()
    for i in range(n):
        fn()
        es[i + 1].record()
    torch.cuda.synchronize()
    print(f"{label:44s}", stats([1e3 * es[i].elapsed_time(es[i + 1]) for i in range(n)]))


def bracket(fn, label):
    pairs = [(ev(), ev()) for _ in range(n)]
    for x, y in pairs:
        x.record(), y.record()
    torch.cuda.synchronize()
    for i in range(n):
        batch.time_next_fill(*pairs[i])
        fn()
    torch.cuda.synchronize()
    print(f"{label:44s}", stats([1e3 * x.elapsed_time(y) for x, y in pairs]))


def loop(fn, label, k=120):
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:44s} {1e3 * e0.elapsed_time(e1) / k:7.2f} us/step (host-enqueued)")


if a.graph_first:
    gf = batch.capture_steps(a.graph_first, seed=1, logits=[logits[i % R] for i in range(a.graph_first)], bitmask=bm,
                             seg_counts=[counts] * a.graph_first, tokens_out=[toks] * a.graph_first)
    gf.launch()
    torch.cuda.synchronize()
    bracket(split, "split: fill bracketed (right after the graph)")
batch.set_stats(True)
between(split, "split: events between steps")
print("  stats", batch.fill_stats(), eng.cache_stats())
batch.set_stats(False)
bracket(split, "split: fill bracketed")
between(two_call, "two-call: events between steps")
bracket(two_call, "two-call: fill bracketed")
loop(split, "split: back to back")
loop(two_call, "two-call: back to back")
# The fill alone, re-run on a frozen state (no accept: same slots, same items).
torch.cuda.synchronize()
es = [ev() for _ in range(n + 1)]
es[0].record()
for i in range(n):
    batch.fill(bm, logits[i % R], counts)
    es[i + 1].record()
torch.cuda.synchronize()
print(f"{'fill only, frozen state, events between':44s}", stats([1e3 * es[i].elapsed_time(es[i + 1]) for i in range(n)]))
es[0].record()
for i in range(n):
    batch.fill(bm, None, counts)
    es[i + 1].record()
torch.cuda.synchronize()
print(f"{'fill only, no logits':44s}", stats([1e3 * es[i].elapsed_time(es[i + 1]) for i in range(n)]))
# A plain -inf write of the same rows (the store-stream floor at this size).
es[0].record()
for i in range(n):
    logits[i % R].fill_(float("-inf"))
    es[i + 1].record()
torch.cuda.synchronize()
print(f"{'torch fill_ of the logits rows':44s}", stats([1e3 * es[i].elapsed_time(es[i + 1]) for i in range(n)]))
graph = batch.capture_steps(120, seed=1, logits=[logits[i % R] for i in range(120)], bitmask=bm,
                            seg_counts=[counts] * 120, tokens_out=[toks] * 120)
torch.cuda.synchronize()
e0, e1 = ev(), ev()
e0.record()
graph.launch()
e1.record()
torch.cuda.synchronize()
print(f"{'graph of 120 split steps':44s} {1e3 * e0.elapsed_time(e1) / 120:7.2f} us/step")
batch.check()
