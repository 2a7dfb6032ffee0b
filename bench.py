#!/usr/bin/env python
"""bench.py — masked decode steps/sec of the constrained-decoding hot path.

Default workload (the largest single-GPU BASELINE.json config, "config 3"):
JSON-schema-derived LR(1) grammar, Llama-3-sized vocabulary (128,255 tokens +
EOS = 128,256 mask bits), batch 1024 sequences per GPU.  One step = mask fill
+ in-place bf16 -inf logit masking + synthetic-stream sampling + accept_token
with restart, for every sequence of the batch (gm_decode_step_stream_split:
the fill and the overlapping sample/accept kernel).

Other BASELINE configs:
    --config 2   JSON grammar, batch 256/GPU
    --config 4   SQL-subset grammar, 4096 sequences in total split over the
                 GPUs (strong scaling)
    --config 5   JSON, 512/GPU, greedy decode: mask + argmax over the allowed
                 bf16 logits + accept (gm_decode_step_greedy)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Under torchrun each rank drives one GPU with its own sequences (no collective
on the hot path — NCCL only reduces the final timings and counters).  Prints
ONE JSON line on rank 0.  See DESIGN.md §7 for every field.

Both arms print `check`: an FNV-1a digest of the token ids sequences 0..31
chose in the timed steps and the sum of their mask popcounts (EOS excluded) —
the GPU arm's timed output must equal the CPU reference's on the same streams.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "masked decode steps/sec (batch×steps) and per-step mask latency at 128k vocab"
UNIT = "seq-steps/s"
L2_BYTES = 126 * 1024 * 1024
DIGEST_SEQS = 32
LOGIT_SEED = 0x5EED10C175  # config 5's synthetic logits (gp_synth_logit)

# BASELINE.json configs (index 1.. = config 2..5).
CONFIGS = {
    2: dict(grammar="json", flavor=0, batch=256, mode="stream", scaling="weak", K=20, slots=65536,
            desc="config2: JSON LR(1) grammar, 128256-bit vocab (synthetic 128k tokens), batch {b}/GPU, "
                 "fused mask-fill + in-place bf16 -inf logit masking + stream sample + accept_token"),
    3: dict(grammar="schema", flavor=0, batch=1024, mode="stream", scaling="weak", K=16, slots=16384,
            desc="config3: JSON-schema-derived LR(1) grammar (nested objects/arrays), 128256-bit vocab, "
                 "batch {b}/GPU, fused mask-fill + bf16 -inf logit masking + stream sample + accept_token"),
    4: dict(grammar="sql", flavor=1, batch=4096, mode="stream", scaling="strong", K=20, slots=262144, R=6,
            prewarm=30000,
            desc="config4: SQL-subset LR(1) grammar, 128256-bit SQL-flavoured vocab, 4096 sequences in total "
                 "({b}/GPU), fused mask-fill + bf16 -inf logit masking + stream sample + accept_token"),
    5: dict(grammar="json", flavor=0, batch=512, mode="greedy", scaling="weak", K=12, slots=16384,
            desc="config5: simulated decode loop, JSON grammar, 128256-bit vocab, batch {b}/GPU: synthetic bf16 "
                 "logits, mask + greedy argmax over allowed ids + DPDA advance"),
}
DEFAULT_CONFIG = 3


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=30)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    p.add_argument("--batch", type=int, default=None, help="sequences per GPU (default: the config's)")
    p.add_argument("--vocab", type=int, default=128255, help="regular tokens (EOS adds one bit)")
    p.add_argument("--grammar", default=None, help="override the config's grammar")
    p.add_argument("--context-depth", type=int, default=None,
                   help="K: stack entries keying the context cache (default: the config's; SQL conditions pop up "
                        "to 34 entries, so config 4 keys deeper)")
    p.add_argument("--context-slots", type=int, default=None, help="context-cache hash table slots (power of two)")
    p.add_argument("--parent-depth", type=int, default=None,
                   help="R: new contexts are built from the context keyed R deep (default: the config's, else the "
                        "engine default min(4, K-1); -1: full builds)")
    p.add_argument("--prewarm-steps", type=int, default=None,
                   help="context-cache preprocessing: synthetic decode steps (other seed) before timing (default: "
                        "the config's — 10,000; 30,000 for SQL, whose context space is ~6x JSON's)")
    p.add_argument("--prewarm-batch", type=int, default=1024)
    p.add_argument("--stack-cap", type=int, default=1024)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--one-launch", action="store_true", help="stream mode: the one-launch fused step")
    p.add_argument("--no-graph", action="store_true",
                   help="enqueue every step from Python instead of replaying a captured CUDA graph")
    p.add_argument("--fill-samples", type=int, default=120,
                   help="steps of the roofline sub-loop (the fill kernel bracketed by events every step)")
    p.add_argument("--latency-samples", type=int, default=64,
                   help="steps of the latency sub-loop (events between steps: per-step latency p50/p99)")
    p.add_argument("--cold-steps", type=int, default=100, help="steps timed from an empty context table")
    p.add_argument("--no-snapshot", action="store_true",
                   help="time on the prewarmed engine itself (default: save its context table and run on a fresh "
                        "engine loaded from the snapshot)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    a = p.parse_args(argv)
    cfg = CONFIGS[a.config]
    a.mode = cfg["mode"]
    a.flavor = cfg["flavor"]
    a.scaling = cfg["scaling"]
    if a.grammar is None:
        a.grammar = cfg["grammar"]
    if a.context_depth is None:
        a.context_depth = cfg["K"]
    if a.context_slots is None:
        a.context_slots = cfg["slots"]
    if a.prewarm_steps is None:
        a.prewarm_steps = cfg.get("prewarm", 10000)
    if a.parent_depth is None:
        a.parent_depth = cfg.get("R", 0)  # SQL: parents keyed 6 deep leave fewer tokens to re-walk
    a.batch_given = a.batch is not None
    return a


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def per_gpu_batch(args, world):
    if args.batch_given:
        return args.batch
    b = CONFIGS[args.config]["batch"]
    return max(1, b // world) if args.scaling == "strong" else b


def rank_seed(seed, rank):
    """Sequence streams of rank r (sequences are independent: each rank's
    batch is its own shard; rank 0's equal the CPU reference arm's)."""
    return seed + 7919 * rank


def logits_buffers(B, V1):
    """Rotating logits buffers: >= 3 x L2 of rows, so no step reads a row
    still resident in the 126 MB L2."""
    return max(2, -(-3 * L2_BYTES // (B * V1 * 2)))


def max_over_ranks(values, device, world):
    """Max of each timing over all ranks (NCCL on the GPUs, gloo in tests)."""
    if world <= 1:
        return [float(v) for v in values]
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def sum_over_ranks(values, device, world):
    """Sum of integer counters over all ranks (exact in int64)."""
    if world <= 1:
        return [int(v) for v in values]
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t]


def aggregate_rate(world, units_per_rank, seconds):
    """Whole-job throughput: every rank's units over the slowest rank's time
    (each rank owns its own sequences)."""
    return world * units_per_rank / seconds


def token_digest(tokens):
    """FNV-1a over the int32 ids of tokens[seq][step] in (sequence, step)
    order, 4 little-endian bytes each, >> 11 (ref_decode_run stats[5])."""
    h = 1469598103934665603
    for row in tokens:
        for v in row:
            v = int(v) & 0xFFFFFFFF
            for k in range(4):
                h = ((h ^ ((v >> (8 * k)) & 0xFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h >> 11


def summarize(samples):
    """Summarize (tools/gmask_main.cpp:135-149): mean, and p50/p99 by the
    rank rule idx = ceil(q*n) - 1."""
    s = sorted(samples)
    n = len(s)

    def rank(q):
        idx = max(0, int(q * n + 0.999999) - 1)
        return s[min(idx, n - 1)]
    return {"mean": sum(s) / n, "p50": rank(0.50), "p99": rank(0.99), "n": n}


def automaton_bytes(grammar: str) -> bytes:
    """json: the reference-built fixture automaton (tests/golden); the
    repo-authored workload grammars are compiled by our own compiler
    (gm_automaton_compile) — preprocessing, outside every timed region."""
    bnf = os.path.join(ROOT, "paper_2506_03887_b200", "grammars", grammar + ".bnf")
    if os.path.exists(bnf):
        import paper_2506_03887_b200 as pk
        with open(bnf) as f:
            return pk.Automaton.compile(f.read()).save()
    with open(os.path.join(ROOT, "tests", "golden", grammar + ".p3dpda"), "rb") as f:
        return f.read()


def reference_automaton_bytes(grammar: str) -> bytes:
    """The CPU arm's automaton, built without the product: the reference's
    own BuildDpda (oracle/_ref) for the repo-authored grammars, the
    reference-built fixture otherwise."""
    bnf = os.path.join(ROOT, "paper_2506_03887_b200", "grammars", grammar + ".bnf")
    if os.path.exists(bnf):
        import oracle
        if oracle.ref_available():
            rc, flat, _ = oracle.Ref.compile_flat(open(bnf).read())
            if rc == 0:
                return flat
        return automaton_bytes(grammar)
    with open(os.path.join(ROOT, "tests", "golden", grammar + ".p3dpda"), "rb") as f:
        return f.read()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """Samples SM clocks + throttle reasons via NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x1: "gpu_idle", 0x10: "sync_boost", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit and bit != 0x1:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU reference
def cpu_reference_run(flat: bytes, vocab, structural, batch_cpu: int, warmup: int, steps: int, seed: int,
                      threads: int, stack_cap: int, mode: str, rows: int):
    """The reference matcher (oracle/_ref, built from the reference's own
    sources) or, when absent, the C port — the only oracle use in bench.py."""
    import oracle
    greedy = mode == "greedy"
    if oracle.ref_available():
        eng = oracle.Ref(flat, vocab)
        stats, _, _ = eng.decode_run(structural, batch_cpu, steps, seed, threads=threads, stack_cap=stack_cap,
                                     warmup=warmup, logits_row=2 if greedy else 1, rows=rows,
                                     logit_seed=LOGIT_SEED, digest_seqs=DIGEST_SEQS)
        return stats, "reference", threads
    eng = oracle.Port(flat, vocab)
    stats, _, _ = eng.decode_run(structural, batch_cpu, warmup + steps, seed, stack_cap=stack_cap,
                                 greedy_rows=rows if greedy else 0, logit_seed=LOGIT_SEED, warmup=warmup,
                                 digest_seqs=DIGEST_SEQS)
    stats[0] *= steps / max(1, warmup + steps)
    stats[1] = batch_cpu * steps
    return stats, "port", 1


def cpu_step_rule(mode):
    if mode == "greedy":
        return "Engine::ComputeMask + argmax over allowed bf16 logits + Step per byte"
    return "Engine::ComputeMask + bf16 -inf row mask + stream sample + Step per byte"


def cpu_inputs(args):
    """The CPU arm's inputs, built from the oracle only (no product code)."""
    import oracle
    flat = reference_automaton_bytes(args.grammar)
    vocab = oracle.synth_vocab(args.vocab, args.flavor)
    return flat, vocab, oracle.structural_words(vocab)


def workload_config(args, world, B, R):
    cfg = CONFIGS[args.config]
    step = ("gm_decode_step_greedy (argmax fill + accept kernels)" if args.mode == "greedy" else
            "gm_decode_step_stream (one launch)" if args.one_launch else
            "gm_decode_step_stream_split (fill + overlapped sample/accept kernel: pure-CI sequences sample from "
            "their cached context row at once, the rest as their fill items arrive)")
    return {"workload": cfg["desc"].format(b=B), "config_index": args.config, "grammar": args.grammar,
            "vocab_bits": args.vocab + 1, "batch_per_gpu": B, "global_batch": B * world,
            "context_depth": args.context_depth, "parent_depth": args.parent_depth, "mode": args.mode,
            "step": step, "context_slots": args.context_slots,
            "l2": f"inputs larger than L2: {R} rotating logits buffers of {B * (args.vocab + 1) * 2 / 2**20:.0f} MiB "
                  f"(> 3 x 126 MB L2 in total)",
            "parallelism": f"dp{world} (sequence shards, no hot-path collective)"}


def reference_arm(args):
    """`--impl reference`: the reference's own CPU matcher (oracle/_ref) on
    all host cores, on this config's streams; rank 0 only."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    flat, vocab, structural = cpu_inputs(args)
    threads = os.cpu_count() or 1
    batch_cpu = max(DIGEST_SEQS, 2 * threads)
    B = per_gpu_batch(args, world)
    R = logits_buffers(B, args.vocab + 1)
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, args.warmup, args.steps,
                                        rank_seed(args.seed, 0), threads, args.stack_cap, args.mode, R)
    value = st[1] / st[0]
    sample = (f"{batch_cpu} sequences x {args.steps} timed steps (+{args.warmup} warm-up) of the same "
              f"workload (sequences 0..{batch_cpu - 1} of rank 0's streams); per seq-step: "
              f"{cpu_step_rule(args.mode)}; {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * st[0] / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": workload_config(args, world, B, R),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mask_latency_us_mean": 1e6 * st[0] / st[1] * cores,
        "check": {"token_digest": int(st[5]), "popcount_sum": int(st[6]), "sequences": DIGEST_SEQS,
                  "steps": args.steps, "after_warmup": args.warmup},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        reference_arm(args)
        return
    rank, local, world = dist_env()
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2506_03887_b200 as pk

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    t_comp = time.perf_counter()
    flat = automaton_bytes(args.grammar)
    t_comp = time.perf_counter() - t_comp
    vocab = pk.synth_vocab(args.vocab, args.flavor)
    automaton = pk.Automaton.load(flat)
    eng = pk.DeviceEngine(automaton, vocab, device=local, context_depth=args.context_depth,
                          context_slots=args.context_slots, parent_depth=args.parent_depth)
    B = per_gpu_batch(args, world)
    V, W = eng.V, eng.W
    V1 = V + 1
    seed = rank_seed(args.seed, rank)
    stream = torch.cuda.current_stream()
    greedy = args.mode == "greedy"
    R = logits_buffers(B, V1)
    logits = [torch.empty((B, V1), dtype=torch.bfloat16, device=dev) for _ in range(R)]
    for k, t in enumerate(logits):
        if greedy:  # the CPU reference arm reads the same rows (gp_synth_logit)
            pk.synth_logits(t, k, LOGIT_SEED)
        else:
            t.normal_()
    nseg = eng.info()["num_segments"]

    def make_step(batch, bm, counts, toks):
        def step(g, bm_=None, counts_=None, toks_=None):
            """Global step g reads logits buffer g % R (as the CPU arm does)."""
            bm_ = bm if bm_ is None else bm_
            counts_ = counts if counts_ is None else counts_
            toks_ = toks if toks_ is None else toks_
            if greedy:
                batch.decode_step_greedy(logits[g % R], tokens_out=toks_, bitmask=bm_)
            elif args.one_launch:
                batch.decode_step_stream(seed, bitmask=bm_, logits=logits[g % R], tokens_out=toks_)
            else:
                batch.decode_step_stream_split(seed, bitmask=bm_, logits=logits[g % R], seg_counts=counts_,
                                               tokens_out=toks_)
        return step

    # ---- cold cache: the first steps from an EMPTY context table (every
    # context met is built on the device inside the step), events between
    # steps; other streams than the timed ones.
    cold = None
    if args.cold_steps > 0:
        # CUDA loads kernels lazily, at their first launch: run the step's
        # kernels once on a throwaway engine so the cold-cache timing holds
        # only context builds, not module loading.
        weng = pk.DeviceEngine(automaton, vocab[:2000], device=local, context_depth=args.context_depth,
                               context_slots=64)
        wb = weng.batch(4, args.stack_cap)
        wlg = torch.zeros((4, 2001), dtype=torch.bfloat16, device=dev)
        for _ in range(2):
            if greedy:
                wb.decode_step_greedy(wlg)
            else:
                wb.decode_step_stream_split(1, logits=wlg)
        wb.check()
        del wb, weng, wlg
        torch.cuda.synchronize()
        cb = eng.batch(B, args.stack_cap)
        cbm = torch.zeros((B, W), dtype=torch.int32, device=dev)
        ccn = torch.zeros((B, nseg * 2), dtype=torch.int32, device=dev)
        ctk = torch.zeros(B, dtype=torch.int32, device=dev)
        cstep = make_step(cb, cbm, ccn, ctk)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.cold_steps + 1)]
        evs[0].record(stream)
        seed_saved = seed
        seed = seed ^ 0xC01DCAFE
        for i in range(args.cold_steps):
            cstep(i)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        seed = seed_saved
        cb.check()
        lat = [1e3 * evs[i].elapsed_time(evs[i + 1]) for i in range(args.cold_steps)]
        cold = dict(summarize(lat), first_step_us=lat[0], unit="us",
                    contexts_built=eng.info()["context_slots_used"],
                    note=f"{args.cold_steps} steps of {B} sequences from an empty context table (before the "
                         "prewarm; streams seeded apart from the timed ones)")
        del cstep, cb, cbm, ccn, ctk  # the batch goes away: its queued builds are drained

    t_pre = time.perf_counter()
    if args.prewarm_steps > 0:
        eng.prewarm(args.prewarm_batch, args.prewarm_steps, seed=0xC0FFEE + rank, stack_capacity=args.stack_cap)
    t_pre = time.perf_counter() - t_pre
    pre_info = eng.info()
    # The prewarmed context table as a snapshot file (gm_engine_snapshot_*,
    # "P3GMCTX1"): saved, then loaded into a fresh engine that runs everything
    # below — the load a restarted server (or every rank of a node) does
    # instead of the prewarm; the timed digests check the loaded table.
    snap = None
    if args.prewarm_steps > 0 and not args.no_snapshot:
        import tempfile
        path = os.path.join(tempfile.gettempdir(), f"pre3_contexts_rank{rank}.p3gmctx")
        t0 = time.perf_counter()
        nbytes = eng.save_contexts(path)
        t_save = time.perf_counter() - t0
        del eng
        t0 = time.perf_counter()
        eng = pk.DeviceEngine(automaton, vocab, device=local, context_depth=args.context_depth,
                              context_slots=args.context_slots, parent_depth=args.parent_depth)
        t_create = time.perf_counter() - t0
        t0 = time.perf_counter()
        eng.load_contexts(path)
        torch.cuda.synchronize()
        t_load = time.perf_counter() - t0
        os.unlink(path)
        snap = {"bytes": int(nbytes), "contexts": eng.info()["context_slots_used"], "save_s": t_save,
                "engine_create_s": t_create, "load_s": t_load,
                "note": "the timed engine was created fresh and loaded from the prewarmed engine's snapshot"}

    batch = eng.batch(B, args.stack_cap)
    K, Wm = args.steps, args.warmup
    bm = torch.zeros((B, W), dtype=torch.int32, device=dev)
    toks = torch.zeros(B, dtype=torch.int32, device=dev)
    # Per-timed-step outputs, so the timed region leaves its own evidence:
    # token ids [K][B] and sampler counts [K][B][nseg][2] (greedy: bitmask
    # rows [K][B][W] when they fit 8 GB) — written by the kernels in place of
    # the single buffers, no extra work in the step.
    toks_all = torch.zeros((K, B), dtype=torch.int32, device=dev)
    counts_all = None if greedy else torch.zeros((K, B, nseg * 2), dtype=torch.int32, device=dev)
    counts = torch.zeros((B, nseg * 2), dtype=torch.int32, device=dev)
    bm_all = None
    if greedy and K * B * W * 4 <= 8 << 30:
        bm_all = torch.zeros((K, B, W), dtype=torch.int32, device=dev)
    step = make_step(batch, bm, counts, toks)

    for i in range(Wm):
        step(i)
    batch.check()
    # The timed steps as one captured CUDA graph (gm_decode_graph_create; a
    # multiple of 6 steps, the rest enqueued eagerly): one host call launches
    # them, with every step's own buffers baked in.
    Kg = 0 if (args.no_graph or args.one_launch) else K - K % 6
    graph = None
    if Kg:
        graph = batch.capture_steps(
            Kg, greedy=greedy, seed=seed, logits=[logits[(Wm + i) % R] for i in range(Kg)],
            bitmask=[bm_all[i] for i in range(Kg)] if bm_all is not None else bm,
            seg_counts=None if greedy else [counts_all[i] for i in range(Kg)],
            tokens_out=[toks_all[i] for i in range(Kg)])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        h0 = time.perf_counter()
        e0.record(stream)
        if graph is not None:
            graph.launch()
        for i in range(Kg, K):
            step(Wm + i, bm_=bm_all[i] if bm_all is not None else None,
                 counts_=counts_all[i] if counts_all is not None else None, toks_=toks_all[i])
        e1.record(stream)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
    del graph
    batch.check()
    if world > 1:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    host_ms = (h1 - h0) * 1e3 / K
    g = Wm + K  # next global step

    # ---- in-run evidence of the timed steps (sequences 0..31).
    tk = toks_all[:, :DIGEST_SEQS].cpu().numpy().T  # [seq][step]
    digest = token_digest(tk)
    if counts_all is not None:
        pop = int(counts_all[:, :DIGEST_SEQS, 0::2].to(torch.int64).sum().item())
    elif bm_all is not None:
        rows = bm_all[:, :DIGEST_SEQS].cpu().numpy().view(np.uint32).copy()
        rows[:, :, V >> 5] &= np.uint32(~(1 << (V & 31)) & 0xFFFFFFFF)  # EOS excluded
        pop = int(np.unpackbits(rows.view(np.uint8)).sum())
    else:
        pop = None
    del bm_all, counts_all

    # ---- roofline sub-loop: every step's fill kernel bracketed by events
    # (an event between two launches stops the accept from overlapping that
    # fill, so this runs apart from the timed loop).
    nf = max(10, args.fill_samples)
    fev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(nf)]
    for pair in fev:  # create the CUDA events (their handles go through the C ABI)
        for e_ in pair:
            e_.record(stream)
    torch.cuda.synchronize()
    for i in range(nf):
        batch.time_next_fill(*fev[i])
        step(g)
        g += 1
    torch.cuda.synchronize()
    fill = [a.elapsed_time(b) for a, b in fev]
    fill_ms = sum(fill) / len(fill)
    fill_s = summarize([1e3 * x for x in fill])

    # ---- latency sub-loop: events between steps (per-step latency, no
    # overlap with the neighbouring steps).
    nl = max(10, args.latency_samples)
    lev = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
    lev[0].record(stream)
    for i in range(nl):
        step(g)
        g += 1
        lev[i + 1].record(stream)
    torch.cuda.synchronize()
    step_lat = summarize([1e3 * lev[i].elapsed_time(lev[i + 1]) for i in range(nl)])

    # ---- device-counted logit bytes per sequence-step (stats on, apart).
    batch.set_stats(True)
    ns = 8
    for i in range(ns):
        step(g)
        g += 1
    batch.check()
    fstats = batch.fill_stats()
    batch.set_stats(False)
    logit_rd = fstats["logit_bytes_read"] / (B * ns)
    logit_wr = fstats["logit_bytes_written"] / (B * ns)
    max_depth = max(len(batch.get(b).stack) for b in range(min(B, 256)))
    counters = batch.counters()

    elapsed_ms, fill_ms = max_over_ranks([elapsed_ms, fill_ms], dev, world)
    value = aggregate_rate(world, B * K, elapsed_ms / 1e3)
    tot_seq_steps, tot_restarts, digest_sum = sum_over_ranks(
        [B * K, counters["restarts"], digest], dev, world)

    # ---- e2e through the public C ABI with host buffers, driven by a C++
    # caller (paper_2506_03887_b200/tools/e2e_driver.cpp; Python's per-call
    # overhead would otherwise dominate).  Every step: H2D of the host-held
    # token ids, gm_accept_tokens + gm_fill_and_mask_logits + gm_sample_stream
    # (greedy: gm_decode_step_greedy), D2H of the sampled ids (stored by the
    # kernel straight into mapped pinned memory, waited for: the next step
    # needs them) and of the full bitmask (a copy stream into double-buffered
    # pinned memory, overlapping the next step); the timed region ends after
    # the last copy lands.
    e2e = None
    if not args.no_e2e:
        import ctypes
        drv = ctypes.CDLL(os.path.join(ROOT, "paper_2506_03887_b200", "libpre3e2e.so"))
        drv.e2e_run.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
        drv.e2e_run.restype = ctypes.c_int
        Ke = max(10, min(K, 200))
        ptrs = (ctypes.c_uint64 * R)(*[t.data_ptr() for t in logits])
        secs = ctypes.c_double()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        rc = drv.e2e_run(batch._h, 1 if greedy else 0, B, W, batch.nseg, ptrs, R, V1, seed & (2**64 - 1), 3, Ke,
                         local, 1, ctypes.byref(secs))
        if rc != 0:
            raise RuntimeError(f"e2e driver failed: {rc} {pk.lib().gm_last_error().decode()}")
        t_full = secs.value
        # The same loop without the 16 KB/sequence bitmask read-back (the mask
        # consumed only on the device): reported beside, not as the headline.
        rc = drv.e2e_run(batch._h, 1 if greedy else 0, B, W, batch.nseg, ptrs, R, V1, seed & (2**64 - 1), 3, Ke,
                         local, 0, ctypes.byref(secs))
        if rc != 0:
            raise RuntimeError(f"e2e driver failed: {rc} {pk.lib().gm_last_error().decode()}")
        t_full, t_ids = max_over_ranks([t_full, secs.value], dev, world)
        path = ("C++ caller: gm_decode_step_greedy(device logits) → ids into mapped host memory; D2H bitmask "
                "on a copy stream" if greedy else "C++ caller: H2D ids → gm_accept_tokens → "
                "gm_fill_and_mask_logits → gm_sample_stream (ids into mapped host memory) → stream sync; D2H "
                "bitmask on a copy stream (double-buffered)")
        e2e = {"value": aggregate_rate(world, B * Ke, t_full), "unit": UNIT,
               "h2d_bytes_per_step": 0 if greedy else B * 4, "d2h_bytes_per_step": B * W * 4 + B * 4,
               "steps": Ke, "path": path,
               "ids_only": {"value": aggregate_rate(world, B * Ke, t_ids), "d2h_bytes_per_step": B * 4,
                            "note": "same loop without the bitmask read-back (mask consumed on the device)"}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src, _ = peaks()
    if greedy:
        # Bytes the argmax formulation moves (never count bytes
        # it does not have to move): bitmask write + context bitset read + the
        # 16-B logit chunks holding an allowed token (device-counted).
        alg_bytes_seq = 8 * W + logit_rd
        alg_rule = "8W (bitmask write + CI read) + device-counted allowed-chunk logit reads"
    else:
        alg_bytes_seq = 2 * V1 + 8 * W  # write-only -inf formulation
        alg_rule = "2(V+1) (-inf row write) + 8W (bitmask write + CI read); mixed-chunk reads not counted"
    # The roofline kernel's launch duration: when it is the step's only
    # kernel (the one-grid split step, the one-launch step) the timed loop's
    # time per launch (consecutive launches pipelined by PDL, as in a decode
    # loop); otherwise the isolated launches of the sub-loop above (the accept
    # kernel cannot overlap them).  Both are reported.
    split_launches = batch.split_step_launches
    launches_per_step = 2 if greedy else 1 if args.one_launch else split_launches
    kernel_ms = elapsed_ms / K if launches_per_step == 1 else fill_ms
    duration_src = ("timed loop: elapsed / launches (the step is one launch of this kernel)"
                    if launches_per_step == 1 else
                    "isolated launches (events around each fill in a sub-loop; mean)")
    achieved = B * alg_bytes_seq / (kernel_ms / 1e3) / 1e9
    isolated_frac = B * alg_bytes_seq / (fill_ms / 1e3) / 1e9 / peak
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            key = f"{args.grammar}:{args.vocab}:{B}:{args.mode}:{'fused' if args.one_launch else 'separate'}"
            entry = json.load(open(tpath)).get(key)
            traffic = entry["dram_bytes_per_launch"] if entry else None
        except Exception:
            traffic = None

    # ---- CPU reference beside the GPU (rank 0, N=1): the reference matcher
    # on the host cores over a bounded sample, and its digest of the SAME
    # timed steps of sequences 0..31 (the parity check of the timed output).
    cpu = None
    check = {"token_digest": digest, "popcount_sum": pop, "sequences": DIGEST_SEQS, "steps": K,
             "after_warmup": Wm}
    if world == 1 and not args.no_cpu_baseline:
        cflat, cvocab, cstruct = cpu_inputs(args)
        threads = os.cpu_count() or 1
        st, kind, cores = cpu_reference_run(cflat, cvocab, cstruct, DIGEST_SEQS, Wm, K, seed, threads,
                                            args.stack_cap, args.mode, R)
        check.update(cpu_reference_digest=int(st[5]), cpu_reference_popcount=int(st[6]), cpu_kind=kind,
                     equal=(int(st[5]) == digest and (pop is None or int(st[6]) == pop)))
        bcpu = max(DIGEST_SEQS, 2 * threads)
        st, kind, cores = cpu_reference_run(cflat, cvocab, cstruct, bcpu, 0, 1, seed, threads, args.stack_cap,
                                            args.mode, R)
        steps_cpu = int(max(2, min(200, args.cpu_seconds / max(st[0], 1e-4))))
        st, kind, cores = cpu_reference_run(cflat, cvocab, cstruct, bcpu, 1, steps_cpu, seed, threads,
                                            args.stack_cap, args.mode, R)
        st1, _, _ = cpu_reference_run(cflat, cvocab, cstruct, 4, 1, max(2, steps_cpu // 4), seed, 1,
                                      args.stack_cap, args.mode, R)
        cpu = {"value": st[1] / st[0], "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{bcpu} sequences x {steps_cpu} steps of the same workload ({st[0]:.1f} s), "
                         f"threads={cores}, per seq-step {cpu_step_rule(args.mode)}",
               "cpu_model": cpu_model(), "one_core": {"value": st1[1] / st1[0], "unit": UNIT,
                                                      "sample": f"4 sequences x {max(2, steps_cpu // 4)} steps"}}

    info = eng.info()
    kname = ("FillKernel<greedy> (mask + argmax over allowed logits; accept runs in AcceptKernel)" if greedy else
             "FillKernel (one-launch step: fill + -inf logits + sample/accept tail)" if args.one_launch else
             "FillKernel (split step in one grid: fill + -inf logits, the sample/accept CTAs interleaved with "
             "the light CTAs)" if split_launches == 1 else
             "FillKernel (fill + -inf logits; accept runs in AcceptKernel)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (seeded token-level streams, "
                                  + ("gp_synth_logit bf16 logits)" if greedy else "random bf16 logits)"),
        "config": workload_config(args, world, B, R),
        "mask_latency_us": 1e3 * fill_ms,
        "step_latency_us": step_lat,
        "step_breakdown_us": {"step_mean_timed_loop": 1e3 * elapsed_ms / K, "roofline_kernel": fill_s,
                              "host_enqueue_per_step": 1e3 * host_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": kname,
                     "samples": nf, "alg_bytes_per_seq_step": alg_bytes_seq, "alg_bytes_rule": alg_rule,
                     "duration_us": 1e3 * kernel_ms, "duration_source": duration_src,
                     "isolated_launch_frac": isolated_frac,
                     "timed_loop_frac": B * alg_bytes_seq / (elapsed_ms / K / 1e3) / 1e9 / peak,
                     "device_counted_logit_bytes_per_seq_step": {"read": logit_rd, "written": logit_wr}},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "check": check,
        "gpu_launches": K * launches_per_step,  # greedy: fill + accept per step; split: gm_split_step_launches()
        "launch": (f"CUDA graph of {Kg} steps (one gm_graph_launch)" + (f" + {K - Kg} eager steps" if K > Kg else "")
                   if Kg else "eager, one ABI call per step"),
        "clocks": clocks.summary(),
        "cold_cache": cold,
        "preprocessing": {"compile_s": t_comp, "prewarm_s": t_pre, "snapshot": snap,
                          "prewarm": f"{args.prewarm_steps} steps x {args.prewarm_batch} seqs "
                          f"(seed differs from the timed streams)",
                          "contexts_after_prewarm": pre_info["context_slots_used"],
                          "automaton": automaton.info()},
        "cache": {"contexts": info["context_slots_used"], "segment_builds": info["segment_builds"],
                  "private_builds": info["private_builds"], "parent_builds": info["parent_builds"],
                  "last_fill": fstats},
        "totals": {"seq_steps": tot_seq_steps, "restarts": tot_restarts, "digest_sum_over_ranks": digest_sum},
        "max_stack_depth_seen": max_depth,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
