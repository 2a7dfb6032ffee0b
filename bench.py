#!/usr/bin/env python
"""bench.py — masked decode steps/sec of the constrained-decoding hot path.

Default workload (BASELINE.json configs[1], "config 2"): JSON LR(1) grammar,
Llama-3-sized vocabulary (128,255 tokens + EOS = 128,256 mask bits), batch
256 sequences per GPU.  One step = mask fill + in-place bf16 -inf logit
masking + synthetic-stream sampling + accept_token with restart, for every
sequence of the batch, as one launch (gm_decode_step_stream; --separate: the
reference-shaped two calls gm_fill_and_mask_logits + gm_sample_stream_and_accept).

Other BASELINE configs (parity cases for the judge's scaling / extra lines):
    --config 3   schema grammar (repo-authored, compiled here), batch 1024
    --config 4   SQL-subset grammar, 4096 sequences in total split over the
                 GPUs (strong scaling)
    --config 5   JSON, 512/GPU, greedy decode: mask + argmax over the allowed
                 bf16 logits + accept (gm_decode_step_greedy)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Under torchrun each rank drives one GPU with its own sequences (no collective
on the hot path — NCCL only reduces the final timings).  Prints ONE JSON line
on rank 0.  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "masked decode steps/sec (batch×steps) and per-step mask latency at 128k vocab"
UNIT = "seq-steps/s"
L2_BYTES = 126 * 1024 * 1024

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


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=30)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, choices=sorted(CONFIGS), default=2)
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
    p.add_argument("--separate", action="store_true",
                   help="stream mode: two launches per step (fill+mask logits, then sample+accept; the default)")
    p.add_argument("--one-launch", action="store_true", help="stream mode: force the one-launch fused step")
    p.add_argument("--sample-every", type=int, default=16,
                   help="bracket the roofline kernel with events on every Nth timed step (diagnostics: a large N "
                        "shows the step rate without the sampled steps)")
    p.add_argument("--fused", action="store_true", help=argparse.SUPPRESS)  # the default; kept for scripts
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    p.add_argument("--no-north-star", action="store_true",
                   help="skip the extra batch-1024 fill-kernel roofline measurement of the default config")
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


def max_over_ranks(values, device, world):
    """Max of each timing over all ranks (NCCL on the GPUs, gloo in tests)."""
    if world <= 1:
        return [float(v) for v in values]
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def aggregate_rate(world, units_per_rank, seconds):
    """Whole-job throughput: every rank's units over the slowest rank's time
    (each rank owns its own sequences)."""
    return world * units_per_rank / seconds


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


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


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


def cpu_reference_run(flat: bytes, vocab, structural, batch_cpu: int, warmup: int, steps: int, seed: int,
                      threads: int, stack_cap: int, mode: str):
    """The reference matcher (oracle/_ref, built from the reference's own
    sources) or, when absent, the C port — the only oracle use in bench.py."""
    import oracle
    if oracle.ref_available():
        eng = oracle.Ref(flat, vocab)
        stats, _, _ = eng.decode_run(structural, batch_cpu, steps, seed, threads=threads, stack_cap=stack_cap,
                                     warmup=warmup, logits_row=2 if mode == "greedy" else 1)
        return stats, "reference", threads
    eng = oracle.Port(flat, vocab)
    stats, _, _ = eng.decode_run(structural, batch_cpu, warmup + steps, seed, stack_cap=stack_cap)
    stats[0] *= steps / max(1, warmup + steps)
    stats[1] = batch_cpu * steps
    return stats, "port", 1


def cpu_step_rule(mode):
    if mode == "greedy":
        return "Engine::ComputeMask + argmax over allowed bf16 logits + Step per byte"
    return "Engine::ComputeMask + bf16 -inf row mask + stream sample + Step per byte"


def calibrated_cpu_sample(flat, vocab, structural, seed, stack_cap, budget_s, mode):
    threads = os.cpu_count() or 1
    batch_cpu = 2 * threads
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, 0, 1, seed, threads, stack_cap, mode)
    per_step = max(st[0], 1e-4)
    steps = int(max(2, min(200, budget_s / per_step)))
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, 1, steps, seed, threads, stack_cap,
                                        mode)
    return st, kind, cores, batch_cpu, steps


def workload_config(args, world, B):
    cfg = CONFIGS[args.config]
    return {"workload": cfg["desc"].format(b=B), "config_index": args.config, "grammar": args.grammar,
            "vocab_bits": args.vocab + 1, "batch_per_gpu": B, "global_batch": B * world,
            "context_depth": args.context_depth, "parent_depth": args.parent_depth, "mode": args.mode,
            "step": (f"gm_decode_step_greedy (argmax fill + accept kernels; every {args.sample_every}th step with "
                     "events around its fill kernel)" if args.mode == "greedy" else
                     "gm_decode_step_stream (one launch)" if args.one_launch else
                     "gm_decode_step_stream_split (fill + overlapped sample/accept kernel: pure-CI sequences "
                     "sample from their cached context row at once, the rest as their fill items arrive); "
                     f"every {args.sample_every}th step with events around its fill kernel (no overlap "
                     "in that step)"),
            "context_slots": args.context_slots,
            "parallelism": f"dp{world} (sequence shards, no hot-path collective)"}


def reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import paper_2506_03887_b200 as pk
    flat = automaton_bytes(args.grammar)
    vocab = pk.synth_vocab(args.vocab, args.flavor)
    structural = pk.structural_words(vocab)
    threads = os.cpu_count() or 1
    batch_cpu = 2 * threads
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, args.warmup, args.steps, args.seed,
                                        threads, args.stack_cap, args.mode)
    value = st[1] / st[0]
    sample = (f"{batch_cpu} sequences x {args.steps} timed steps (+{args.warmup} warm-up) of the same "
              f"workload; per seq-step: {cpu_step_rule(args.mode)}")
    B = per_gpu_batch(args, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * st[0] / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": workload_config(args, world, B),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mask_latency_us_mean": 1e6 * st[0] / st[1] * cores,
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        reference_arm(args)
        return
    rank, local, world = dist_env()
    import numpy as np  # noqa: F401
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
    t_pre = time.perf_counter()
    if args.prewarm_steps > 0:
        eng.prewarm(args.prewarm_batch, args.prewarm_steps, seed=0xC0FFEE + rank)
    t_pre = time.perf_counter() - t_pre
    pre_info = eng.info()
    B = per_gpu_batch(args, world)
    V, W = eng.V, eng.W
    V1 = V + 1
    batch = eng.batch(B, args.stack_cap)
    seed = args.seed + 7919 * rank
    stream = torch.cuda.current_stream()
    bm = torch.zeros((B, W), dtype=torch.int32, device=dev)
    counts = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=dev)
    toks = torch.zeros(B, dtype=torch.int32, device=dev)
    row_bytes = B * V1 * 2
    R = max(2, -(-3 * L2_BYTES // row_bytes))
    logits = [torch.randn((B, V1), dtype=torch.bfloat16, device=dev) for _ in range(R)]
    greedy = args.mode == "greedy"
    # One launch per step wins while the batch leaves the GPU latency-bound;
    # above 512 sequences the standalone accept kernel's parallelism wins.
    separate = not greedy and not args.one_launch

    def step(i):
        if greedy:
            batch.decode_step_greedy(logits[i % R], tokens_out=toks, bitmask=bm)
        elif separate:
            batch.decode_step_stream_split(seed, bitmask=bm, logits=logits[i % R], seg_counts=counts, tokens_out=toks)
        else:
            batch.decode_step_stream(seed, bitmask=bm, logits=logits[i % R], tokens_out=toks)

    for i in range(args.warmup):
        step(i)
    batch.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    K = args.steps
    # The roofline kernel is bracketed by events on every 16th step only: an
    # event between two launches stops the next kernel from starting under the
    # previous one's last wave (programmatic dependent launch), which the
    # other steps keep.
    SAMPLE_EVERY = max(1, args.sample_every)
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(0, K, SAMPLE_EVERY)]
    for pair in ev:  # create the CUDA events (their handles go through the C ABI)
        for e_ in pair:
            e_.record(stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        h0 = time.perf_counter()
        e0.record(stream)
        for i in range(K):
            timed = i % SAMPLE_EVERY == 0
            if timed:  # events bracket the step's fill kernel alone (the roofline kernel)
                batch.time_next_fill(*ev[i // SAMPLE_EVERY])
            step(i)
        e1.record(stream)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
    batch.check()
    if world > 1:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    kern = sorted(a.elapsed_time(b) for a, b in ev)
    kern_ms = sum(kern) / len(kern)
    kern_p50 = kern[len(kern) // 2]
    host_ms = (h1 - h0) * 1e3 / K
    elapsed_ms, kern_ms = max_over_ranks([elapsed_ms, kern_ms], dev, world)
    value = aggregate_rate(world, B * K, elapsed_ms / 1e3)

    # North-star check (BASELINE.json: >= 60 % of HBM bandwidth at batch >= 1024):
    # the same grammar and step at 1,024 sequences, fill kernel timed alone
    # (outside the headline timed region; its own warm-up and rotation).
    north = None
    if (world == 1 and not args.no_north_star and not greedy and B < 1024 and args.config == 2):
        Bn = 1024
        bn = eng.batch(Bn, args.stack_cap)
        bmn = torch.zeros((Bn, W), dtype=torch.int32, device=dev)
        cn = torch.zeros((Bn, bn.nseg * 2), dtype=torch.int32, device=dev)
        tn = torch.zeros(Bn, dtype=torch.int32, device=dev)
        Rn = max(2, -(-3 * L2_BYTES // (Bn * V1 * 2)))
        lgn = [torch.randn((Bn, V1), dtype=torch.bfloat16, device=dev) for _ in range(Rn)]
        for i in range(30):
            bn.decode_step_stream_split(seed, bitmask=bmn, logits=lgn[i % Rn], seg_counts=cn, tokens_out=tn)
        torch.cuda.synchronize()
        Kn = 120
        evn = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(0, Kn, 8)]
        for pair in evn:
            for e_ in pair:
                e_.record(stream)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for i in range(Kn):
            if i % 8 == 0:
                bn.time_next_fill(*evn[i // 8])
            bn.decode_step_stream_split(seed, bitmask=bmn, logits=lgn[i % Rn], seg_counts=cn, tokens_out=tn)
        f1.record(stream)
        torch.cuda.synchronize()
        bn.check()
        fill_ms_n = sum(a.elapsed_time(c) for a, c in evn) / len(evn)
        pk_gbs, _, _ = peaks()
        ach_n = Bn * (2 * V1 + 8 * W) / (fill_ms_n / 1e3) / 1e9
        north = {"batch": Bn, "step": "gm_decode_step_stream_split (every 8th step with events around its fill)",
                 "fill_kernel_us": 1e3 * fill_ms_n, "achieved_gbs": ach_n, "frac": ach_n / pk_gbs,
                 "seq_steps_per_s": Bn * Kn / (f0.elapsed_time(f1) / 1e3), "steps": Kn}
        del bn, lgn

    # Device-counted logit bytes of one more step (outside the timed region).
    batch.set_stats(True)
    step(K)
    batch.check()
    fstats = batch.fill_stats()
    batch.set_stats(False)
    max_depth = max(batch.get(b).stack.__len__() for b in range(min(B, 256)))

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
        t_e2e = t_full
        path = ("C++ caller: gm_decode_step_greedy(device logits) → ids into mapped host memory; D2H bitmask "
                "on a copy stream" if greedy else "C++ caller: H2D ids → gm_accept_tokens → "
                "gm_fill_and_mask_logits → gm_sample_stream (ids into mapped host memory) → stream sync; D2H "
                "bitmask on a copy stream (double-buffered)")
        e2e = {"value": aggregate_rate(world, B * Ke, t_e2e), "unit": UNIT,
               "h2d_bytes_per_step": 0 if greedy else B * 4, "d2h_bytes_per_step": B * W * 4 + B * 4,
               "steps": Ke, "path": path,
               "ids_only": {"value": aggregate_rate(world, B * Ke, t_ids), "d2h_bytes_per_step": B * 4,
                            "note": "same loop without the bitmask read-back (mask consumed on the device)"}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src, _ = peaks()
    alg_bytes_seq = 2 * V1 + 8 * W          # write-only -inf / read-once argmax formulation
    achieved = B * alg_bytes_seq / (kern_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            key = f"{args.grammar}:{args.vocab}:{B}:{args.mode}:{'separate' if separate else 'fused'}"
            entry = json.load(open(tpath)).get(key)
            traffic = entry["dram_bytes_per_launch"] if entry else None
        except Exception:
            traffic = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        st, kind, cores, bcpu, steps_cpu = calibrated_cpu_sample(flat, vocab, eng.structural, args.seed,
                                                                 args.stack_cap, args.cpu_seconds, args.mode)
        cpu = {"value": st[1] / st[0], "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{bcpu} sequences x {steps_cpu} steps of the same workload ({st[0]:.1f} s), "
                         f"threads={cores}, per seq-step {cpu_step_rule(args.mode)}"}

    info = eng.info()
    kname = ("FillKernel<greedy> (mask + argmax over allowed logits; accept runs in AcceptKernel)" if greedy else
             "FillKernel (fill + -inf logits; accept runs in AcceptKernel)" if separate else
             "FillKernel (one-launch step: fill + -inf logits + sample/accept tail)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (seeded token-level streams, random bf16 logits)",
        "config": dict(workload_config(args, world, B),
                       l2=f"rotating {R} logits buffers of {row_bytes / 2**20:.0f} MiB (> 126 MB L2)"),
        "mask_latency_us": 1e3 * kern_ms,
        "step_breakdown_us": {"roofline_kernel_mean": 1e3 * kern_ms, "roofline_kernel_p50": 1e3 * kern_p50,
                              "host_enqueue_per_step": 1e3 * host_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": kname,
                     "alg_bytes_per_seq_step": alg_bytes_seq,
                     "device_counted_logit_bytes_per_seq_step": (fstats["logit_bytes_read"] +
                                                                 fstats["logit_bytes_written"]) / B},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": K * (1 if args.one_launch else 2),  # split / greedy: fill + accept per step
        "clocks": clocks.summary(),
        "preprocessing": {"compile_s": t_comp, "prewarm_s": t_pre,
                          "prewarm": f"{args.prewarm_steps} steps x {args.prewarm_batch} seqs "
                          f"(seed differs from the timed streams)", "contexts_after_prewarm": pre_info["context_slots_used"],
                          "automaton": automaton.info()},
        "cache": {"contexts": info["context_slots_used"], "segment_builds": info["segment_builds"],
                  "private_builds": info["private_builds"], "parent_builds": info["parent_builds"],
                  "last_fill": fstats},
        "max_stack_depth_seen": max_depth,
        "north_star_batch1024": north,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
