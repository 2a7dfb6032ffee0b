#!/usr/bin/env python
"""bench.py — masked decode steps/sec of the constrained-decoding hot path.

Workload (BASELINE.json configs[1]): JSON LR(1) grammar, Llama-3-sized
vocabulary (128,255 tokens + EOS = 128,256 mask bits), batch 256 sequences per
GPU.  One step = fused mask fill + in-place bf16 -inf logit masking
(gm_fill_and_mask_logits) + synthetic-stream sampling + accept_token with
restart (gm_sample_stream_and_accept), every sequence of the batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank drives one GPU with its own 256 sequences (weak
scaling; no collective on the hot path — NCCL only reduces the final timings).
Prints ONE JSON line on rank 0.  See DESIGN.md §7 for every field.
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=30)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--batch", type=int, default=256, help="sequences per GPU")
    p.add_argument("--vocab", type=int, default=128255, help="regular tokens (EOS adds one bit)")
    p.add_argument("--grammar", default="json")
    p.add_argument("--context-depth", type=int, default=12)
    p.add_argument("--context-slots", type=int, default=8192, help="context-cache hash table slots (power of two)")
    p.add_argument("--prewarm-steps", type=int, default=2000,
                   help="context-cache preprocessing: synthetic decode steps (other seed) before timing")
    p.add_argument("--prewarm-batch", type=int, default=1024)
    p.add_argument("--stack-cap", type=int, default=1024)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--fused", action="store_true", help="one-launch decode step (gm_decode_step_stream)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


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
    (weak scaling: each rank owns its own sequences)."""
    return world * units_per_rank / seconds


def automaton_bytes(grammar: str) -> bytes:
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
                      threads: int, stack_cap: int):
    """The reference matcher (oracle/_ref, built from the reference's own
    sources) or, when absent, the C port — the only oracle use in bench.py."""
    import oracle
    if oracle.ref_available():
        eng = oracle.Ref(flat, vocab)
        stats, _, _ = eng.decode_run(structural, batch_cpu, steps, seed, threads=threads, stack_cap=stack_cap,
                                     warmup=warmup)
        return stats, "reference", threads
    eng = oracle.Port(flat, vocab)
    stats, _, _ = eng.decode_run(structural, batch_cpu, warmup + steps, seed, stack_cap=stack_cap)
    stats[0] *= steps / max(1, warmup + steps)
    stats[1] = batch_cpu * steps
    return stats, "port", 1


def calibrated_cpu_sample(flat, vocab, structural, seed, stack_cap, budget_s):
    threads = os.cpu_count() or 1
    batch_cpu = 2 * threads
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, 0, 1, seed, threads, stack_cap)
    per_step = max(st[0], 1e-4)
    steps = int(max(2, min(200, budget_s / per_step)))
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, 1, steps, seed, threads, stack_cap)
    return st, kind, cores, batch_cpu, steps


def reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import paper_2506_03887_b200 as pk
    flat = automaton_bytes(args.grammar)
    vocab = pk.synth_vocab(args.vocab)
    structural = pk.structural_words(vocab)
    threads = os.cpu_count() or 1
    batch_cpu = 2 * threads
    st, kind, cores = cpu_reference_run(flat, vocab, structural, batch_cpu, args.warmup, args.steps, args.seed,
                                        threads, args.stack_cap)
    value = st[1] / st[0]
    sample = (f"{batch_cpu} sequences x {args.steps} timed steps (+{args.warmup} warm-up) of the same "
              f"workload; per seq-step: Engine::ComputeMask + bf16 -inf row mask + stream sample + Step per byte")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * st[0] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mask_latency_us_mean": 1e6 * st[0] / st[1] * cores,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    return {"workload": f"config2: {args.grammar} LR(1) grammar, {args.vocab + 1}-bit vocab "
                        f"(synthetic 128k tokens), batch {args.batch}/GPU, fused mask-fill + in-place bf16 -inf "
                        f"logit masking + stream sample + accept_token",
            "grammar": args.grammar, "vocab_bits": args.vocab + 1, "batch_per_gpu": args.batch,
            "global_batch": args.batch * world, "context_depth": args.context_depth,
            "parallelism": f"dp{world} (sequence shards, no hot-path collective)"}


def main():
    args = parse()
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
    flat = automaton_bytes(args.grammar)
    vocab = pk.synth_vocab(args.vocab)
    eng = pk.DeviceEngine(pk.Automaton.load(flat), vocab, device=local, context_depth=args.context_depth,
                          context_slots=args.context_slots)
    t_pre = time.perf_counter()
    if args.prewarm_steps > 0:
        eng.prewarm(args.prewarm_batch, args.prewarm_steps, seed=0xC0FFEE + rank)
    t_pre = time.perf_counter() - t_pre
    pre_info = eng.info()
    B, V, W = args.batch, eng.V, eng.W
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

    def step(i):
        if args.fused:
            batch.decode_step_stream(seed, bitmask=bm, logits=logits[i % R], tokens_out=toks)
        else:
            batch.fill(bm, logits[i % R], counts)
            batch.sample_stream_and_accept(bm, counts, seed, toks)

    for i in range(args.warmup):
        step(i)
    batch.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    K = args.steps
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(K)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        h0 = time.perf_counter()
        e0.record(stream)
        for i in range(K):
            ev[i][0].record(stream)
            if args.fused:
                step(i)
                ev[i][1].record(stream)
            else:  # events bracket the fill kernel alone (the roofline kernel)
                batch.fill(bm, logits[i % R], counts)
                ev[i][1].record(stream)
                batch.sample_stream_and_accept(bm, counts, seed, toks)
        e1.record(stream)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
    batch.check()
    if world > 1:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    fill_ms = sum(a.elapsed_time(b) for a, b in ev) / K
    host_ms = (h1 - h0) * 1e3 / K
    elapsed_ms, fill_ms = max_over_ranks([elapsed_ms, fill_ms], dev, world)
    value = aggregate_rate(world, B * K, elapsed_ms / 1e3)

    # Device-counted logit bytes of one more fill (outside the timed region).
    batch.set_stats(True)
    step(K)
    batch.check()
    fstats = batch.fill_stats()
    batch.set_stats(False)

    # ---- e2e through the public API with host buffers.
    e2e = None
    if not args.no_e2e:
        tok_host = torch.full((B,), -1, dtype=torch.int32, pin_memory=True)
        bm_host = torch.empty((B, W), dtype=torch.int32, pin_memory=True)
        picked_host = torch.empty((B,), dtype=torch.int32, pin_memory=True)
        tok_dev = torch.empty(B, dtype=torch.int32, device=dev)
        picked_dev = torch.empty(B, dtype=torch.int32, device=dev)
        Ke = max(10, min(K, 200))

        def e2e_step(i):
            tok_dev.copy_(tok_host, non_blocking=True)                 # H2D: last step's tokens
            batch.accept(tok_dev, restart=True)                        # accept_token
            batch.fill(bm, logits[i % R], counts)                      # fill + -inf logits
            batch.sample_stream(bm, counts, seed, picked_dev)          # sampler (device)
            bm_host.copy_(bm, non_blocking=True)                       # D2H: the bitmask
            picked_host.copy_(picked_dev, non_blocking=True)           # D2H: sampled ids
            stream.synchronize()
            tok_host.copy_(picked_host)

        for i in range(3):
            e2e_step(i)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(Ke):
            e2e_step(i)
        t_e2e = time.perf_counter() - t0
        batch.check()
        (t_e2e,) = max_over_ranks([t_e2e], dev, world)
        e2e = {"value": aggregate_rate(world, B * Ke, t_e2e), "unit": UNIT, "h2d_bytes_per_step": B * 4,
               "d2h_bytes_per_step": B * W * 4 + B * 4, "steps": Ke,
               "path": "gm_accept_tokens(H2D ids) → gm_fill_and_mask_logits → gm_sample_stream → D2H bitmask+ids"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src, peaks_json = peaks()
    alg_bytes_seq = 2 * V1 + 8 * W          # write-only -inf formulation
    achieved = B * alg_bytes_seq / (fill_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            entry = json.load(open(tpath)).get(f"{args.grammar}:{args.vocab}:{B}")
            traffic = entry["dram_bytes_per_launch"] if entry else None
        except Exception:
            traffic = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        st, kind, cores, bcpu, steps_cpu = calibrated_cpu_sample(flat, vocab, eng.structural, args.seed,
                                                                 args.stack_cap, args.cpu_seconds)
        cpu = {"value": st[1] / st[0], "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{bcpu} sequences x {steps_cpu} steps of the same workload ({st[0]:.1f} s), "
                         f"threads={cores}, per seq-step ComputeMask + bf16 -inf row + stream sample + Step"}

    info = eng.info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (seeded token-level JSON streams, random bf16 logits)",
        "config": dict(workload_config(args, world),
                       l2=f"rotating {R} logits buffers of {row_bytes / 2**20:.0f} MiB (> 126 MB L2)"),
        "mask_latency_us": 1e3 * fill_ms,
        "step_breakdown_us": {("decode_step_kernel" if args.fused else "fill_kernel"): 1e3 * fill_ms, "host_enqueue_per_step": 1e3 * host_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": "FillKernel (whole fused step)" if args.fused else "FillKernel + AcceptKernel (one step)",
                     "alg_bytes_per_seq_step": alg_bytes_seq,
                     "device_counted_logit_bytes_per_seq_step": (fstats["logit_bytes_read"] +
                                                                 fstats["logit_bytes_written"]) / B},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": K * (1 if args.fused else 2),
        "clocks": clocks.summary(),
        "preprocessing": {"prewarm_s": t_pre, "prewarm": f"{args.prewarm_steps} steps x {args.prewarm_batch} seqs "
                          f"(seed differs from the timed streams)", "contexts_after_prewarm": pre_info["context_slots_used"]},
        "cache": {"contexts": info["context_slots_used"], "segment_builds": info["segment_builds"],
                  "private_builds": info["private_builds"], "last_fill": fstats},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
