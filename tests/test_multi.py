"""The N>1 path on CPU: world_size-2 gloo process groups exercise bench.py's
max-over-ranks timing and aggregate rate, and torchrun launches of the
reference arm print exactly one JSON line (rank 0) and exit 0 elsewhere.
Sequences shard across ranks with no collective on the hot path,
so the timing reduction is the only cross-rank exchange."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # Rank r "took" 10 + r ms for its 256 sequences x 100 steps.
    elapsed_ms, other = bench.max_over_ranks([10.0 + rank, 1.0 * rank], torch.device("cpu"), world)
    rate = bench.aggregate_rate(world, 256 * 100, elapsed_ms / 1e3)
    out[rank] = (elapsed_ms, other, rate)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        elapsed_ms, other, rate = out[r]
        assert elapsed_ms == 11.0 and other == 1.0
        assert abs(rate - 2 * 256 * 100 / 0.011) < 1e-6


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgmask_ref.so")),
                    reason="reference oracle not built")
def test_reference_arm_under_torchrun_prints_once():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--vocab", "4000", "--config", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["check"]["sequences"] == 32 and d["check"]["popcount_sum"] > 0


def test_bench_config_defaults():
    """bench.py's per-config settings: context depth, parent
    depth, table size, prewarm; the default run is config 3 (the largest
    single-GPU BASELINE config, batch 1024) on one GPU."""
    import bench
    a = bench.parse([])
    assert (a.config, a.context_depth, a.context_slots, a.mode) == (3, 16, 16384, "stream")
    assert bench.per_gpu_batch(a, 1) == 1024
    a = bench.parse(["--config", "2"])
    assert (a.config, a.context_depth, a.context_slots, a.prewarm_steps, a.mode) == (2, 20, 65536, 10000, "stream")
    a = bench.parse(["--config", "4"])
    assert (a.context_depth, a.parent_depth, a.context_slots, a.prewarm_steps) == (20, 6, 262144, 30000)
    a = bench.parse(["--config", "5"])
    assert (a.mode, a.context_depth) == ("greedy", 12)
    a = bench.parse(["--config", "3", "--context-depth", "12"])
    assert a.context_depth == 12 and a.fill_samples >= 10


def _shard_worker(rank, world, port, out):
    """One rank of a sharded decode loop (bench.py's layout: rank r owns its
    own batch with streams seeded rank_seed(seed, r)); the CPU port stands in
    for the GPU.  Seq-steps, restarts and the token digests are reduced with
    bench.sum_over_ranks, the step time with bench.max_over_ranks."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = bench.parse(["--config", "4", "--vocab", "3000"])
    B = bench.per_gpu_batch(a, world)  # strong scaling: the 4096 sequences split
    flat = bench.reference_automaton_bytes("json")
    vocab = oracle.synth_vocab(3000)
    st = oracle.structural_words(vocab)
    p = oracle.Port(flat, vocab)
    Bs, steps = 6, 10  # a shard sample (the port is slow)
    stats, toks, _ = p.decode_run(st, Bs, steps, bench.rank_seed(7, rank), want_tokens=True)
    dig = bench.token_digest(toks)
    tot = bench.sum_over_ranks([Bs * steps, int(stats[2]), dig], torch.device("cpu"), world)
    mx = bench.max_over_ranks([float(stats[0])], torch.device("cpu"), world)
    out[rank] = (B, dig, tot, mx)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_decode_reduces_counters_world2():
    """World-2 gloo: each rank decodes its own shard (no exchange on the hot
    path); the reductions bench.py performs give the totals one process
    computes over both shards."""
    import bench
    import oracle
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == 2048
    flat = bench.reference_automaton_bytes("json")
    vocab = oracle.synth_vocab(3000)
    p = oracle.Port(flat, vocab)
    st = oracle.structural_words(vocab)
    digs, restarts = [], 0
    for r in range(2):
        stats, toks, _ = p.decode_run(st, 6, 10, bench.rank_seed(7, r), want_tokens=True)
        digs.append(bench.token_digest(toks))
        restarts += int(stats[2])
        assert digs[r] == out[r][1]
    assert digs[0] != digs[1]  # the shards are different streams
    for r in range(2):
        assert out[r][2] == [120, restarts, digs[0] + digs[1]]
        assert out[r][3] == out[0][3]


def test_token_digest_and_summarize():
    """bench.token_digest == the C loops' FNV-1a (stats[5]) and summarize ==
    Summarize's rank rule (tools/gmask_main.cpp:135-149)."""
    import bench
    import oracle
    flat = bench.reference_automaton_bytes("json")
    vocab = oracle.synth_vocab(2000)
    p = oracle.Port(flat, vocab)
    st = oracle.structural_words(vocab)
    stats, toks, _ = p.decode_run(st, 40, 9, 3, want_tokens=True, warmup=4, digest_seqs=32)
    assert bench.token_digest(toks[:32, 4:]) == int(stats[5])
    s = bench.summarize([float(x) for x in range(1, 101)])
    assert (s["p50"], s["p99"], s["mean"]) == (50.0, 99.0, 50.5)
    s = bench.summarize([3.0])
    assert s["p50"] == s["p99"] == 3.0
