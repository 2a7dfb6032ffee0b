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
           "--gpus", "2", "--steps", "1", "--warmup", "0", "--vocab", "4000"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


def test_bench_config_defaults():
    """bench.py's per-config settings: context depth, parent
    depth, table size, prewarm; the default run is config 2 on one GPU."""
    import bench
    a = bench.parse([])
    assert (a.config, a.context_depth, a.context_slots, a.prewarm_steps, a.mode) == (2, 20, 65536, 10000, "stream")
    a = bench.parse(["--config", "4"])
    assert (a.context_depth, a.parent_depth, a.context_slots, a.prewarm_steps) == (20, 6, 262144, 30000)
    a = bench.parse(["--config", "5"])
    assert (a.mode, a.context_depth) == ("greedy", 12)
    a = bench.parse(["--config", "3", "--context-depth", "12"])
    assert a.context_depth == 12 and a.sample_every == 16
