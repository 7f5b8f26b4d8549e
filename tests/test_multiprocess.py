"""N>1 host logic on CPU: world_size-2 gloo groups (no GPU).

bench.py shards the C2 workload by rank (weak scaling: one 100-pair shard per
GPU, no data-path collective) and reduces timing as the max over ranks; these
tests run that logic in two real processes over gloo on 127.0.0.1.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = bench.shard(rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, idx)
    # timing reduction used by bench.py: max over ranks; node totals: sum
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(len(idx))], dtype=torch.float64)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    seeds = [bench.c2_pair_seeds(i) for i in idx]
    gathered_seeds = [None] * world
    dist.all_gather_object(gathered_seeds, seeds)
    if rank == 0:
        out.put((gathered, float(t.item()), float(n.item()), gathered_seeds))
    dist.barrier()
    dist.destroy_process_group()


def test_c2_generator_formula():
    # k=i%3, p={.1,.3,.5}[k], j=i//3, G seed 30000+1000k+2j, H = G+1
    assert bench.c2_pair_seeds(0) == (30, 0.1, 30000, 30001)
    assert bench.c2_pair_seeds(1) == (30, 0.3, 31000, 31001)  # the measured seed-31000 pair
    assert bench.c2_pair_seeds(5) == (30, 0.5, 32002, 32003)
    assert bench.c2_pair_seeds(99) == (30, 0.1, 30066, 30067)


def test_shard_single_rank_is_the_c2_batch():
    assert bench.shard(0, 1) == list(range(100))
    with pytest.raises(ValueError):
        bench.shard(2, 2)


def test_two_rank_gloo_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax, ntotal, seeds = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat = sorted(i for part in gathered for i in part)
    assert flat == list(range(200))                      # every pair exactly once
    assert set(gathered[0]).isdisjoint(gathered[1])
    assert tmax == 2.0 and ntotal == 200.0
    all_seeds = [s for part in seeds for s in part]
    assert len(set(all_seeds)) == 200                     # shards are distinct instances


def test_bench_gpus_n_spawns_n_ranks():
    """`bench.py --gpus 2` without an outside launcher re-runs itself under
    torch.distributed.run with two ranks; with the reference arm (CPU only,
    rank 0 measures) the line reports n_gpus 2 and the shared config dict."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3",
                          "--ref-set", "c1"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.bench_config(2)
    assert line["all_optimal"] and line["value"] > 0


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)


def test_strong_scaling_split_covers_every_pair_once():
    for world in (1, 2, 3, 8):
        parts = [bench.split(10000, r, world) for r in range(world)]
        flat = [i for p in parts for i in p]
        assert flat == list(range(10000))
