#!/usr/bin/env python3
"""bench.py — B200 McSplit on BASELINE.json's configs[1] (C2), plus every other
BASELINE config as side measurements.

Headline step = solve one batch of 100 Erdős–Rényi pairs (n = 30,
p ∈ {0.1, 0.3, 0.5}, the SURVEY §8(d) seeds) to PROVEN optimality in one
persistent launch of the sm_100a search kernel (throughput mode: every
resident warp, subtree donation).

Reported (one JSON line on rank 0):
  value   search nodes/s of the whole job, device-timed (CUDA events on the
          launching stream around the search kernel; inputs resident in HBM)
  e2e     the same metric through the public C-ABI call with HOST buffers
          (packing + H2D + kernel + D2H inside the timed region)
  time_to_optimum_s   device time to prove all 100 optima (per step, median)
  roofline            issue-rate roof; see DESIGN.md §4
  cpu_baseline        the reference's thread-pool solver (oracle/_ref, all host
                      threads) PROVING a fixed set of instances (C1 seeds and
                      C2 pairs) to optimality, with per-instance CPU/GPU
                      time-to-optimum ratios on the identical instances
  configs             C1 (5 seeds), C3 (90 pairs), C4 (sharded over the job's
                      GPUs, and a portfolio across them), C5 (10,000 pairs
                      sharded over the ranks): time to proven optimum and
                      nodes/s, optima checked against the reference goldens

Multi-GPU: ``--gpus N`` runs N ranks, one per GPU: under torchrun as the
driver launches it, or by re-launching itself under torch.distributed.run
when WORLD_SIZE is unset. Headline: weak scaling — rank r solves its own
100-pair shard (pair indices [100 r, 100 r + 100)); no data-path collective;
time = max over ranks. C5 is strong scaling (10,000 pairs split over the
ranks); C4 is ONE instance sharded over all N devices from rank 0 with the
incumbent pushed peer-to-peer over NVLink (mcsg n_devices = N).

``--impl reference`` times the reference's own CPU implementation (the
unmodified solver compiled from /root/reference into oracle/_ref) on rank 0:
each step PROVES one instance of a fixed list of C2 pairs to optimality on
every host thread (solve_parallel), so its nodes/s and time-to-optimum come
from complete proofs of instances the GPU arm also solves.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PAIRS = 100
N_VERT = 30
DENSITIES = (0.1, 0.3, 0.5)
METRIC = "search nodes/s (C2 batch solved to proven optimum)"
UNIT = "nodes/s"
WORKLOAD = ("C2: batch of 100 Erdos-Renyi pairs n=30, p in {0.1,0.3,0.5}, unlabelled undirected, "
            "induced MCS to proven optimum (BASELINE.json configs[1]; seeds SURVEY 8(d))")
# Instances the reference arm proves, one per step (rotating): C2 pairs 1 and
# 2 (p = 0.3 / 0.5, the hard cells: ~10 s each on 8 host threads) and the 34
# p = 0.1 pairs (0.2-1.3 s each).
REF_SET = [1, 2] + list(range(0, N_PAIRS, 3))
# cpu_baseline sample (rank 0, N = 1): the five C1 seed pairs and twelve C2
# p = 0.1 pairs, each proven to optimality by the reference pool (~10-20 s).
CPU_SAMPLE = [("C1", s) for s in (1, 3, 5, 7, 9)] + [("C2", i) for i in range(0, 36, 3)]


def c2_pair_seeds(index: int):
    """SURVEY §8(d) C2 generator: k = i%3, p = {.1,.3,.5}[k], j = i//3,
    G seed 30000 + 1000 k + 2 j, H seed = G seed + 1 (extended past i = 99 for shards)."""
    k = index % 3
    j = index // 3
    s = 30000 + 1000 * k + 2 * j
    return N_VERT, DENSITIES[k], s, s + 1


def instance_seeds(kind: str, idx: int):
    """(n, p, G seed, H seed, directed, labels) of a BASELINE config instance
    (SURVEY §8(d)): C1 seed pairs, C2 / C3 / C4 / C5 by index."""
    if kind == "C1":
        return 20, 0.3, idx, idx + 1, False, 0
    if kind == "C2":
        n, p, sg, sh = c2_pair_seeds(idx)
        return n, p, sg, sh, False, 0
    if kind == "C3":  # L in {2,4,8} x p in {.1,.3,.5} x 10, directed + labelled, n = 40
        L = (2, 4, 8)[idx // 30]
        p = DENSITIES[(idx // 10) % 3]
        return 40, p, 40000 + 2 * idx, 40001 + 2 * idx, True, L
    if kind == "C4":
        return 45, 0.5, 45000 + 2 * idx, 45001 + 2 * idx, False, 0
    if kind == "C5":
        return 16 + (idx // 3) % 9, DENSITIES[idx % 3], 50000 + 2 * idx, 50001 + 2 * idx, False, 0
    raise ValueError(kind)


def shard(rank: int, world: int, per_rank: int = N_PAIRS):
    """Weak scaling: rank r owns pair indices [r*per_rank, (r+1)*per_rank)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def split(total: int, rank: int, world: int):
    """Strong scaling: rank r owns the r-th contiguous slice of range(total)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return list(range(lo, hi))


def bench_config(world: int, pairs_per_gpu: int = N_PAIRS):
    """The config dict both arms print (the driver compares them)."""
    return {"workload": WORKLOAD, "pairs_per_gpu": pairs_per_gpu, "n": N_VERT,
            "mode": "throughput (all resident warps, subtree donation)",
            "l2": "flushed between steps (256 MiB device write, outside the timed kernel)",
            "parallelism": f"dp{world} (weak: one 100-pair shard per GPU)"}


def golden(name: str):
    path = os.path.join(ROOT, "tests", "golden", name)
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.dev)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[4:]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r[2] >= 50] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for name, val in zip(names, r[3][1:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(loaded)}


# ------------------------------------------------------------ CPU baseline --
def _ref_graphs(O, kind, idx):
    n, p, sg, sh, directed, labels = instance_seeds(kind, idx)
    if O.ref_available():
        return O.ref_random_graph(n, p, sg, directed, labels), O.ref_random_graph(n, p, sh, directed, labels)
    return O.random_graph(n, p, sg, directed, labels), O.random_graph(n, p, sh, directed, labels)


def cpu_prove(kind: str, idx: int, budget_s: float):
    """The reference thread-pool engine (solve_parallel, workers = all host
    threads, part_level 5: engine_parallel.cpp:20-21) proving one instance;
    the C oracle port (one thread) when oracle/_ref was not built."""
    import oracle as O
    g, h = _ref_graphs(O, kind, idx)
    t0 = time.perf_counter()
    if O.ref_available():
        r = O.ref_solve_parallel(g, h, workers=0, part_level=5, budget=budget_s)
    else:
        r = O.solve(g, h, budget=budget_s)
    secs = time.perf_counter() - t0
    return {"instance": f"{kind}[{idx}]", "status": "optimal" if r.status == 0 else "timeout",
            "size": r.size, "nodes": r.nodes, "seconds": secs}


def cpu_kind():
    import oracle as O
    if O.ref_available():
        return "reference", O.ref_lib().ref_hardware_concurrency()
    return "port", 1


def run_reference(args, rank, world):
    """The reference arm: rank 0 proves REF_SET instances, one per step."""
    if rank != 0:
        return 0
    kind, cores = cpu_kind()
    recs = []
    todo = [("C2", i) for i in REF_SET] if args.ref_set == "c2" else [("C1", s) for s in (1, 3, 5, 7, 9)]
    for it in range(args.warmup + args.steps):
        r = cpu_prove(*todo[it % len(todo)], args.ref_budget)
        if it >= args.warmup:
            recs.append(r)
    nodes = sum(r["nodes"] for r in recs)
    secs = sum(r["seconds"] for r in recs)
    value = nodes / max(secs, 1e-9)
    proven = sum(r["status"] == "optimal" for r in recs)
    sample = (f"steps prove {[r['instance'] for r in recs]} to optimality, one per step, "
              f"solve_parallel on {cores} host threads ({proven}/{len(recs)} proven within "
              f"{args.ref_budget:g} s each)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded random_graph, bit-identical to the reference generator)",
        "config": bench_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_optimum_per_instance_s": {r["instance"]: round(r["seconds"], 4) for r in recs},
        "all_optimal": proven == len(recs),
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- ours --
def _load_profile_summary():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def _measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


def _gpu_pair(M, kind, idx):
    n, p, sg, sh, directed, labels = instance_seeds(kind, idx)
    return M.random_graph(n, p, sg, directed, labels), M.random_graph(n, p, sh, directed, labels)


def cpu_vs_gpu(M, device, budget_s):
    """cpu_baseline: the reference pool proves CPU_SAMPLE instance by instance;
    the GPU proves the same instances one solve call each (every warp on one
    instance): per-instance time-to-optimum ratios on identical instances."""
    kind, cores = cpu_kind()
    rows = []
    for k, i in CPU_SAMPLE:
        c = cpu_prove(k, i, budget_s)
        g, h = _gpu_pair(M, k, i)
        t0 = time.perf_counter()
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device))
        wall = time.perf_counter() - t0
        ok = r.status == M.SolveStatus.optimal and (c["status"] != "optimal" or r.size == c["size"])
        rows.append({**c, "gpu_s": r.stats.kernel_seconds, "gpu_wall_s": wall, "gpu_size": r.size,
                     "gpu_nodes": r.stats.recursions, "sizes_equal": ok})
    nodes = sum(r["nodes"] for r in rows)
    secs = sum(r["seconds"] for r in rows)
    proven = [r for r in rows if r["status"] == "optimal"]
    ratio = [r["seconds"] / max(r["gpu_s"], 1e-9) for r in proven]
    ratio_e2e = [r["seconds"] / max(r["gpu_wall_s"], 1e-9) for r in proven]
    return {
        "value": nodes / max(secs, 1e-9), "unit": UNIT, "cores": cores, "kind": kind,
        "sample": (f"{len(rows)} instances proven to optimality one after another by solve_parallel "
                   f"(all {cores} host threads): C1 seeds 1,3,5,7,9 and C2 p=0.1 pairs "
                   f"{[i for k, i in CPU_SAMPLE if k == 'C2']}; {nodes} nodes in {secs:.2f} s"),
        "time_to_optimum_cpu_s": round(secs, 4),
        "time_to_optimum_gpu_s": round(sum(r["gpu_s"] for r in rows), 6),
        "time_to_optimum_gpu_e2e_s": round(sum(r["gpu_wall_s"] for r in rows), 6),
        "per_instance_cpu_over_gpu": {"median": statistics.median(ratio) if ratio else None,
                                      "min": min(ratio) if ratio else None, "max": max(ratio) if ratio else None,
                                      "median_e2e": statistics.median(ratio_e2e) if ratio_e2e else None},
        "sizes_equal": all(r["sizes_equal"] for r in rows),
        "per_instance": [{k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()} for r in rows],
    }


def side_configs(M, args, rank, world, ndev, device, barrier, max_over_ranks, sum_over_ranks):
    """Every other BASELINE config, outside the timed region: time to the
    proven optimum, nodes/s, and the optimum checked against the reference."""
    out = {}
    thr = M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device)
    small = golden("small.json")
    if rank == 0 and "c1" in args.configs:
        gold = {r["seed"]: r["size"] for r in small["config1"]} if small else {}
        rows = []
        for s in (1, 3, 5, 7, 9):
            g, h = _gpu_pair(M, "C1", s)
            r = M.solve(g, h, thr)
            rows.append({"seed": s, "size": r.size, "time_to_optimum_s": r.stats.kernel_seconds,
                         "nodes": r.stats.recursions, "optimal": r.status == M.SolveStatus.optimal,
                         "golden_ok": gold.get(s) == r.size if gold else None})
        out["C1"] = {"config": "ER n=20 p=0.3 seed pairs (1,2)..(9,10), one solve each (BASELINE configs[0])",
                     "instances": rows}
    if rank == 0 and "c3" in args.configs:
        pairs = [_gpu_pair(M, "C3", i) for i in range(90)]
        res, st = M.solve_batch(pairs, thr)
        gold = golden("c3_sizes.json")
        ok = None
        if gold:
            ok = all(r.size == gd["size"] and r.status == M.SolveStatus.optimal
                     for r, gd in zip(res, gold["pairs"]))
        out["C3"] = {"config": "90 directed vertex-labelled ER pairs n=40, L in {2,4,8} x p in {.1,.3,.5} "
                               "(BASELINE configs[2]), one launch",
                     "time_to_optimum_s": st.kernel_seconds, "nodes": st.recursions,
                     "nodes_per_s": st.recursions / max(st.kernel_seconds, 1e-9),
                     "all_optimal": all(r.status == M.SolveStatus.optimal for r in res), "golden_sizes_ok": ok,
                     "reference_pool_seconds_total": round(sum(p["pool_seconds"] for p in gold["pairs"]), 1)
                     if gold else None}
    if "c5" in args.configs:
        idx = split(10000, rank, world)
        pairs = [_gpu_pair(M, "C5", i) for i in idx]
        barrier()
        res, st = M.solve_batch(pairs, thr)
        gold = golden("c5_sizes.json")
        ok = True
        if gold:
            sz = gold["sizes"]
            ok = all(r.size == ord(sz[i]) - ord("A") for i, r in zip(idx, res))
        else:
            gs = golden("c5_sample.json")
            ref = {p["i"]: p["size"] for p in gs["pairs"]} if gs else {}
            ok = all(r.size == ref[i] for i, r in zip(idx, res) if i in ref)
        ok &= all(r.status == M.SolveStatus.optimal for r in res)
        t = max_over_ranks(st.kernel_seconds)
        nodes = sum_over_ranks(float(st.recursions))
        oks = sum_over_ranks(1.0 if ok else 0.0)
        out["C5"] = {"config": "10,000 ER pairs n=16..24 (BASELINE configs[4]), strong scaling: "
                               f"{len(idx)} pairs per rank, one launch per GPU",
                     "n_gpus": world, "time_to_optimum_s": t, "nodes": nodes, "nodes_per_s": nodes / max(t, 1e-9),
                     "golden_sizes_ok": oks == world,
                     "golden": "c5_sizes.json (all 10,000, reference)" if gold else "c5_sample.json (300, reference)"}
    if "c4" in args.configs:
        proof = golden("c4_proof.json")
        opt = proof["optimum"] if proof else None
        barrier()
        if rank == 0:
            g, h = _gpu_pair(M, "C4", 0)
            devs = tuple(i % ndev for i in range(world)) if world > 1 else ()  # (shared only in test runs)
            cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device, devices=devs, budget_seconds=300)
            t0 = time.perf_counter()
            r = M.solve(g, h, cfg)
            wall = time.perf_counter() - t0
            out["C4"] = {"config": "ER n=45 p=0.5 seeds 45000/45001 (BASELINE configs[3]), ONE instance "
                                   + (f"sharded over {world} GPUs (host frontier, P2P incumbent)" if world > 1
                                      else "on one GPU (every warp)"),
                         "n_gpus": world, "status": r.status.name, "size": r.size,
                         "time_to_optimum_s": r.stats.kernel_seconds, "wall_s": wall,
                         "nodes": r.stats.recursions,
                         "nodes_per_s": r.stats.recursions / max(r.stats.kernel_seconds, 1e-9),
                         "peer_pushes": r.stats.peer_pushes,
                         "mapping_verified": bool(M.verify(g, h, r.best)),
                         "golden_ok": (r.size == opt) if opt is not None else None,
                         "golden": "c4_proof.json (reference solve() with a size floor on each of the 541 pieces of a "
                                   "decomposition of its tree: no 17; GPU 16-mapping "
                                   "accepted by the reference verify)" if proof else None}
            # one member per GPU (two on one GPU): orderings race in one launch
            # spread over their GPUs; restarts / dead-end members are engines
            # of their own; sizes are shared between all (share_incumbent)
            members = ["gpu", "gpu+order=degree", "restarts:1", "jump:plus1+deadend=rel:4",
                       "gpu+order=components", "restarts:2", "gpu+order=block", "restarts:3"][:max(world, 2)]
            t0 = time.perf_counter()
            pr = M.run_portfolio(g, h, members, M.SolveConfig(device=device, devices=devs),
                                 M.PortfolioConfig(budget_seconds=300, share_incumbent=True))
            wall = time.perf_counter() - t0
            out["C4_portfolio"] = {"members": members, "n_gpus": world, "status": pr.status.name,
                                   "winner": pr.winner, "size": pr.size,
                                   "engines": [{"spec": e.spec_name, "outcome": e.outcome, "size": e.size,
                                                "wall_s": round(e.wall_seconds, 4)} for e in pr.engines],
                                   "time_to_optimum_s": pr.stats.kernel_seconds, "wall_s": wall,
                                   "nodes": pr.stats.recursions,
                                   "golden_ok": (pr.size == opt) if opt is not None else None}
        barrier()
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1908_06418_b200 as M  # raises when libmcsg.so is missing: no fallback

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the solver has no CPU path)")
    ndev = torch.cuda.device_count()
    if world > ndev and not args.allow_shared_gpus:
        raise SystemExit(f"bench.py: {world} ranks but only {ndev} visible GPU(s); one rank per GPU "
                         "(--allow-shared-gpus for a test run that stacks ranks on one GPU)")
    device = local_rank % ndev
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # No data-path collective: only barriers and the max/sum of timings.
        # NCCL when every rank owns a GPU; gloo when ranks share one (test runs).
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group("gloo")

    red_dev = "cuda" if (dist is not None and dist.get_backend() == "nccl") else "cpu"
    # host-side barriers for the side measurements: while rank 0 drives every
    # GPU (C4 sharded), the other ranks must not park an NCCL kernel on them
    cpu_group = dist.new_group(backend="gloo") if dist is not None else None

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def cpu_barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(group=cpu_group)

    def reduce(x: float, op) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        return reduce(x, dist.ReduceOp.MAX) if dist is not None else x

    def sum_over_ranks(x: float) -> float:
        return reduce(x, dist.ReduceOp.SUM) if dist is not None else x

    idx = shard(rank, world, args.pairs)
    pairs = []
    for i in idx:
        n, p, sg, sh = c2_pair_seeds(i)
        pairs.append((M.random_graph(n, p, sg), M.random_graph(n, p, sh)))
    cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        res, st = M.solve_batch(pairs, cfg)
        return res, st

    for _ in range(args.warmup):
        step()
    sizes_ref = None
    kernel_s, wall_s, nodes, ttos = 0.0, 0.0, 0, []
    per_inst = []  # time from launch to each instance's proof (device clock), every step
    h2d = d2h = launches = 0
    all_optimal = True
    st = None
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    barrier()
    if sampler:
        sampler.start()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, st = step()
        wall_s += time.perf_counter() - t0
        kernel_s += st.kernel_seconds
        nodes += st.recursions
        ttos.append(max(r.stats.solve_seconds for r in res))
        per_inst.extend(r.stats.solve_seconds for r in res)
        h2d, d2h = st.h2d_bytes, st.d2h_bytes
        launches += st.launches
        sizes = [r.size for r in res]
        all_optimal &= all(r.status == M.SolveStatus.optimal for r in res)
        if sizes_ref is None:
            sizes_ref = sizes
        elif sizes != sizes_ref:
            raise SystemExit("bench.py: optimum sizes changed between steps (correctness failure)")
    barrier()
    clocks = sampler.stop() if sampler else None

    # cross-check sizes against the golden fixture for the pairs it covers
    golden_ok = None
    gold = golden("c2_sizes.json")
    if gold:
        g2 = {int(k): v for k, v in gold["sizes"].items()}
        checked = [(i, s) for i, s in zip(idx, sizes_ref) if i in g2]
        golden_ok = all(g2[i] == s for i, s in checked) if checked else None

    t_dev = max_over_ranks(kernel_s)
    t_e2e = max_over_ranks(wall_s)
    total_nodes = sum_over_ranks(float(nodes))

    # ---- outside the timed region: the other configs and the CPU baseline
    configs = side_configs(M, args, rank, world, ndev, device, cpu_barrier, max_over_ranks, sum_over_ranks)
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_baseline = cpu_vs_gpu(M, device, args.cpu_budget)
        except Exception as e:  # the baseline is reported, never required
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                            "sample": f"{type(e).__name__}: {e}"}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    value = total_nodes / t_dev
    e2e = total_nodes / t_e2e
    prof = _load_profile_summary()
    peaks = _measured_peaks()
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    sms = props.multi_processor_count
    clk_mhz = float(peaks.get("sm_max_mhz") or 1965.0)
    peak_issue = sms * 4 * clk_mhz * 1e6  # warp-instructions / s (4 schedulers per SM)
    inst_per_node = prof.get("warp_inst_per_node")
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from sass_key import kernel_sass_sha1
    sass = kernel_sass_sha1(M.LIB_PATH, prof.get("kernel", "")) if prof.get("kernel") else None
    profile_current = sass is not None and prof.get("kernel_sass_sha1") == sass
    roofline = {
        "bound": "issue",
        "achieved": (value / world) * inst_per_node if inst_per_node else None,
        "peak": peak_issue, "unit": "warp-inst/s",
        "frac": ((value / world) * inst_per_node / peak_issue) if inst_per_node else None,
        "traffic": prof.get("dram_bytes_per_launch"),
        "profile_matches_kernel": profile_current,  # False: profiles/ measured other machine code
        "basis": (f"issue roof = {sms} SMs x 4 schedulers x {clk_mhz:g} MHz (sm_max_mhz, "
                  f"MEASURED_PEAKS.json); per-node cost {inst_per_node} warp-instructions from "
                  f"profiles/ncu_summary.json (its kernel's SASS hash is checked against the built "
                  f"library); neither HBM nor tensor cores bind (SURVEY 8(d))"),
    }
    # the other two views of SURVEY 8(d): the algorithmic op count per node
    # (20 + 14 S, S measured by the C oracle on C2) against the same issue roof,
    # and shared-memory bytes per node (the GPU's own, measured with the
    # diagnostic counters build; the algorithmic model's) against the smem roof
    smem_peak = sms * 128 * clk_mhz * 1e6  # B/s: 128 B per SM per clock
    trf = {}
    tpath = os.path.join(ROOT, "profiles", "r2_smem_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            trf = json.load(f)
    alg = trf.get("alg", {})
    gsm = trf.get("gpu", {})
    per_gpu = value / world
    roofline["algorithmic_issue"] = {
        "ops_per_node": alg.get("ops_per_node"),
        "frac": per_gpu * alg["ops_per_node"] / peak_issue if alg.get("ops_per_node") else None,
        "basis": "SURVEY 8(d) ops = 20 + 14 S per node, S (parent classes re-read per refinement) measured "
                 "by the C oracle on C2 (profiles/r2_smem_traffic.json)"}
    roofline["smem"] = {
        "peak": smem_peak, "unit": "B/s",
        "gpu_bytes_per_node": gsm.get("bytes_per_node"),
        "gpu_frac": per_gpu * gsm["bytes_per_node"] / smem_peak if gsm.get("bytes_per_node") else None,
        "alg_bytes_per_node": alg.get("bytes_per_node"),
        "alg_frac": per_gpu * alg["bytes_per_node"] / smem_peak if alg.get("bytes_per_node") else None,
        "basis": "smem roof = SMs x 128 B/clk x sm_max_mhz; GPU bytes/node from the class-traffic counters "
                 "(diagnostic build, profiles/r2_smem_traffic.json), algorithmic B = 32 C + 16 S + 16"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded random_graph, bit-identical to the reference generator)",
        "config": bench_config(world, len(idx)),
        "time_to_optimum_s": statistics.median(ttos),
        "time_to_optimum_per_instance_s": {
            "median": statistics.median(per_inst),
            "p90": sorted(per_inst)[int(0.9 * (len(per_inst) - 1))],
            "max": max(per_inst),
            "note": "rank 0's instances; device time from kernel start to the instance's proof"},
        "all_optimal": all_optimal, "golden_sizes_ok": golden_ok,
        "nodes_per_step": nodes / args.steps,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "seconds_per_step": t_e2e / args.steps},
        "gpu_launches": launches,
        "roofline": roofline,
        "configs": configs,
        "cpu_baseline": cpu_baseline,
        "clocks": clocks,
        "kernel": {"warps": st.warps, "ctas": st.ctas, "smem_per_cta": st.smem_per_cta,
                   "donations_per_step": st.donations},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(argv, n: int) -> int:
    """`--gpus N` without an outside launcher: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--pairs", type=int, default=N_PAIRS, help="pairs per GPU (default 100 = C2)")
    ap.add_argument("--cpu-budget", type=float, default=120.0, help="per-instance budget of the cpu_baseline proofs")
    ap.add_argument("--ref-budget", type=float, default=120.0, help="per-step budget of --impl reference")
    ap.add_argument("--ref-set", choices=("c2", "c1"), default="c2",
                    help="--impl reference: instances proven per step (c1 = the fast C1 seeds, for tests)")
    ap.add_argument("--configs", default="c1,c3,c4,c5", help="side measurements (comma list; '' = none)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 side measurements")
    ap.add_argument("--allow-shared-gpus", action="store_true",
                    help="test runs only: let more ranks than GPUs share devices")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    args.configs = {c for c in args.configs.split(",") if c}
    if args.no_c4:
        args.configs.discard("c4")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(argv, args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: one rank per GPU")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
