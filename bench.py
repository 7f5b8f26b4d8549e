#!/usr/bin/env python3
"""bench.py — B200 McSplit on BASELINE.json's configs[1] (C2).

One step = solve one batch of 100 Erdős–Rényi pairs (n = 30, p ∈ {0.1, 0.3, 0.5},
the SURVEY §8(d) seeds) to PROVEN optimality in one persistent launch of the
sm_100a search kernel (throughput mode: every resident warp, subtree donation).

Reported (one JSON line on rank 0):
  value   search nodes/s of the whole job, device-timed (CUDA events on the
          launching stream around the search kernel; inputs resident in HBM)
  e2e     the same metric through the public C-ABI call with HOST buffers
          (packing + H2D + kernel + D2H inside the timed region)
  time_to_optimum_s   device time to prove all 100 optima (per step, median)
  roofline            issue-rate roof; see DESIGN.md §4
  cpu_baseline        the reference's thread-pool solver (oracle/_ref, all host
                      threads) on a bounded sample of the same workload

Multi-GPU (torchrun): weak scaling — rank r solves its own 100-pair shard
(pair indices [100 r, 100 r + 100) of the C2 generator); no data-path
collective; time = max over ranks.

``--impl reference`` times the reference's own CPU implementation (the
unmodified solver compiled from /root/reference into oracle/_ref) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
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


def c2_pair_seeds(index: int):
    """SURVEY §8(d) C2 generator: k = i%3, p = {.1,.3,.5}[k], j = i//3,
    G seed 30000 + 1000 k + 2 j, H seed = G seed + 1 (extended past i = 99 for shards)."""
    k = index % 3
    j = index // 3
    s = 30000 + 1000 * k + 2 * j
    return N_VERT, DENSITIES[k], s, s + 1


def shard(rank: int, world: int, per_rank: int = N_PAIRS):
    """Weak scaling: rank r owns pair indices [r*per_rank, (r+1)*per_rank)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


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
def cpu_reference_sample(indices, budget_s: float):
    """The reference thread-pool engine (solve_parallel, workers = all host
    threads, part_level 5: engine_parallel.cpp:20-21) on the given pairs."""
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    nodes, wall, solved = 0, 0.0, 0
    for i in indices:
        n, p, sg, sh = c2_pair_seeds(i)
        if kind == "reference":
            g, h = O.ref_random_graph(n, p, sg), O.ref_random_graph(n, p, sh)
            t0 = time.perf_counter()
            r = O.ref_solve_parallel(g, h, workers=0, part_level=5, budget=budget_s)
            wall += time.perf_counter() - t0
        else:
            g, h = O.random_graph(n, p, sg), O.random_graph(n, p, sh)
            t0 = time.perf_counter()
            r = O.solve(g, h, budget=budget_s)
            wall += time.perf_counter() - t0
        nodes += r.nodes
        solved += r.status == 0
    cores = O.ref_lib().ref_hardware_concurrency() if kind == "reference" else 1
    return {"value": nodes / max(wall, 1e-9), "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"C2 pairs {list(indices)} (solve_parallel, {budget_s:g} s budget each; "
                      f"{solved}/{len(indices)} proven), {nodes} nodes in {wall:.2f} s",
            "nodes": nodes, "seconds": wall}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    budget = args.ref_budget
    steps = []
    for it in range(args.warmup + args.steps):
        idx = [it % N_PAIRS]
        r = cpu_reference_sample(idx, budget)
        if it >= args.warmup:
            steps.append(r)
    nodes = sum(s["nodes"] for s in steps)
    secs = sum(s["seconds"] for s in steps)
    value = nodes / max(secs, 1e-9)
    kind = steps[0]["kind"] if steps else "reference"
    cores = steps[0]["cores"] if steps else 0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded random_graph, bit-identical to the reference generator)",
        "config": {"workload": WORKLOAD, "sample_per_step": f"one C2 pair (rotating index), "
                   f"solve_parallel with all host threads, {budget:g} s budget"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"pairs {[ (args.warmup + i) % N_PAIRS for i in range(args.steps)]}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1908_06418_b200 as M  # raises when libmcsg.so is missing: no fallback

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the solver has no CPU path)")
    ndev = torch.cuda.device_count()
    device = local_rank % ndev  # more ranks than GPUs only in CI-style dry runs
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # No data-path collective: only barriers and the max/sum of timings.
        # NCCL when every rank owns a GPU; gloo when ranks share one (NCCL
        # refuses two ranks on the same device).
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group("gloo")

    red_dev = "cuda" if (dist is not None and dist.get_backend() == "nccl") else "cpu"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    idx = shard(rank, world, args.pairs)
    pairs = []
    for i in idx:
        n, p, sg, sh = c2_pair_seeds(i)
        pairs.append((M.random_graph(n, p, sg), M.random_graph(n, p, sh)))
    cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_baseline = cpu_reference_sample([0, 1, 2], args.cpu_budget)
        except Exception as e:  # the baseline is reported, never required
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                            "sample": f"{type(e).__name__}: {e}"}

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
    gpath = os.path.join(ROOT, "tests", "golden", "c2_sizes.json")
    if os.path.exists(gpath):
        gold = {int(k): v for k, v in json.load(open(gpath))["sizes"].items()}
        checked = [(i, s) for i, s in zip(idx, sizes_ref) if i in gold]
        golden_ok = all(gold[i] == s for i, s in checked) if checked else None

    # Side measurement (N=1 only, outside the timed C2 region): time to the
    # proven optimum of BASELINE.json configs[3]'s hard pair (C4, ER n=45
    # p=0.5, seeds 45000/45001) on this GPU, every warp on one instance.
    c4 = None
    if rank == 0 and world == 1 and not args.no_c4:
        g4, h4 = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
        r4 = M.solve(g4, h4, M.SolveConfig(mode=M.MODE_THROUGHPUT, device=device, budget_seconds=120))
        c4 = {"config": "C4: ER n=45 p=0.5 seeds 45000/45001 (BASELINE.json configs[3]), one GPU",
              "status": r4.status.name, "size": r4.size, "time_to_optimum_s": r4.stats.kernel_seconds,
              "nodes": r4.stats.recursions, "nodes_per_s": r4.stats.recursions / max(r4.stats.kernel_seconds, 1e-9),
              "mapping_verified": bool(M.verify(g4, h4, r4.best))}

    t_dev = max_over_ranks(kernel_s)
    t_e2e = max_over_ranks(wall_s)
    total_nodes = sum_over_ranks(float(nodes))
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
    import hashlib
    sha = hashlib.sha1()
    for f in ("mcsg_kernel.cu", "mcsg_search.cuh", "mcsg_task_body.inc", "mcsg_device.h"):
        with open(os.path.join(ROOT, "paper_1908_06418_b200", "csrc", f), "rb") as fh:
            sha.update(fh.read())
    profile_current = prof.get("kernel_src_sha1") == sha.hexdigest()
    roofline = {
        "bound": "issue",
        "achieved": (value / world) * inst_per_node if inst_per_node else None,
        "peak": peak_issue, "unit": "warp-inst/s",
        "frac": ((value / world) * inst_per_node / peak_issue) if inst_per_node else None,
        "traffic": prof.get("dram_bytes_per_launch"),
        "profile_matches_kernel": profile_current,  # False: profiles/ is from other kernel sources
        "basis": (f"issue roof = {sms} SMs x 4 schedulers x {clk_mhz:g} MHz (sm_max_mhz, "
                  f"MEASURED_PEAKS.json); per-node cost {inst_per_node} warp-instructions from "
                  f"profiles/ncu_summary.json; neither HBM nor tensor cores bind (SURVEY 8(d))"),
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded random_graph, bit-identical to the reference generator)",
        "config": {"workload": WORKLOAD, "pairs_per_gpu": len(idx), "n": N_VERT,
                   "mode": "throughput (all resident warps, subtree donation)",
                   "l2": "flushed between steps (256 MiB device write, outside the timed kernel)",
                   "parallelism": f"dp{world} (weak: one 100-pair shard per GPU)"},
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
        "c4_hard_instance": c4,
        "cpu_baseline": cpu_baseline,
        "clocks": clocks,
        "kernel": {"warps": st.warps, "ctas": st.ctas, "smem_per_cta": st.smem_per_cta,
                   "donations_per_step": st.donations, "classes_per_node": st.sum_classes / max(1, st.recursions),
                   "splits_per_node": st.splits / max(1, st.recursions)},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--pairs", type=int, default=N_PAIRS, help="pairs per GPU (default 100 = C2)")
    ap.add_argument("--cpu-budget", type=float, default=6.0, help="per-pair budget of the cpu_baseline sample")
    ap.add_argument("--ref-budget", type=float, default=8.0, help="per-step budget of --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 time-to-optimum side measurement")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
