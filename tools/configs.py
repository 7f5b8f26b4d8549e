"""Runs BASELINE.json configs C1-C5 on one GPU and prints a JSON line per config.

C1 ER n=20 p=0.3 seeds (1,2),(3,4),(5,6),(7,8),(9,10)
C2 100 ER pairs n=30 (bench.py's workload)
C3 90 directed vertex-labelled pairs n=40: L in {2,4,8} x p in {.1,.3,.5} x 10, seeds 40000+2i / 40001+2i
C4 ER n=45 p=0.5 seeds 45000+2k / 45001+2k (hard; budgeted)
C5 10,000 ER pairs, n = 16 + (i/3)%9, p = {.1,.3,.5}[i%3], seeds 50000+2i / 50001+2i

"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import paper_1908_06418_b200 as M  # noqa: E402


def run_batch(name, pairs, cfg, extra=None):
    t = time.perf_counter()
    res, st = M.solve_batch(pairs, cfg)
    wall = time.perf_counter() - t
    line = {"config": name, "pairs": len(pairs), "optimal": sum(r.status == M.SolveStatus.optimal for r in res),
            "kernel_s": st.kernel_seconds, "wall_s": wall, "nodes": st.recursions,
            "nodes_per_s": st.recursions / max(st.kernel_seconds, 1e-9),
            "max_time_to_optimum_s": max(r.stats.solve_seconds for r in res),
            "busy_frac": st.busy_cycles / max(1, st.busy_cycles + st.idle_cycles),
            "warps": st.warps, "spills": st.spills, "sizes": [r.size for r in res][:12]}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c3,c4,c5")
    ap.add_argument("--c4-budget", type=float, default=120.0)
    ap.add_argument("--c4-count", type=int, default=1)
    ap.add_argument("--c5-count", type=int, default=10000)
    a = ap.parse_args()
    todo = a.only.split(",")
    thr = M.SolveConfig(mode=M.MODE_THROUGHPUT)
    if "c1" in todo:
        pairs = [(M.random_graph(20, 0.3, s), M.random_graph(20, 0.3, s + 1)) for s in (1, 3, 5, 7, 9)]
        for s, (g, h) in zip((1, 3, 5, 7, 9), pairs):
            r = M.solve(g, h, thr)
            p = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY))
            print(json.dumps({"config": "C1", "seed": s, "size": r.size, "throughput_kernel_s": r.stats.kernel_seconds,
                              "throughput_wall_s": r.stats.wall_seconds, "parity_nodes": p.stats.recursions,
                              "parity_kernel_s": p.stats.kernel_seconds}), flush=True)
        run_batch("C1-batch", pairs, thr)
    if "c3" in todo:
        pairs = []
        i = 0
        for L in (2, 4, 8):
            for p in (0.1, 0.3, 0.5):
                for _ in range(10):
                    pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L),
                                  M.random_graph(40, p, 40001 + 2 * i, True, L)))
                    i += 1
        run_batch("C3", pairs, thr)
    if "c4" in todo:
        for k in range(a.c4_count):
            g, h = M.random_graph(45, 0.5, 45000 + 2 * k), M.random_graph(45, 0.5, 45001 + 2 * k)
            r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=a.c4_budget))
            print(json.dumps({"config": "C4", "k": k, "status": r.status.name, "size": r.size,
                              "kernel_s": r.stats.kernel_seconds, "nodes": r.stats.recursions,
                              "nodes_per_s": r.stats.recursions / max(r.stats.kernel_seconds, 1e-9),
                              "spills": r.stats.spills, "warps": r.stats.warps}), flush=True)
    if "c5" in todo:
        pairs = []
        for i in range(a.c5_count):
            n = 16 + (i // 3) % 9
            p = (0.1, 0.3, 0.5)[i % 3]
            pairs.append((M.random_graph(n, p, 50000 + 2 * i), M.random_graph(n, p, 50001 + 2 * i)))
        run_batch("C5", pairs, thr)


if __name__ == "__main__":
    main()
