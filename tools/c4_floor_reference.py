"""Pins C4's optimum with the UNMODIFIED reference (oracle/_ref): the thread pool
solve_parallel seeded with an external size floor of 16 (SolveConfig::shared_bound,
proj/src/solve.hpp:70-81; consumed at proj/src/engine_parallel.cpp:75-83).
Status optimal with floor 16 proves that no common subgraph of size 17 exists;
the reference's own oracle::verify (proj/src/oracle.cpp) then checks a size-16
mapping found by the GPU (written by tools/c4_floor.py / the golden test), so
C4 = 16 rests on the reference alone. Long-running (hours on the dev box):
writes tests/golden/c4.json. Dev tool, imports the oracle only as the checker."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import oracle as O  # noqa: E402

floor = int(sys.argv[1]) if len(sys.argv) > 1 else 16
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 0
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 6 * 3600.0
g = O.ref_random_graph(45, 0.5, 45000)
h = O.ref_random_graph(45, 0.5, 45001)
t = time.time()
r = O.ref_solve_parallel_floor(g, h, floor, workers=workers, part_level=5, budget=budget)
out = {"config": "C4 ER n=45 p=0.5 seeds 45000/45001 (BASELINE.json configs[3])",
       "engine": "reference mcs::solve_parallel (oracle/_ref), SolveConfig::shared_bound seeded at floor",
       "floor": floor, "workers": workers or os.cpu_count(), "cores": os.cpu_count(),
       "status": {0: "optimal", 1: "timeout", 2: "cancelled"}.get(r.status, r.status),
       "size_above_floor": r.size, "nodes": r.nodes, "wall_s": round(time.time() - t, 1),
       "pairs": r.pairs}
print(json.dumps({k: v for k, v in out.items() if k != "pairs"}), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/c4_floor{floor}_reference.json", "w"))
