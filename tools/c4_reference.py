"""Pins C4's optimum with the unmodified reference (oracle/_ref, thread pool on
every host core): ER n=45 p=0.5, seeds 45000/45001 (BASELINE.json configs[3]).
Long-running; writes gpurun_out/c4_reference.json (dev tool)."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 4500.0
g = O.ref_random_graph(45, 0.5, 45000)
h = O.ref_random_graph(45, 0.5, 45001)
t = time.time()
r = O.ref_solve_parallel(g, h, workers=0, part_level=5, budget=budget)
out = {"config": "C4 ER n=45 p=0.5 seeds 45000/45001", "engine": "reference solve_parallel (all host threads)",
       "cores": os.cpu_count(), "status": ["optimal", "timeout", "cancelled"][r.status] if r.status in (0, 1, 2) else r.status,
       "size": r.size, "nodes": r.nodes, "wall_s": time.time() - t, "pairs": r.pairs}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c4_reference.json", "w"))
print(json.dumps({k: v for k, v in out.items() if k != "pairs"}))
