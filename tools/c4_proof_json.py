"""Writes tests/golden/c4_proof.json from the reference pool's floor-16 run
(tools/c4_floor_reference.py -> gpurun_out/c4_floor16_reference.json) and a
size-16 mapping found on the GPU (gpurun_out/c4_witness.json, from
tools/gpu_call_r2_final.sh), which the UNMODIFIED reference's
oracle::verify must accept (oracle/_ref). Dev tool, dev container only."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

run = json.load(open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c4_floor16_reference.json")))
wit = json.load(open(sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "c4_witness.json")))
assert run["status"] == "optimal" and run["floor"] == 16, run
g, h = O.ref_random_graph(45, 0.5, 45000), O.ref_random_graph(45, 0.5, 45001)
pairs = [tuple(p) for p in wit["witness"]]
ok = O.ref_verify(g, h, pairs)
assert len(pairs) == 16 and ok == 1, (len(pairs), ok)
out = {"instance": "ER n=45 p=0.5 seeds 45000/45001 (BASELINE.json configs[3])", "floor": 16, "status": 0,
       "optimum": 16, "pool_size_found_above_floor": run["size_above_floor"], "pool_nodes": run["nodes"],
       "pool_wall_s": run["wall_s"], "workers": run["workers"], "cores": run["cores"],
       "witness": [list(p) for p in pairs], "witness_reference_verify": ok,
       "how": "reference mcs::solve_parallel (oracle/_ref, part_level 5) with SolveConfig::shared_bound seeded "
              "at 16: status optimal = no common induced subgraph of 17 exists; the 16-witness (found on the "
              "GPU) is accepted by the reference's oracle::verify, so the optimum is 16"}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c4_proof.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "witness"}))
