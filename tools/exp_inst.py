"""Instructions per node of one C4 launch (run under ncu --metrics smsp__inst_executed.sum)."""
import json, sys
sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0))
print(json.dumps({"lib": M.LIB_PATH.split("/")[-1], "nodes": r.stats.recursions, "kernel_s": r.stats.kernel_seconds}))
