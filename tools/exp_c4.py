import sys, json, time
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=120))
print(json.dumps({"lib": M.LIB_PATH, "c4_size": r.size, "status": r.status.name, "kernel_s": r.stats.kernel_seconds, "nodes": r.stats.recursions, "rate": r.stats.recursions / r.stats.kernel_seconds, "warps": r.stats.warps}), flush=True)
