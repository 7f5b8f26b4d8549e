import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
for i in range(8):
    r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=60))
    print(json.dumps({"s": round(r.stats.kernel_seconds, 3), "nodes": r.stats.recursions, "gnps": round(r.stats.recursions / r.stats.kernel_seconds / 1e9, 3)}), flush=True)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=60, shared_bound=16))
print("floor16", json.dumps({"s": round(r.stats.kernel_seconds, 3), "nodes": r.stats.recursions, "size": r.size}))
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=60, shared_bound=15))
print("floor15", json.dumps({"s": round(r.stats.kernel_seconds, 3), "nodes": r.stats.recursions, "size": r.size}))
