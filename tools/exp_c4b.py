import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=float(sys.argv[1])))
print(json.dumps({"nodes": r.stats.recursions, "s": r.stats.kernel_seconds, "rate": r.stats.recursions / r.stats.kernel_seconds / 1e9}), flush=True)
