import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
for fl in (0, 14, 15):
    r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, shared_bound=fl, budget_seconds=60))
    print(json.dumps({"floor": fl, "size": r.size, "status": r.status.name, "s": round(r.stats.kernel_seconds, 3), "nodes": r.stats.recursions}), flush=True)
# goal probe 17 (prove no 17)
r = M.solve_goal_directed(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT))
print(json.dumps({"goal_directed": r.size, "probes": r.stats.probes, "nodes": r.stats.recursions, "s": round(r.stats.kernel_seconds, 3)}))
