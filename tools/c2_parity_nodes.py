"""Sequential (reference-order) node counts of the 100 C2 pairs via parity mode."""
import json, sys
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
pairs = []
for i in range(100):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_PARITY, budget_seconds=float(sys.argv[1]) if len(sys.argv) > 1 else 300))
out = {"status": [int(r.status) for r in res], "size": [r.size for r in res], "nodes": [r.stats.recursions for r in res],
       "solve_s": [r.stats.solve_seconds for r in res]}
print(json.dumps({"total_nodes": sum(out["nodes"]), "optimal": sum(1 for s in out["status"] if s == 0),
                  "kernel_s": st.kernel_seconds}))
json.dump(out, open("gpurun_out/c2_parity_nodes.json", "w"))
