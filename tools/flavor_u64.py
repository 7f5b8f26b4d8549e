"""64-bit kernel rate on C2's node mix (C2 + one 33-vertex pair) and on C4 (dev tool)."""
import json, sys
sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
pairs = []
for i in range(100):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    pairs.append((M.random_graph(30, (0.1, 0.3, 0.5)[k], s), M.random_graph(30, (0.1, 0.3, 0.5)[k], s + 1)))
cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT)
batch = pairs + [(M.from_edge_list(33, []), M.from_edge_list(1, []))]
M.solve_batch(batch, cfg)
res, st = M.solve_batch(batch, cfg)
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, cfg)
print(json.dumps({"lib": M.LIB_PATH.split("/")[-1], "c2_u64_rate": st.recursions / st.kernel_seconds / 1e9,
                  "c4_s": r.stats.kernel_seconds, "c4_rate": r.stats.recursions / r.stats.kernel_seconds / 1e9,
                  "c4_size": r.size, "warps": r.stats.warps}))
