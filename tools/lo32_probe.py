"""Measures how many 64-bit-kernel nodes sit at levels whose live vertex sets fit 32 bits (needs a build with the EXPERIMENT block described in DESIGN §9; dev tool)."""
import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=3))
st = r.stats
print("C4 nodes", st.recursions, "lo32 nodes", st.sum_classes, round(st.sum_classes / st.recursions, 3), "compactable", st.split_classes, round(st.split_classes / st.recursions, 3))
pairs = []
i = 0
for L in (2, 4, 8):
    for p in (0.1, 0.3, 0.5):
        for _ in range(10):
            pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L), M.random_graph(40, p, 40001 + 2 * i, True, L))); i += 1
res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
print("C3 nodes", st.recursions, "lo32", round(st.sum_classes / st.recursions, 3), "compactable", round(st.split_classes / st.recursions, 3))
