import json, sys
sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
pairs = []
i = 0
for L in (2, 4, 8):
    for p in (0.1, 0.3, 0.5):
        for _ in range(10):
            pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L), M.random_graph(40, p, 40001 + 2 * i, True, L)))
            i += 1
cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT)
M.solve_batch(pairs, cfg)
res, st = M.solve_batch(pairs, cfg)
print(json.dumps({"lib": M.LIB_PATH.split("/")[-1], "c3_s": st.kernel_seconds, "c3_rate": st.recursions / st.kernel_seconds / 1e9, "sizes": sum(r.size for r in res)}))
