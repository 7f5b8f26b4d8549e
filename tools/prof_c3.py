"""Profile driver: one C3 batch launch (90 directed labelled pairs, n=40, the
64-bit kernel with compacted subtrees), no budget, so kernel replay is valid.
Prints the node count of the launch (ncu replays restore memory, so the
printed stats belong to one replay)."""
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
res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
print(json.dumps({"nodes": st.recursions, "kernel_s": st.kernel_seconds, "sizes": [r.size for r in res],
                  "rate_g": st.recursions / st.kernel_seconds / 1e9, "warps": st.warps}), flush=True)
