"""Profile driver: one throughput launch of the undirected 64-bit kernel
without a deadline (replay-safe, unlike C4): 8 ER pairs n=40, p=0.5 — the C4
kernel on C4-like trees (dev tool)."""
import json
import sys

sys.path.insert(0, ".")
import paper_1908_06418_b200 as M  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pairs = [(M.random_graph(40, 0.5, 46000 + 2 * i), M.random_graph(40, 0.5, 46001 + 2 * i)) for i in range(k)]
res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
print(json.dumps({"nodes": st.recursions, "kernel_s": st.kernel_seconds, "sizes": [r.size for r in res],
                  "rate_g": st.recursions / st.kernel_seconds / 1e9}), flush=True)
