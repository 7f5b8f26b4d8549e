"""Profile driver: one throughput launch of the undirected 64-bit kernel
without a deadline (replay-safe, unlike C4): k ER pairs n (default 40) with
density p — the C4 kernel on C4-like trees (dev tool).
usage: prof_u64.py [k] [n] [p]"""
import json
import sys

sys.path.insert(0, ".")
import paper_1908_06418_b200 as M  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
pairs = [(M.random_graph(n, p, 46000 + 2 * i), M.random_graph(n, p, 46001 + 2 * i)) for i in range(k)]
res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
print(json.dumps({"k": k, "n": n, "p": p, "nodes": st.recursions, "kernel_s": st.kernel_seconds,
                  "sizes": [r.size for r in res][:8], "rate_g": st.recursions / st.kernel_seconds / 1e9}), flush=True)
