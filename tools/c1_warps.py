import sys, json, statistics
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
pairs = [(M.random_graph(20, 0.3, s), M.random_graph(20, 0.3, s + 1)) for s in (1, 3, 5, 7, 9)]
for w in (0, 2048, 1024, 512, 256, 128, 64):
    ts = []
    for rep in range(3):
        for g, h in pairs:
            r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, max_warps=w))
            ts.append(r.stats.kernel_seconds)
    print(json.dumps({"max_warps": w, "median_ms": round(1e3 * statistics.median(ts), 4), "max_ms": round(1e3 * max(ts), 4)}), flush=True)
