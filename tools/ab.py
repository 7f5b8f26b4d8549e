"""A/B of library builds on one GPU (dev tool): C2 batch (bench workload),
C3 batch, C4 proof; each lib loaded in its own process via MCSG_LIB.
usage: python tools/ab.py LIB1.so LIB2.so ... [--reps N] [--only c2,c3,c4,c5]"""
import json, os, subprocess, sys

libs = [a for a in sys.argv[1:] if a.endswith(".so")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 2
only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else "c2,c3,c4"
CHILD = r'''
import json, sys, time
sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
only = sys.argv[1].split(",")
out = {"lib": M.LIB_PATH.split("/")[-1]}
thr = M.SolveConfig(mode=M.MODE_THROUGHPUT)
if "c2" in only:
    pairs = []
    for i in range(100):
        k, j = i % 3, i // 3
        s = 30000 + 1000 * k + 2 * j
        p = (0.1, 0.3, 0.5)[k]
        pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
    M.solve_batch(pairs, thr)
    best = None
    for _ in range(3):
        res, st = M.solve_batch(pairs, thr)
        if best is None or st.kernel_seconds < best[0]:
            best = (st.kernel_seconds, st.recursions)
    out["c2_s"] = round(best[0], 4)
    out["c2_gnps"] = round(best[1] / best[0] / 1e9, 3)
if "c3" in only:
    pairs = []
    i = 0
    for L in (2, 4, 8):
        for p in (0.1, 0.3, 0.5):
            for _ in range(10):
                pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L), M.random_graph(40, p, 40001 + 2 * i, True, L)))
                i += 1
    M.solve_batch(pairs, thr)
    res, st = M.solve_batch(pairs, thr)
    out["c3_s"] = round(st.kernel_seconds, 4)
    out["c3_gnps"] = round(st.recursions / st.kernel_seconds / 1e9, 3)
if "c5" in only:
    pairs = []
    for i in range(10000):
        n, p = 16 + (i // 3) % 9, (0.1, 0.3, 0.5)[i % 3]
        pairs.append((M.random_graph(n, p, 50000 + 2 * i), M.random_graph(n, p, 50001 + 2 * i)))
    M.solve_batch(pairs, thr)
    best = None
    for _ in range(3):
        res, st = M.solve_batch(pairs, thr)
        if best is None or st.kernel_seconds < best[0]:
            best = (st.kernel_seconds, st.recursions)
    out["c5_s"] = round(best[0], 4)
    out["c5_gnps"] = round(best[1] / best[0] / 1e9, 3)
if "c4" in only:
    g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
    r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=60))
    out["c4_s"] = round(r.stats.kernel_seconds, 3)
    out["c4_size"] = r.size
    out["c4_gnps"] = round(r.stats.recursions / r.stats.kernel_seconds / 1e9, 3)
print(json.dumps(out), flush=True)
'''
for rep in range(reps):
    for lib in libs:
        env = dict(os.environ, MCSG_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CHILD, only], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
