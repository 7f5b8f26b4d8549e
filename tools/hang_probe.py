import sys, json, time
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
def c2(i):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    return M.random_graph(30, p, s), M.random_graph(30, p, s + 1)
for count in (1, 2, 3, 10, 100):
    pairs = [c2(i) for i in range(count)]
    t = time.time()
    res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=3.0))
    print(count, "wall", round(time.time() - t, 3), "kernel", round(st.kernel_seconds, 3), "nodes", st.recursions,
          "status", sorted(set(r.status.name for r in res)), "donations", st.donations, "tasks", st.tasks, flush=True)
