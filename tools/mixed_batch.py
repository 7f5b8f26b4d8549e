import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
pairs = []
for i in range(6):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
c4 = (M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001))
res, st = M.solve_batch(pairs + [c4], M.SolveConfig(budget_seconds=1.0))
print([(r.status.name, r.size, round(r.stats.solve_seconds, 3)) for r in res])
