"""First-call vs steady-state latency of one small solve (dev tool)."""
import sys, time
sys.path.insert(0, '.')
t0 = time.perf_counter()
import paper_1908_06418_b200 as M
g, h = M.random_graph(20, 0.3, 1), M.random_graph(20, 0.3, 2)
t1 = time.perf_counter()
r = M.solve(g, h)
t2 = time.perf_counter()
r = M.solve(g, h)
t3 = time.perf_counter()
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY))
t4 = time.perf_counter()
g45, h45 = M.random_graph(40, 0.3, 1), M.random_graph(40, 0.3, 2)
r = M.solve(g45, h45, M.SolveConfig(budget_seconds=0.5))
t5 = time.perf_counter()
r = M.solve(g45, h45, M.SolveConfig(budget_seconds=0.5))
t6 = time.perf_counter()
print(f"import {t1-t0:.3f}s first solve {t2-t1:.3f}s second {t3-t2:.4f}s parity-first {t4-t3:.3f}s "
      f"wide-first {t5-t4:.3f}s wide-second {t6-t5:.3f}s")
