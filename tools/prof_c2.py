"""Profile driver: one throughput-mode launch over a C2 subset (ncu target)."""
import sys
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mode = int(sys.argv[2]) if len(sys.argv) > 2 else M.MODE_THROUGHPUT
pairs = []
for i in range(n):
    k = i % 3; p = (0.1, 0.3, 0.5)[k]; j = i // 3
    s = 30000 + 1000 * k + 2 * j
    pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
res, st = M.solve_batch(pairs, M.SolveConfig(mode=mode, budget_seconds=60))
print("nodes", st.recursions, "kernel_s", st.kernel_seconds, "rate G/s", st.recursions / st.kernel_seconds / 1e9,
      "C/node", st.sum_classes / st.recursions, "splits/node", st.splits / st.recursions,
      "split_cls/split", st.split_classes / max(1, st.splits),
      "busy_frac", st.busy_cycles / max(1, st.busy_cycles + st.idle_cycles), "tasks", st.tasks,
      "donations", st.donations, "busy cycles/node", st.busy_cycles / st.recursions)
