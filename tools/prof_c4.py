"""Profile driver: C4 (n=45, p=0.5) throughput-mode launch with a time budget
(ncu target). The deadline is absolute, so only single-pass metric sets give
valid numbers: a replayed pass would start after the deadline and stop at once.
"""
import sys
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
b = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=b))
st = r.stats
print("nodes", st.recursions, "kernel_s", st.kernel_seconds, "rate G/s", st.recursions / st.kernel_seconds / 1e9,
      "busy", st.busy_cycles / max(1, st.busy_cycles + st.idle_cycles), "warps", st.warps, "spills", st.spills, flush=True)
