import sys, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=3))
st = r.stats
print(M.LIB_PATH.split('/')[-1], "nodes", st.recursions, "rate", round(st.recursions/st.kernel_seconds/1e9,2), "donations", st.donations, "tasks", st.tasks, "busy", round(st.busy_cycles/(st.busy_cycles+st.idle_cycles),3), "smem_classes", st.smem_classes, "warps", st.warps, "splits", st.splits)
