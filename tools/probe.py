"""Dev probe: quick speed numbers for the search kernel (not the bench)."""
import sys, time, json
sys.path.insert(0, '.')
import paper_1908_06418_b200 as M

def c2_pairs():
    out = []
    for i in range(100):
        k = i % 3; p = (0.1, 0.3, 0.5)[k]; j = i // 3
        s = 30000 + 1000 * k + 2 * j
        out.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
    return out

g, h = M.random_graph(20, .3, 1), M.random_graph(20, .3, 2)
M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY))
for mode in (M.MODE_PARITY, M.MODE_THROUGHPUT):
    t = time.time(); r = M.solve(g, h, M.SolveConfig(mode=mode)); w = time.time() - t
    s = r.stats
    print(f"C1 s1 mode={mode} size={r.size} nodes={s.recursions} kernel={s.kernel_seconds*1e3:.2f}ms wall={w*1e3:.2f}ms "
          f"rate={s.recursions/s.kernel_seconds/1e6:.2f}M/s warps={s.warps} smem_cls={s.smem_classes} donations={s.donations}")
pairs = c2_pairs()
for mode, budget in ((M.MODE_THROUGHPUT, 120), (M.MODE_PARITY, 20)):
    t = time.time()
    res, st = M.solve_batch(pairs, M.SolveConfig(mode=mode, budget_seconds=budget))
    w = time.time() - t
    nopt = sum(r.status == M.SolveStatus.optimal for r in res)
    print(f"C2 mode={mode} optimal={nopt}/100 nodes={st.recursions} kernel={st.kernel_seconds:.3f}s wall={w:.3f}s "
          f"rate={st.recursions/st.kernel_seconds/1e9:.3f}G/s warps={st.warps} ctas={st.ctas} smem/cta={st.smem_per_cta} "
          f"donations={st.donations} tasks={st.tasks} spills={st.spills} C/node={st.sum_classes/max(1,st.recursions):.2f}")
    print(" sizes", [r.size for r in res][:12], "solve_s max", max(r.stats.solve_seconds for r in res))
    if mode == M.MODE_PARITY:
        rates = sorted(r.stats.recursions / max(r.stats.solve_seconds, 1e-9) for r in res if r.status == 0)
        print(" per-warp node rates (M/s) min/med/max", rates[0]/1e6, rates[len(rates)//2]/1e6, rates[-1]/1e6)
