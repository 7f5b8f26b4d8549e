import sys; sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
k, j = 5 % 3, 5 // 3
s = 30000 + 1000 * k + 2 * j
g, h = M.random_graph(30, 0.5, s), M.random_graph(30, 0.5, s + 1)
which = sys.argv[1] if len(sys.argv) > 1 else "race"
if which == "alone":
    for ws in (1, 2, 3):
        try:
            r = M.run_engine(g, h, M.parse_engine_spec("restarts:3"), M.SolveConfig(warp_share=ws))
            print("alone", ws, r.status, r.size, r.stats.warps, flush=True)
        except Exception as e:
            print("EXC alone", ws, e, flush=True)
else:
    specs = [M.parse_engine_spec(x) for x in ["recursive", "restarts:3", "restarts:9+order=degree", "recursive+order=block"]]
    w, b, reps, gv = M._race(g, h, specs, M.SolveConfig(), 1e9, None, 1.0)
    print(w and w[0], [(e.spec_name, e.outcome, e.error) for e in reps], flush=True)
