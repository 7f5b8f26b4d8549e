"""Node rate of each kernel flavour on the same workload (dev tool).

The C2 batch (100 ER pairs, n = 30) is solved as is (32-bit kernel) and with
one trivial extra pair of 33 / 65 / 129 isolated vertices, which makes the
whole batch run the 64-bit / 128-bit / 256-bit kernel. Node counts differ a
little between runs (throughput mode); the rate is what is compared.
"""
import json
import sys

sys.path.insert(0, ".")
import paper_1908_06418_b200 as M  # noqa: E402

pairs = []
for i in range(100):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT)
for extra in (0, 33, 65, 129):
    batch = pairs + ([(M.from_edge_list(extra, []), M.from_edge_list(1, []))] if extra else [])
    M.solve_batch(batch, cfg)  # warm-up
    res, st = M.solve_batch(batch, cfg)
    print(json.dumps({"extra_n": extra, "kernel_s": st.kernel_seconds, "nodes": st.recursions,
                      "nodes_per_s": st.recursions / st.kernel_seconds, "warps": st.warps,
                      "smem_per_cta": st.smem_per_cta, "spills": st.spills,
                      "sizes_ok": [r.size for r in res[:100]] == [r.size for r in M.solve_batch(pairs, cfg)[0]]}),
          flush=True)
