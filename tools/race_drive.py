"""compute-sanitizer target (racecheck / synccheck / memcheck): small throughput
launches that exercise the ring hard — a 16-node poll interval
(MCSG_DEBUG_POLL_INTERVAL, set by the caller) makes every warp donate and
consume subtrees constantly. Covers the 32-bit kernel (C1-shaped pairs), the
64-bit kernel with compacted subtrees (n=40 directed labelled, C3-shaped), the
restart instantiation and a wide pair. Sizes are checked against the oracle.
Dev tool (imports the oracle as the checker only)."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from util import to_oracle  # noqa: E402
import oracle as O  # noqa: E402
import paper_1908_06418_b200 as M  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
warps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = {}


def check(tag, pairs, **kw):
    cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT, max_warps=warps, **kw)
    res, st = M.solve_batch(pairs, cfg)
    ok = True
    for (g, h), r in zip(pairs, res):
        ref = O.solve(to_oracle(g), to_oracle(h))
        ok &= (r.size == ref.size) and M.verify(g, h, r.best)
    out[tag] = {"pairs": len(pairs), "ok": bool(ok), "nodes": st.recursions, "donations": st.donations}
    print(json.dumps({tag: out[tag]}), flush=True)


if which in ("all", "u32"):
    check("u32", [(M.random_graph(20, 0.3, s), M.random_graph(20, 0.3, s + 1)) for s in (1, 3, 5)])
if which in ("all", "u64"):
    check("u64_compact", [(M.random_graph(40, 0.3, 40000 + 2 * i, True, 4), M.random_graph(40, 0.3, 40001 + 2 * i, True, 4))
                          for i in range(2)])
if which in ("all", "u64u"):
    # the undirected 64-bit kernel (C4's): compacted subtrees in shared memory
    # (PEXT entry, s0 room bound), and a level of more than 32 classes (the
    # second class slot read from the stack copy, HiSlot)
    import numpy as np
    pairs = [(M.random_graph(36, 0.5, 46000 + 2 * i, False, 4), M.random_graph(36, 0.5, 46001 + 2 * i, False, 4))
             for i in range(2)]
    rng = np.random.default_rng(7)
    gr, hr = M.random_graph(48, 0.5, 21), M.random_graph(48, 0.5, 22)
    pairs.append((M.Graph(48, gr.codes, False, rng.permutation(np.arange(48) % 40).astype(np.int32)),
                  M.Graph(48, hr.codes, False, rng.permutation(np.arange(48) % 40).astype(np.int32))))
    check("u64_undirected", pairs)
if which in ("all", "rst"):
    check("u32_restarts", [(M.random_graph(22, 0.4, 7), M.random_graph(22, 0.4, 8))], restart_multiplier=2.0)
if which in ("all", "wide"):
    # path P70 vs cycle C70 (n > 64: the 128-bit policy): the optimum is P69, 69
    path = M.from_edge_list(70, [(i, i + 1) for i in range(69)])
    cyc = M.from_edge_list(70, [(i, (i + 1) % 70) for i in range(70)])
    check("wide", [(path, cyc)])
print(json.dumps({"all_ok": all(v["ok"] for v in out.values())}))
