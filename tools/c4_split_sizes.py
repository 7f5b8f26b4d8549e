"""Node counts of the C4 proof's decomposition pieces (tools/c4_split_proof.py),
measured on the GPU with the same floors (dev tool): how the reference's
floor-16 tree splits between the labelled branch pieces and the unmatched
remainder."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1908_06418_b200 as M  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
cg, ch = np.asarray(g.codes), np.asarray(h.codes)


def sub(codes, keep, labels=None):
    idx = np.array(keep)
    return M.Graph(len(keep), codes[np.ix_(idx, idx)], False, None if labels is None else np.array(labels, np.int32))


gl = list(range(45))
total = 0
for level in range(depth):
    deg = {x: int(sum(1 for y in gl if y != x and cg[x, y])) for x in gl}
    v = min(gl, key=lambda x: (-deg[x], x))
    rest = [x for x in gl if x != v]
    lvl_nodes = 0
    mx = 0
    for u in range(45):
        hrest = [y for y in range(45) if y != u]
        r = M.solve(sub(cg, rest, [int(cg[v, x]) for x in rest]), sub(ch, hrest, [int(ch[u, y]) for y in hrest]),
                    M.SolveConfig(mode=M.MODE_THROUGHPUT, shared_bound=15))
        assert r.size <= 15
        lvl_nodes += r.stats.recursions
        mx = max(mx, r.stats.recursions)
    total += lvl_nodes
    print(json.dumps({"level": level, "v": v, "nodes": lvl_nodes, "max_piece": mx}), flush=True)
    gl = rest
    r = M.solve(sub(cg, gl), h, M.SolveConfig(mode=M.MODE_THROUGHPUT, shared_bound=16))
    print(json.dumps({"unmatched_after": level + 1, "nodes": r.stats.recursions, "size": r.size}), flush=True)
print(json.dumps({"labelled_total": total}))
