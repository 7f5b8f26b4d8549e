"""C4's "no 17" with the UNMODIFIED reference, decomposed at the top of its
own search tree (dev tool, hours of CPU). Resumable: every finished piece is
appended to tests/golden/c4_pieces.jsonl (committed as it grows), and a rerun
skips the pieces already there; tools/c4_proof_json.py turns a complete
ledger into tests/golden/c4_proof.json.

McSplit branches on one vertex v of G: v -> u for each u of H, or v left
unmatched. A common induced subgraph that maps v to u is {v->u} plus a common
induced subgraph of G - v and H - u that preserves adjacency to v / u, i.e.
a common subgraph of the vertex-LABELLED pair (label x = code(v, x), label y =
code(u, y)); one that leaves v unmatched is a common subgraph of G - v and H.
So
    MCS(G, H) <= 16  <=>  for every u: MCS_labelled(G-v, H-u) <= 15
                          and MCS(G - v, H) <= 16,
and the last term is decomposed again on the next vertex (depth levels). Each
piece is the reference's own sequential solve() with a SharedBound floor
(oracle/_ref ref_solve_floor, SolveConfig::shared_bound, solve.hpp:70-81):
status optimal with a result no larger than the floor proves the piece. The
pieces are the top branches of the reference's own tree (v = its first
choice, max degree), so the total work is about the floor-16 tree's, spread
over every core instead of the thread pool's part_level-5 tasks (whose tail
ran on one thread for hours).

usage: python tools/c4_split_proof.py [DEPTH=12] [WORKERS=nproc] [LEDGER]"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def sub(g, keep, labels=None):
    idx = np.array(keep, dtype=np.int64)
    codes = np.ascontiguousarray(np.asarray(g.codes).reshape(g.n, g.n)[np.ix_(idx, idx)])
    lab = None if labels is None else np.ascontiguousarray(np.array(labels, dtype=np.int32))
    return O.G(len(keep), codes, g.directed, lab)


def decomposition(depth, g=None, h=None, floor=16):
    """[(tag, G piece, H piece, floor)]: the remainder first, then the branch
    pieces level by level (largest first, for the tail). MCS(g, h) <= floor
    iff every piece's MCS is at most its floor."""
    if g is None:
        g, h = O.ref_random_graph(45, 0.5, 45000), O.ref_random_graph(45, 0.5, 45001)
    n, m = g.n, h.n
    cg = np.asarray(g.codes).reshape(n, n)
    ch = np.asarray(h.codes).reshape(m, m)
    gl = list(range(n))
    tasks, removed = [], []
    for level in range(depth):
        # the reference's choice: max degree among G's remaining vertices, lowest id on ties
        deg = {x: int(sum(1 for y in gl if y != x and cg[x, y])) for x in gl}
        v = min(gl, key=lambda x: (-deg[x], x))
        rest = [x for x in gl if x != v]
        for u in range(m):
            hrest = [y for y in range(m) if y != u]
            tasks.append((f"v{v}->u{u}@{level}", sub(g, rest, [int(cg[v, x]) for x in rest]),
                          sub(h, hrest, [int(ch[u, y]) for y in hrest]), floor - 1))
        removed.append(v)
        gl = rest
    return [(f"unmatched{removed}", sub(g, gl), sub(h, list(range(m))), floor)] + tasks, removed


def piece(args):
    tag, gs, hs, floor = args
    t = time.time()
    r = O.ref_solve_floor(gs, hs, floor, budget=1e9)
    return {"piece": tag, "floor": floor, "status": r.status, "size": r.size, "nodes": r.nodes,
            "seconds": round(time.time() - t, 1), "proved": r.status == 0 and r.size <= floor}


def main():
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    ledger = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "tests", "golden", "c4_pieces.jsonl")
    tasks, removed = decomposition(depth)
    done = set()
    if os.path.exists(ledger):
        done = {json.loads(l)["piece"] for l in open(ledger) if l.strip()}
    todo = [t for t in tasks if t[0] not in done]
    print(json.dumps({"depth": depth, "removed": removed, "pieces": len(tasks), "todo": len(todo),
                      "workers": workers}), flush=True)
    with ProcessPoolExecutor(workers) as ex, open(ledger, "a") as out:
        futs = [ex.submit(piece, t) for t in todo]
        for f in as_completed(futs):
            res = f.result()
            out.write(json.dumps(res) + "\n")
            out.flush()
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
