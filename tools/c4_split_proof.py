"""C4's "no 17" with the UNMODIFIED reference, decomposed at the top of its
own search tree (dev tool, hours of CPU; writes gpurun_out/c4_split_proof.json).

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
choice, max degree), so the total work is the floor-16 tree's, spread over
every core instead of the thread pool's part_level-5 tasks (whose tail ran on
one thread for hours)."""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def sub(g, keep, labels=None):
    idx = np.array(keep, dtype=np.int64)
    codes = np.ascontiguousarray(np.asarray(g.codes).reshape(g.n, g.n)[np.ix_(idx, idx)])
    lab = None if labels is None else np.ascontiguousarray(np.array(labels, dtype=np.int32))
    return O.G(len(keep), codes, g.directed, lab)


def piece(args):
    tag, gs, hs, floor = args
    t = time.time()
    r = O.ref_solve_floor(gs, hs, floor, budget=1e9)
    return {"piece": tag, "floor": floor, "status": r.status, "size": r.size, "nodes": r.nodes,
            "seconds": round(time.time() - t, 1), "proved": r.status == 0 and r.size <= floor}


def main():
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # levels whose branch pieces another run covers
    g, h = O.ref_random_graph(45, 0.5, 45000), O.ref_random_graph(45, 0.5, 45001)
    cg = np.asarray(g.codes).reshape(45, 45)
    ch = np.asarray(h.codes).reshape(45, 45)
    gl = list(range(45))
    tasks = []
    removed = []
    for level in range(depth):
        # the reference's choice: max degree among G's remaining vertices, lowest id on ties
        deg = {x: int(sum(1 for y in gl if y != x and cg[x, y])) for x in gl}
        v = min(gl, key=lambda x: (-deg[x], x))
        rest = [x for x in gl if x != v]
        for u in (range(45) if level >= skip else ()):
            hrest = [y for y in range(45) if y != u]
            tasks.append((f"v{v}->u{u}@{level}", sub(g, rest, [int(cg[v, x]) for x in rest]),
                          sub(h, hrest, [int(ch[u, y]) for y in hrest]), 15))
        removed.append(v)
        gl = rest
    tasks.append((f"unmatched{removed}", sub(g, gl), sub(h, list(range(45))), 16))
    t0 = time.time()
    out = {"instance": "C4 ER n=45 p=0.5 seeds 45000/45001", "removed_vertices": removed, "pieces": []}
    with ProcessPoolExecutor(workers) as ex:
        for res in ex.map(piece, tasks[::-1]):  # the big unmatched piece first (results print in this order)
            out["pieces"].append(res)
            print(json.dumps(res), flush=True)
    out["all_proved"] = all(p["proved"] for p in out["pieces"])
    out["nodes"] = sum(p["nodes"] for p in out["pieces"])
    out["wall_s"] = round(time.time() - t0, 1)
    out["workers"] = workers
    out["skip_levels"] = skip
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    name = "c4_split_proof.json" if skip == 0 else f"c4_split_proof_skip{skip}.json"
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", name), "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "pieces"}))


if __name__ == "__main__":
    main()
