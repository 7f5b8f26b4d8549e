"""Shared-memory roofline figures for the search kernel; writes
profiles/r2_smem_traffic.json (dev tool).

gpu  (needs a B200; the diagnostic library built with -DMCSG_COUNT_CLASSES,
      `make -C paper_1908_06418_b200/csrc counters` -> ablibs/libmcsg_counters.so,
      which adds class-traffic counters to the product kernel at +1.2%
      instructions): one C2 batch (bench.py's workload). Per materialised child
      the kernel writes the child's classes and, at the pop back, reloads the
      parent's; the frame (f_word 8 B + f_cand 4 B) is stored at the split and
      loaded at the pop. B_node(GPU) = (split_classes x 8 B + splits x 24 B) / nodes.
alg  (CPU, the C oracle = the reference's sequential algorithm): the SURVEY's
      algorithmic model on a bounded C2 sample — C = classes of each counted
      node, S = parent classes re-read per refinement — B_node(alg) =
      (32 C + 16 S + 16) per node and ops(alg) = 20 + 14 S per node.

usage: python tools/smem_traffic.py gpu|alg   (merges into the JSON file)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "profiles", "r2_smem_traffic.json")


def c2_pair(i):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    return (0.1, 0.3, 0.5)[k], s


def load():
    return json.load(open(OUT)) if os.path.exists(OUT) else {}


def gpu():
    os.environ.setdefault("MCSG_LIB", os.path.join(ROOT, "ablibs", "libmcsg_counters.so"))
    import paper_1908_06418_b200 as M
    pairs = []
    for i in range(100):
        p, s = c2_pair(i)
        pairs.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
    cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT)
    M.solve_batch(pairs, cfg)
    _, st = M.solve_batch(pairs, cfg)
    n = st.recursions
    b = (st.split_classes * 8 + st.splits * 24) / n
    return {"workload": "C2 batch (100 pairs, throughput mode), diagnostic library -DMCSG_COUNT_CLASSES",
            "lib": os.path.basename(M.LIB_PATH), "nodes": n, "splits": st.splits,
            "split_classes": st.split_classes, "splits_per_node": st.splits / n,
            "classes_moved_per_split": st.split_classes / max(1, st.splits),
            "bytes_per_node": b, "kernel_s": st.kernel_seconds,
            "note": "class 8 B (32-bit kernel), frame 12 B stored + 12 B loaded per split; adjacency rows "
                    "(4 B per entered child, read from shared memory) not counted"}


def alg(budget_per_density=60.0):
    """Per density p in {.1,.3,.5}: C and S over the C2 pairs of that density the
    oracle finishes within the budget; the workload figure weights the
    densities by their share of C2's sequential node count
    (tests/golden/c2_sequential_nodes.json)."""
    import oracle as O
    seq = json.load(open(os.path.join(ROOT, "tests", "golden", "c2_sequential_nodes.json")))["nodes"]
    per = {}
    for k in range(3):
        C = S = nodes = 0
        used = []
        t0 = time.time()
        for i in sorted(range(k, 100, 3), key=lambda i: seq[i]):  # cheapest first
            p, s = c2_pair(i)
            g, h = O.random_graph(30, p, s), O.random_graph(30, p, s + 1)
            r = O.solve(g, h)
            C += r.extra["sum_classes"]
            S += r.extra["sum_splits"]
            nodes += r.nodes
            used.append(i)
            if time.time() - t0 > budget_per_density:
                break
        share = sum(seq[i] for i in range(k, 100, 3)) / sum(seq)
        per[str((0.1, 0.3, 0.5)[k])] = {"pairs": used, "nodes": nodes, "C_bar": C / nodes, "S_bar": S / nodes,
                                        "node_share": share}
    cb = sum(v["C_bar"] * v["node_share"] for v in per.values())
    sb = sum(v["S_bar"] * v["node_share"] for v in per.values())
    return {"workload": "C2 (node-share-weighted over the densities), sequential C oracle = the reference's tree",
            "per_density": per, "C_bar": cb, "S_bar": sb, "bytes_per_node": 32 * cb + 16 * sb + 16,
            "ops_per_node": 20 + 14 * sb,
            "model": "SURVEY 8(d): B = 16 C (written by the parent's refinement) + 16 C (read for bound and "
                     "select) + 16 S + 16 (rows); ops = 20 + 14 S (n <= 64 classes of 16 B)"}


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "alg"
    d = load()
    d[what] = gpu() if what == "gpu" else alg()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    json.dump(d, open(OUT, "w"), indent=1)
    print(json.dumps(d[what]))
