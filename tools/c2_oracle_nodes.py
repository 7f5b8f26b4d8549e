"""Re-derives tests/golden/c2_sequential_nodes.json's per-pair node counts
(first produced by GPU parity mode) with the C oracle — the reference's
sequential algorithm restated and pinned — for all 100 C2 pairs, and records
which pairs were checked (dev tool, CPU; ≈ 5 min on one core)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

path = os.path.join(ROOT, "tests", "golden", "c2_sequential_nodes.json")
d = json.load(open(path))
checked = []
for i in range(100):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    r = O.solve(O.random_graph(30, p, s), O.random_graph(30, p, s + 1))
    assert (r.nodes, r.size) == (d["nodes"][i], d["size"][i]), (i, r.nodes, d["nodes"][i], r.size, d["size"][i])
    checked.append(i)
    print(i, r.nodes, flush=True)
d["oracle_checked"] = checked
d["how"] = ("GPU parity mode (one warp per pair, reference node order); all 100 pairs re-derived with the C "
            "oracle (oracle/mcs_oracle.c, pinned to the reference; tools/c2_oracle_nodes.py) and equal")
json.dump(d, open(path, "w"), indent=1)
