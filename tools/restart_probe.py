"""Exhaustive node counts with and without restarts on small pairs (dev tool)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle as O
import paper_1908_06418_b200 as M
from util import pair, random_pairs
for n, d, s in random_pairs(6, 8, 11, 999):
    g, h, go, ho = pair(n, d, s)
    o = O.solve(go, ho, prune=False)
    row = [n, d, s, o.nodes]
    for mult in (0.0, 1.0, 1.0, 1.0):
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, disable_pruning=True, restart_multiplier=mult))
        row.append((r.stats.recursions - o.nodes, r.stats.restarts, r.stats.frozen))
    print(row, flush=True)
