"""The exact restart engine (parity mode): mcsg_solve_with_restarts against the
reference's RestartDriver (restarts.cpp:35-246, heuristics.hpp:77-107).

The host keeps the segment pool as position keys and draws with the
reference's seeded mt19937_64; each segment runs on one GPU warp (replay to
the segment's node, resume at from_iter, per-node restart check). Size,
mapping, stats.recursions, stats.restarts, stats.visited_ranges and the
visited ranges themselves must equal the unmodified reference's
(tests/golden/restarts.json, make_golden.py restarts). The tiling audit of
test_heuristics.cpp:177-199 and the "infinite threshold" check of :157-175
run on the GPU; random pairs beyond the fixtures are checked against the C
oracle's restatement (oracle/mcs_oracle.c, itself pinned to the same
fixtures by tests/test_oracle.py).
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import pair, random_pairs, to_oracle

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "restarts.json")))["cases"]
KEY_MAX = 2**31 - 1


def _graphs(c):
    dr, lb = c.get("directed", False), c.get("labels", 0)
    return (M.random_graph(c["n"], c["d"], c["seed"], dr, lb),
            M.random_graph(c.get("nh", c["n"]), c["d"], c["seed"] + 1, dr, lb))


def _run(g, h, seed, mult, prune=True, order=0, ranges=None):
    return M.solve_with_restarts(g, h, M.RestartConfig(
        seed=seed, multiplier=mult, disable_pruning=not prune, order=M.OrderingStrategy(order),
        ranges_out=ranges, mode=M.MODE_PARITY))


@pytest.mark.parametrize("idx", range(0, len(CASES), 8))
def test_restarts_match_reference(idx):
    for c in CASES[idx:idx + 8]:
        g, h = _graphs(c)
        vr = M.VisitedRanges() if "ranges" in c else None
        r = _run(g, h, c["rseed"], c["mult"], c["prune"], c["order"], vr)
        got = (int(r.status), r.size, r.stats.recursions, r.stats.restarts, r.stats.visited_ranges)
        want = (0, c["size"], c["nodes"], c["restarts"], c["visited_ranges"])
        assert got == want, (c, got, want)
        assert [list(p) for p in r.best] == c["pairs"], c
        assert r.stats.seed == c["rseed"]
        if vr is not None:
            assert [[[x for _, x in lo], [x for _, x in hi]] for lo, hi in vr.runs] == c["ranges"], c


def test_visited_ranges_tile_the_tree():
    """test_heuristics.cpp:177-199: eager restarts, pruning off — the ranges are
    disjoint and merge into one run spanning the root's whole range."""
    fired = 0
    for n, d, s in random_pairs(10, 4, 6, 999):
        g, h, go, ho = pair(n, d, s)
        vr = M.VisitedRanges()
        r = _run(g, h, s, 1.0, prune=False, ranges=vr)
        assert r.status == M.SolveStatus.optimal
        fired += r.stats.restarts > 0
        assert vr.normalize()
        assert vr.size() == 1
        assert vr.runs[0] == ([], [(0, KEY_MAX)])
        assert vr.covers([(0, 0)])
    assert fired > 0


def test_restarts_fragment_the_run():
    """test_heuristics.cpp:201-212."""
    g, h = M.random_graph(12, 0.5, 71), M.random_graph(12, 0.5, 72)
    r = _run(g, h, 5, 1.0)
    assert r.status == M.SolveStatus.optimal
    assert r.stats.restarts > 0 and r.stats.visited_ranges > 1
    assert r.size == M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY)).size


def test_infinite_threshold_is_the_sequential_search():
    """test_heuristics.cpp:157-175: multiplier 0 — the sequential visit order
    (same node count and mapping as solve()), no restarts, one range."""
    for n, d, s in random_pairs(8, 4, 7, 271) + [(20, 0.3, 1), (24, 0.4, 5)]:
        g, h, go, ho = pair(n, d, s)
        r = _run(g, h, 3, 0.0)
        o = O.solve(go, ho)
        assert (r.size, r.stats.recursions, r.stats.restarts, r.stats.visited_ranges) == (o.size, o.nodes, 0, 1)
        assert [tuple(p) for p in r.best] == [tuple(p) for p in o.pairs]


def test_restarts_deterministic():
    """test_heuristics.cpp:143-152."""
    g, h = M.random_graph(9, 0.5, 61), M.random_graph(9, 0.5, 62)
    a, b = _run(g, h, 42, 2.0), _run(g, h, 42, 2.0)
    assert a.canonical_bytes() == b.canonical_bytes() and a.stats.seed == 42


@pytest.mark.parametrize("shape", ["u32", "u32_directed_labelled", "u64", "u64_directed", "wide"])
def test_restarts_match_the_oracle_on_every_kernel_flavour(shape):
    """Random pairs through each kernel flavour (one-word 32/64-bit, the 128-bit
    wide policy) against the C oracle's restatement: size, recursions,
    restarts, visited ranges, mapping and the ranges."""
    if shape == "wide":
        # P70 vs C70: n > 64 runs the 128-bit policy
        pairs = [(M.from_edge_list(70, [(i, i + 1) for i in range(69)]),
                  M.from_edge_list(70, [(i, (i + 1) % 70) for i in range(70)]), 0.5)]
    else:
        # (n_G range, n_H, directed, labels); n_H > 32 selects the 64-bit kernel
        lo, hi, nh, dr, lb = {"u32": (14, 20, 0, False, 0), "u32_directed_labelled": (12, 18, 0, True, 3),
                              "u64": (10, 13, 40, False, 0), "u64_directed": (10, 12, 36, True, 2)}[shape]
        pairs = []
        for i, (n, d, s) in enumerate(random_pairs(4, lo, hi, 31337)):
            g = M.random_graph(n, d, s, dr, lb)
            h = M.random_graph(nh or n, d, s + 1, dr, lb)
            pairs.append((g, h, (0.5, 1.0, 2.0, 4.0)[i % 4]))
    for k, (g, h, mult) in enumerate(pairs):
        o = O.solve_with_restarts(to_oracle(g), to_oracle(h), seed=11 + k, multiplier=mult)
        vr = M.VisitedRanges()
        r = _run(g, h, 11 + k, mult, ranges=vr)
        assert (r.size, r.stats.recursions, r.stats.restarts, r.stats.visited_ranges) == \
            (o.size, o.nodes, o.extra["restarts"], o.extra["visited_ranges"]), (shape, k)
        assert [tuple(p) for p in r.best] == [tuple(p) for p in o.pairs]
        assert vr.runs == [(list(a), list(b)) for a, b in o.extra["ranges"]]


def test_run_engine_parity_restarts():
    """run_engine("restarts:<seed>") with a parity-mode config is the exact engine."""
    c = CASES[0]
    g, h = _graphs(c)
    r = M.run_engine(g, h, M.parse_engine_spec(f"restarts:{c['rseed']}"), M.SolveConfig(mode=M.MODE_PARITY))
    assert (r.size, r.stats.recursions, r.stats.restarts) == (c["size"], c["nodes"], c["restarts"])


def test_restarts_timeout_and_errors():
    g, h = M.random_graph(10, 0.5, 1), M.random_graph(10, 0.5, 2)
    r = M.solve_with_restarts(g, h, M.RestartConfig(budget_seconds=0))
    assert r.status == M.SolveStatus.timeout
    d = M.random_graph(10, 0.5, 3, True)
    with pytest.raises(M.GraphError):
        M.solve_with_restarts(g, d, M.RestartConfig())
