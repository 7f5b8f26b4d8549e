"""Pins the CPU oracle (oracle/mcs_oracle.c) to the reference.

Golden vectors in tests/golden/small.json were produced by the UNMODIFIED
reference solver (oracle/_ref, built from /root/reference/proj/src) via
tests/golden/make_golden.py. Everything is integer: exact equality.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "small.json")))


def test_generator_bit_identical():
    for rec in GOLD["generator"]:
        g = O.random_graph(rec["n"], rec["p"], rec["seed"], rec["directed"], rec["labels"])
        assert g.codes.reshape(-1).tobytes().hex() == rec["codes_hex"]
        if rec["vlabels"] is not None:
            assert g.labels.tolist() == rec["vlabels"]


def test_config1_seeds():
    # s=1 -> 13 / 159,486 nodes, s=3 -> 12 / 261,455, ...
    expect = {1: (13, 159486), 3: (12, 261455), 5: (13, 118671), 7: (13, 132345), 9: (12, 239329)}
    for rec in GOLD["config1"]:
        s = rec["seed"]
        g, h = O.random_graph(20, 0.3, s), O.random_graph(20, 0.3, s + 1)
        r = O.solve(g, h)
        assert (r.size, r.nodes) == expect[s] == (rec["size"], rec["nodes"])
        assert [list(p) for p in r.pairs] == rec["pairs"]


def test_acceptance_corpus():
    for rec in GOLD["acceptance"]:
        g, h = O.random_graph(rec["n"], rec["d"], rec["seed"]), O.random_graph(rec["n"], rec["d"], rec["seed"] + 1)
        r = O.solve(g, h)
        assert r.size == rec["size"] == rec["bf"]
        assert r.nodes == rec["nodes"]
        assert [list(p) for p in r.pairs] == rec["pairs"]
        assert O.verify(g, h, r.pairs)


def test_bruteforce_matches_reference_sizes():
    for rec in GOLD["acceptance"][:150]:
        g, h = O.random_graph(rec["n"], rec["d"], rec["seed"]), O.random_graph(rec["n"], rec["d"], rec["seed"] + 1)
        k, wit = O.bruteforce(g, h)
        assert k == rec["bf"] and O.verify(g, h, wit)


def test_directed_and_labelled():
    for rec in GOLD["kinds"]:
        g = O.random_graph(rec["n"], 0.5, rec["seed"], rec["directed"], rec["labels"])
        h = O.random_graph(rec["n"], 0.5, rec["seed_h"], rec["directed"], rec["labels"])
        r = O.solve(g, h)
        assert (r.size, r.nodes) == (rec["size"], rec["nodes"])
        assert [list(p) for p in r.pairs] == rec["pairs"]


def test_goal_directed_and_bound_jump():
    for rec in GOLD["probes"]:
        g, h = O.random_graph(rec["n"], rec["d"], rec["seed"]), O.random_graph(rec["n"], rec["d"], rec["seed"] + 1)
        r = O.solve_goal_directed(g, h)
        assert (r.size, r.nodes, r.probes) == (rec["goal"]["size"], rec["goal"]["nodes"], rec["goal"]["probes"])
        for dbl in (0, 1):
            for cb in (0, 2):
                j = O.bound_jump(g, h, cb, dbl)
                ex = rec[f"jump_{dbl}_{cb}"]
                assert (j.size, j.nodes, j.probes) == (ex["size"], ex["nodes"], ex["probes"])


def test_orderings():
    names = {1: "degree", 2: "components", 3: "block"}
    for rec in GOLD["orderings"]:
        g = O.random_graph(rec["n"], 0.4, rec["seed"])
        h = O.random_graph(rec["n"], 0.4, rec["seed_h"])
        for o, nm in names.items():
            assert O.ordering(g, o).tolist() == rec[f"perm_{nm}"]
            r = O.solve(g, h, order=o)
            ex = rec[f"solve_{nm}"]
            assert (r.size, r.nodes) == (ex["size"], ex["nodes"])
            assert [list(p) for p in r.pairs] == ex["pairs"]


def test_exhaustive_enumeration():
    for rec in GOLD["exhaustive"]:
        g, h = O.random_graph(rec["n"], rec["d"], rec["seed"]), O.random_graph(rec["n"], rec["d"], rec["seed"] + 1)
        r = O.solve(g, h, prune=False)
        assert (r.size, r.nodes) == (rec["size"], rec["nodes"])


def test_reference_kats():
    kat = GOLD["kat"]
    diamond = O.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3)])
    k4 = O.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
    k3 = O.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    c4 = O.from_edges(4, [(0, 1), (1, 2), (2, 3), (0, 3)])
    p2 = O.from_edges(2, [(0, 1)])
    p3 = O.from_edges(3, [(0, 1), (1, 2)])
    assert O.solve(diamond, k4).size == kat["diamond_k4"]["size"] == 3
    assert O.verify(diamond, k4, [(0, 1), (1, 2), (2, 0)])  # test_oracle.cpp:16
    assert O.solve(k3, c4).size == kat["k3_c4"]["size"] == 2
    assert O.solve(p2, p3).size == kat["p2_p3"]["size"] == 2
    r = O.solve_goal_directed(p3, k3)
    assert (r.size, r.probes) == (kat["p3_k3_goal"]["size"], kat["p3_k3_goal"]["probes"]) == (2, 2)
    j = O.bound_jump(p3, k3, 1, 0)
    assert (j.size, j.probes) == (kat["p3_k3_jump_plus1_from1"]["size"], kat["p3_k3_jump_plus1_from1"]["probes"]) == (2, 2)
    g7 = O.random_graph(7, 0.4, 99)
    assert O.solve(g7, g7).size == kat["rg7_self"]["size"] == 7
    # refine chain of the worked example (test_label_classes.cpp:85-108): bound 3 after two pairs
    assert kat["refine_chain_diamond_k4"][2]["bound"] == 3
    assert len(kat["refine_chain_diamond_k4"][3]["classes"]) == 0
    assert len(kat["refine_directed_4way"]["classes"]) == 4


def test_verify_rejections():
    p3 = O.from_edges(3, [(0, 1), (1, 2)])
    two = O.from_edges(3, [(0, 1)])
    assert not O.verify(p3, two, [(1, 1), (2, 2)])
    assert not O.verify(p3, p3, [(0, 0), (1, 0)])
    with pytest.raises(ValueError):
        O.verify(p3, p3, [(0, 9)])
    la = O.G(2, np.zeros((2, 2), np.uint8), False, np.array([0, 1], np.int32))
    assert not O.verify(la, la, [(0, 1)])
    assert O.verify(la, la, [(0, 0), (1, 1)])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (dev container only)")
def test_live_reference_agreement():
    """Direct cross-check of the restatement against the reference library."""
    for s in range(1, 25):
        for directed, labels in ((False, 0), (True, 0), (False, 3)):
            g = O.random_graph(11, 0.45, s, directed, labels)
            h = O.random_graph(11, 0.45, s + 31, directed, labels)
            r = O.solve(g, h)
            rr = O.ref_run_engine(g, h, "recursive")
            assert (r.size, r.nodes, r.pairs) == (rr.size, rr.nodes, rr.pairs)


def test_restarts_match_reference():
    """solve_with_restarts restated (restarts.cpp:195-246) vs the unmodified
    reference's (tests/golden/restarts.json): size, recursions, restarts,
    visited ranges, mapping and the ranges themselves."""
    cases = json.load(open(os.path.join(HERE, "golden", "restarts.json")))["cases"]
    assert len(cases) >= 80
    for c in cases:
        dr, lb = c.get("directed", False), c.get("labels", 0)
        g = O.random_graph(c["n"], c["d"], c["seed"], dr, lb)
        h = O.random_graph(c.get("nh", c["n"]), c["d"], c["seed"] + 1, dr, lb)
        r = O.solve_with_restarts(g, h, seed=c["rseed"], multiplier=c["mult"], prune=c["prune"], order=c["order"])
        got = (r.status, r.size, r.nodes, r.extra["restarts"], r.extra["visited_ranges"])
        assert got == (0, c["size"], c["nodes"], c["restarts"], c["visited_ranges"]), c
        assert [list(p) for p in r.pairs] == c["pairs"]
        if "ranges" in c:
            assert [[[x for _, x in lo], [x for _, x in hi]] for lo, hi in r.extra["ranges"]] == c["ranges"]


def test_restart_ranges_tile_the_tree():
    """test_heuristics.cpp:177-199 on the restatement: disjoint ranges merging
    into one run from the root key to successor({})."""
    for n, d, s in [(4 + i % 3, (0.2, 0.5, 0.8)[i % 3], 999 + 977 * i) for i in range(10)]:
        g, h = O.random_graph(n, d, s), O.random_graph(n, d, s + 1)
        r = O.solve_with_restarts(g, h, seed=s, multiplier=1.0, prune=False)
        runs = sorted((list(lo), list(hi)) for lo, hi in r.extra["ranges"])
        merged = []
        for lo, hi in runs:
            assert not merged or lo >= merged[-1][1]  # disjoint
            if merged and lo == merged[-1][1]:
                merged[-1][1] = hi
            else:
                merged.append([lo, hi])
        assert merged == [[[], [(0, 2**31 - 1)]]]
