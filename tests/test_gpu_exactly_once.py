"""Exactly-once coverage of the work-sharing machinery.

With pruning disabled (SolveConfig::disable_pruning, solve.hpp:122) the
search tree no longer depends on the incumbent, so every traversal order must
visit exactly the same node multiset — the GPU counterpart of the reference's
parallel-completeness criterion (acceptance_main.cpp:141-168). Donation to
idle warps, the ticket ring, and the multi-device frontier split must
neither lose nor duplicate a subtree: the GPU node count must equal the
sequential oracle's on the same (kernel-ordered) graphs.

Throughput mode relabels G in (degree desc, id asc) order before searching,
which changes only class tie-breaks; the oracle is run on that relabelled G.
"""
import numpy as np
import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import random_pairs

pytestmark = pytest.mark.gpu


def degree_relabel(g):
    n = g.n()
    order = sorted(range(n), key=lambda v: (-g.degree(v), v))
    fwd = np.empty(n, np.int64)
    fwd[order] = np.arange(n)
    return M.permute(g, fwd)


def oracle_nodes(g, h):
    gr = degree_relabel(g)
    go = O.G(gr.n(), gr.codes.copy(), gr.directed(), None if gr.labels is None else gr.labels.copy())
    ho = O.G(h.n(), h.codes.copy(), h.directed(), None if h.labels is None else h.labels.copy())
    return O.solve(go, ho, prune=False)


@pytest.mark.parametrize("devices", [(), (0, 0, 0)])
def test_no_pruning_node_counts_equal_sequential(devices):
    for n, d, s in random_pairs(12, 7, 11, 8181):
        g, h = M.random_graph(n, d, s), M.random_graph(n, d, s + 1)
        o = oracle_nodes(g, h)
        cfg = M.SolveConfig(mode=M.MODE_THROUGHPUT, disable_pruning=True, devices=devices, frontier=4)
        r = M.solve(g, h, cfg)
        assert r.status == M.SolveStatus.optimal and r.size == o.size
        assert r.stats.recursions == o.nodes, (n, d, s, r.stats.recursions, o.nodes)


def test_no_pruning_directed_labelled_batch():
    pairs, expect = [], []
    for s in range(1, 9):
        g = M.random_graph(9, 0.5, s, True, 2)
        h = M.random_graph(9, 0.5, s + 70, True, 2)
        pairs.append((g, h))
        expect.append(oracle_nodes(g, h).nodes)
    res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT, disable_pruning=True))
    assert [r.stats.recursions for r in res] == expect
    assert st.donations > 0  # the trees really were shared between warps
