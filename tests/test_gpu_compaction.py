"""Compacted subtrees in the 64-bit kernel (CompactSearch).

A level whose live vertex sets fit 32 bits runs its subtree in place with the
32-bit policy on renumbered vertices (the task body nested at that level,
its class stack above the level in shared memory; a subtree whose stack
would not fit there runs in the 64-bit policy). Renumbering keeps id order,
so the search is the same tree: with pruning disabled the node count is
identical with compaction on and off (MCSG_DEBUG_NO_COMPACT) and with most
subtrees refused for room (MCSG_DEBUG_COMPACT_ROOM=150: only small nests run
compacted, the rest fall back to the 64-bit policy); optima and mappings
stay exact.
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import pair

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _exhaustive(g, h):
    return M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, disable_pruning=True))


def test_compaction_keeps_the_exhaustive_tree(monkeypatch):
    # n = 34..40 (64-bit kernel), sparse labelled pairs small enough to enumerate
    # (the CPU oracle enumerates each in 0-3 s: 2e4..6e7 nodes)
    cases = [(34, 0.2, 71, False, 8), (36, 0.3, 73, True, 8), (40, 0.2, 77, False, 12), (38, 0.5, 79, True, 16),
             (33, 0.3, 5, False, 10), (36, 0.5, 9, True, 12), (40, 0.4, 21, False, 16)]
    for n, p, s, directed, labels in cases:
        g, h, go, ho = pair(n, p, s, directed, labels)
        on = _exhaustive(g, h)
        monkeypatch.setenv("MCSG_DEBUG_COMPACT_ROOM", "150")
        smem = _exhaustive(g, h)
        monkeypatch.setenv("MCSG_DEBUG_COMPACT_ROOM", "60")
        hbm = _exhaustive(g, h)
        monkeypatch.delenv("MCSG_DEBUG_COMPACT_ROOM")
        monkeypatch.setenv("MCSG_DEBUG_NO_COMPACT", "1")
        off = _exhaustive(g, h)
        monkeypatch.delenv("MCSG_DEBUG_NO_COMPACT")
        assert on.status == off.status == smem.status == hbm.status == M.SolveStatus.optimal
        assert on.size == off.size == smem.size == hbm.size, (n, p, s)
        assert on.stats.recursions == off.stats.recursions == smem.stats.recursions == hbm.stats.recursions, (n, p, s)
        assert M.verify(g, h, on.best)


def test_compaction_optima_match_the_oracle():
    for n, p, s, directed, labels in [(48, 0.3, 3, False, 6), (60, 0.3, 5, True, 8), (64, 0.5, 7, False, 10),
                                      (40, 0.5, 11, False, 4), (45, 0.5, 13, True, 6)]:
        g, h, go, ho = pair(n, p, s, directed, labels)
        o = O.solve(go, ho, budget=120)
        assert o.status == 0
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT))
        assert r.status == M.SolveStatus.optimal and r.size == o.size and M.verify(g, h, r.best)


def test_compaction_c3_and_c4():
    i, sizes = 0, []
    pairs = []
    for L in (2, 4, 8):
        for p in (0.1, 0.3, 0.5):
            for _ in range(10):
                pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L),
                              M.random_graph(40, p, 40001 + 2 * i, True, L)))
                i += 1
    on, _ = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    os.environ["MCSG_DEBUG_NO_COMPACT"] = "1"
    try:
        off, _ = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    finally:
        del os.environ["MCSG_DEBUG_NO_COMPACT"]
    assert [r.size for r in on] == [r.size for r in off]
    assert all(r.status == M.SolveStatus.optimal for r in on)
    for (g, h), r in zip(pairs, on):
        assert M.verify(g, h, r.best)
    g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
    r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=120))
    assert r.status == M.SolveStatus.optimal and r.size == 16 and M.verify(g, h, r.best)


def test_compacted_subtrees_under_heavy_donation(monkeypatch):
    # 16-node polls: the nested 32-bit DFS donates its levels (ids mapped
    # back to the 64-bit ring format) hundreds of thousands of times; the
    # exhaustive tree must stay the same tree, node for node
    monkeypatch.setenv("MCSG_DEBUG_POLL_INTERVAL", "16")
    for n, p, s, directed, labels in [(40, 0.4, 21, False, 16), (40, 0.2, 77, False, 12), (36, 0.5, 9, True, 12)]:
        g, h, go, ho = pair(n, p, s, directed, labels)
        on = _exhaustive(g, h)
        monkeypatch.setenv("MCSG_DEBUG_NO_COMPACT", "1")
        off = _exhaustive(g, h)
        monkeypatch.delenv("MCSG_DEBUG_NO_COMPACT")
        assert on.status == off.status == M.SolveStatus.optimal
        assert on.size == off.size and on.stats.recursions == off.stats.recursions, (n, p, s)
        assert M.verify(g, h, on.best)
    # and C3-style directed labelled pairs, pruning on: the same optima as
    # without compaction
    pairs = []
    i = 0
    for L in (2, 4, 8):
        for p in (0.1, 0.3, 0.5):
            for _ in range(2):
                pairs.append((M.random_graph(40, p, 40000 + 2 * i, True, L),
                              M.random_graph(40, p, 40001 + 2 * i, True, L)))
                i += 1
    on, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    monkeypatch.setenv("MCSG_DEBUG_NO_COMPACT", "1")
    off, _ = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    monkeypatch.delenv("MCSG_DEBUG_NO_COMPACT")
    assert [r.size for r in on] == [r.size for r in off]
    assert all(r.status == M.SolveStatus.optimal for r in on)
    assert st.donations > 10000
    for (g, h), r in zip(pairs, on):
        assert M.verify(g, h, r.best)
