"""Portfolio heuristics on the GPU engine.

restarts:<seed>  seeded search order (throughput mode); optimum unchanged.
+deadend=...     dead-end monitor: with a jump, the monitored all-warp solve
                 stops on a suspect verdict and the bound jump resumes from
                 the incumbent (portfolio.cpp:136-155). Optimum unchanged.
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import pair, random_pairs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def c2(i):
    k, j = i % 3, i // 3
    s = 30000 + 1000 * k + 2 * j
    p = (0.1, 0.3, 0.5)[k]
    return M.random_graph(30, p, s), M.random_graph(30, p, s + 1)


def test_restart_seeds_keep_the_optimum():
    for n, d, s in random_pairs(10, 10, 24, 991):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho)
        sizes = set()
        for seed in (1, 7, 123456789):
            r = M.run_engine(g, h, M.parse_engine_spec(f"restarts:{seed}"))
            assert r.status == M.SolveStatus.optimal and M.verify(g, h, r.best)
            sizes.add(r.size)
        assert sizes == {o.size}


def test_deadend_with_jump_resumes_to_the_optimum():
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    for i in (1, 2):
        g, h = c2(i)
        for spec in ("jump:plus1+deadend=abs:2000", "jump:double+deadend=rel:1.5"):
            r = M.run_engine(g, h, M.parse_engine_spec(spec))
            assert r.status == M.SolveStatus.optimal and r.size == gold[str(i)], spec
            assert M.verify(g, h, r.best)
        r = M.run_engine(g, h, M.parse_engine_spec("jump:plus1+deadend=abs:2000"))
        assert r.stats.deadend_suspects == 1 and r.stats.probes >= 1


def test_deadend_without_jump_is_a_plain_solve():
    g, h = c2(4)
    r = M.run_engine(g, h, M.parse_engine_spec("recursive+deadend=abs:10"))
    assert r.status == M.SolveStatus.optimal and r.stats.deadend_suspects == 0
    assert M.verify(g, h, r.best)


def test_portfolio_with_restarts_and_orderings():
    g, h = c2(5)
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]["5"]
    pr = M.run_portfolio(g, h, ["recursive", "restarts:3", "restarts:9+order=degree", "recursive+order=block"])
    assert pr.status == M.SolveStatus.optimal and pr.size == gold and M.verify(g, h, pr.mapping)
