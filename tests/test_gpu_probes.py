"""Parallel goal probes and portfolio members with their
own semantics (portfolio.cpp:101-157, 249-292).

probe_parallel: bound_jump_search's bracket (heuristics.cpp:114-185) probed
many targets per round; a reached target implies the lower ones and an
exhausted one the higher ones (probe ladder), within a launch and across
devices. The optimum must equal the reference's on every pair.
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import pair, random_pairs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_probe_parallel_matches_oracle_all_widths():
    for n, d, s in random_pairs(18, 8, 24, 4242):
        g, h, go, ho = pair(n, d, s)
        opt = O.solve(go, ho).size
        for width in (1, 3, 32):
            r = M.probe_parallel(g, h, 0, width)
            assert r.status == M.SolveStatus.optimal and r.size == opt, (n, d, s, width)
            assert M.verify(g, h, r.best)
            assert r.stats.probes >= 1


def test_probe_parallel_from_a_lower_bound_recovers_a_witness():
    for n, d, s in random_pairs(8, 10, 20, 99):
        g, h, go, ho = pair(n, d, s)
        opt = O.solve(go, ho).size
        r = M.probe_parallel(g, h, opt, 4)  # nothing to search: a witness probe at opt
        assert r.size == opt and M.verify(g, h, r.best)
        r = M.probe_parallel(g, h, max(opt - 3, 0), 8)
        assert r.size == opt and M.verify(g, h, r.best)
    with pytest.raises(M.GraphError):
        M.probe_parallel(*pair(6, 0.5, 1)[:2], 7)


def test_probe_parallel_directed_labelled_and_orderings():
    for s in range(1, 9):
        g, h, go, ho = pair(14, 0.4, s, directed=True, labels=3)
        opt = O.solve(go, ho).size
        for order in (M.OrderingStrategy.none, M.OrderingStrategy.degree_desc):
            r = M.probe_parallel(g, h, 0, 6, M.SolveConfig(order=order))
            assert r.size == opt and M.verify(g, h, r.best)


def test_probe_parallel_over_two_device_contexts():
    """Targets dealt over two device contexts (repeated ordinal on a one-GPU
    box); the ladder's implications cross contexts through the same
    system-scope atomics as a P2P peer's GroupState."""
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    for i in (0, 1, 3, 4):
        k, j = i % 3, i // 3
        sd = 30000 + 1000 * k + 2 * j
        p = (0.1, 0.3, 0.5)[k]
        g, h = M.random_graph(30, p, sd), M.random_graph(30, p, sd + 1)
        r = M.probe_parallel(g, h, 0, 8, M.SolveConfig(devices=(0, 0)))
        assert r.status == M.SolveStatus.optimal and r.size == gold[str(i)] and M.verify(g, h, r.best)


def test_probe_parallel_c4_brackets_the_optimum():
    """C4: the probes at 16 (reached) and 17 (exhausted) run concurrently."""
    g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
    r = M.probe_parallel(g, h, 15, 2, M.SolveConfig(budget_seconds=300))
    proof = os.path.join(HERE, "golden", "c4_proof.json")
    opt = json.load(open(proof))["optimum"] if os.path.exists(proof) else 16
    assert r.status == M.SolveStatus.optimal and r.size == opt and M.verify(g, h, r.best)
    assert 2 <= r.stats.probes <= 6  # (16, 45), then (17, 44): 17 is the proof


def test_portfolio_probe_members_run_as_probes():
    """goal / jump members are GPU probe engines, not plain searches: the
    winner reports probes and the race reports every member."""
    for n, d, s in random_pairs(6, 12, 22, 515):
        g, h, go, ho = pair(n, d, s)
        opt = O.solve(go, ho).size
        pr = M.run_portfolio(g, h, ["goal", "jump:double"])
        assert pr.status == M.SolveStatus.optimal and pr.size == opt and M.verify(g, h, pr.mapping)
        assert pr.winner in ("goal", "jump:double")
        assert pr.stats.probes > 0
        assert sorted(e.spec_name for e in pr.engines) == ["goal", "jump:double"]


def test_portfolio_mixed_members_race_and_cancel():
    g, h, go, ho = pair(26, 0.5, 777)
    opt = O.solve(go, ho).size
    specs = ["recursive", "recursive+order=degree", "goal", "restarts:3", "jump:plus1+deadend=abs:1000"]
    pr = M.run_portfolio(g, h, specs, M.SolveConfig(budget_seconds=120),
                         M.PortfolioConfig(share_incumbent=True))
    assert pr.status == M.SolveStatus.optimal and pr.size == opt and M.verify(g, h, pr.mapping)
    assert len(pr.engines) == 4  # the two searchers race in one launch; three engines
    finished = [e for e in pr.engines if e.outcome == "finished"]
    assert finished and pr.winner
    for e in pr.engines:
        if e.outcome == "cancelled":
            assert 0 <= e.cancel_ack_seconds < 1.0


def test_portfolio_staged_falls_through_to_stage_two():
    g, h, go, ho = pair(24, 0.5, 31)
    opt = O.solve(go, ho).size
    s1, s2 = M.parse_engine_spec("goal"), M.parse_engine_spec("recursive")
    s2.stage = 2
    pr = M.run_portfolio(g, h, [s1, s2], None, M.PortfolioConfig(mode="staged", stage1_budget_seconds=1e-9))
    assert pr.status == M.SolveStatus.optimal and pr.size == opt
    assert [e.spec_name for e in pr.engines][-1] == "recursive"
    with pytest.raises(M.GraphError):
        M.run_portfolio(g, h, ["parallel:2+order=degree", "gpu"], None, M.PortfolioConfig(mode="bogus"))
