"""Multi-device paths exercised on one GPU.

Repeated device ordinals place several shards on the same B200: each shard
has its own context (ring, instance state) and its own persistent launch, the
shards run one after another, and incumbent sizes still travel between their
GroupStates with system-scope atomics — the same code path as 8 GPUs over
NVLink, minus the concurrency. Results must be exact: frontier subtrees
cover the whole tree exactly once.
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import pair, random_pairs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("devices,frontier", [((0, 0), 0), ((0, 0, 0, 0), 8), ((0, 0, 0), 1)])
def test_sharded_single_instance_exact(devices, frontier):
    for n, d, s in random_pairs(12, 12, 26, 31337):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho, budget=30)
        assert o.status == 0
        r = M.solve(g, h, M.SolveConfig(devices=devices, frontier=frontier))
        assert r.status == M.SolveStatus.optimal and r.size == o.size, (n, d, s)
        assert M.verify(g, h, r.best)


def test_sharded_c2_pairs_match_reference_pool():
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    for i in (1, 2, 4, 5, 7, 8):  # the p=0.3 / p=0.5 pairs (the hard ones)
        k, j = i % 3, i // 3
        s = 30000 + 1000 * k + 2 * j
        p = (0.1, 0.3, 0.5)[k]
        g, h = M.random_graph(30, p, s), M.random_graph(30, p, s + 1)
        r = M.solve(g, h, M.SolveConfig(devices=(0, 0)))
        assert r.status == M.SolveStatus.optimal and r.size == gold[str(i)]
        assert M.verify(g, h, r.best)


def test_sharded_directed_labelled():
    for s in range(1, 6):
        g, h, go, ho = pair(14, 0.5, s, True, 2, seed_h=s + 500)
        o = O.solve(go, ho)
        r = M.solve(g, h, M.SolveConfig(devices=(0, 0), frontier=4))
        assert r.size == o.size and M.verify(g, h, r.best)


def test_sharded_trivial_instances_finish_on_host():
    g = M.random_graph(6, 0.5, 3)
    r = M.solve(g, g, M.SolveConfig(devices=(0, 0)))
    assert r.size == 6 and M.verify(g, g, r.best)
    e = M.from_edge_list(3, [])
    assert M.solve(e, e, M.SolveConfig(devices=(0, 0))).size == 3


def test_multi_device_portfolio():
    for n, d, s in random_pairs(6, 14, 22, 4242):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho)
        cfg = M.SolveConfig(devices=(0, 0))
        pr = M.run_portfolio(g, h, ["recursive", "recursive+order=degree", "recursive+order=block"], cfg)
        assert pr.status == M.SolveStatus.optimal and pr.size == o.size and M.verify(g, h, pr.mapping)
        assert pr.winner


def test_c4_sharded():
    g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
    r = M.solve(g, h, M.SolveConfig(devices=(0, 0), budget_seconds=300))
    assert r.status == M.SolveStatus.optimal and r.size == 16 and M.verify(g, h, r.best)
