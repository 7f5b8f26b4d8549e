"""GPU parity: the sm_100a search kernel (through the C ABI) against the oracle.

Parity mode (one warp per instance, no donation) must reproduce the reference's
sequential solve() node-for-node: same optimum size, same node count
(stats.recursions), same mapping. Throughput mode (donation + shared
incumbent) must reproduce the optimum size and return a verified mapping; its
node count legitimately differs (pruning order changes).
Tolerance: none — everything here is integer, bit-exact.
"""
import ctypes

import numpy as np
import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import diamond, k4, pair, random_pairs, to_oracle

pytestmark = pytest.mark.gpu

PARITY = M.SolveConfig(mode=M.MODE_PARITY)
THROUGHPUT = M.SolveConfig(mode=M.MODE_THROUGHPUT)


def _same(r, o):
    assert r.status == M.SolveStatus.optimal
    assert r.size == o.size
    assert r.stats.recursions == o.nodes
    assert [tuple(p) for p in r.best] == [tuple(p) for p in o.pairs]


@pytest.mark.parametrize("seed", [1, 3, 5, 7, 9])
def test_config1_seeds_node_exact(seed):
    # SURVEY §8(c) golden values: s=1 -> 13/159,486 ... (checked against the oracle here)
    g, h, go, ho = pair(20, 0.3, seed)
    o = O.solve(go, ho)
    r = M.solve(g, h, PARITY)
    _same(r, o)
    assert M.verify(g, h, r.best)


def test_worked_pair_and_kats():
    r = M.solve(diamond(), k4(), PARITY)
    assert r.size == 3 and M.verify(diamond(), k4(), r.best)
    k3 = M.from_edge_list(3, [(0, 1), (1, 2), (0, 2)])
    c4 = M.from_edge_list(4, [(0, 1), (1, 2), (2, 3), (0, 3)])
    p2 = M.from_edge_list(2, [(0, 1)])
    p3 = M.from_edge_list(3, [(0, 1), (1, 2)])
    assert M.solve(k3, c4, PARITY).size == 2
    assert M.solve(p2, p3, PARITY).size == 2
    g = M.random_graph(7, 0.4, 99)
    assert M.solve(g, g, PARITY).size == 7
    for cfg in (PARITY, THROUGHPUT):
        assert M.solve(diamond(), k4(), cfg).size == 3


def test_acceptance_corpus_parity_and_bruteforce():
    # acceptance_main.cpp:49-70 corpus (first 200 of random_pairs(500,4,9,20260801))
    for n, d, s in random_pairs(200, 4, 9, 20260801):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho)
        bf, _ = O.bruteforce(go, ho)
        r = M.solve(g, h, PARITY)
        _same(r, o)
        assert r.size == bf
        t = M.solve(g, h, THROUGHPUT)
        assert t.size == bf and M.verify(g, h, t.best)


@pytest.mark.parametrize("directed,labels", [(True, 0), (False, 2), (True, 3)])
def test_directed_labelled_parity(directed, labels):
    for s in range(1, 16):
        g, h, go, ho = pair(9, 0.5, s, directed, labels, seed_h=s + 500)
        o = O.solve(go, ho)
        _same(M.solve(g, h, PARITY), o)
        t = M.solve(g, h, THROUGHPUT)
        assert t.size == o.size and M.verify(g, h, t.best)


@pytest.mark.parametrize("n,p,seed,directed,labels", [(48, 0.3, 3, False, 6), (60, 0.3, 5, True, 8),
                                                      (64, 0.5, 7, False, 10), (40, 0.5, 11, False, 4)])
def test_wide_kernel_parity(n, p, seed, directed, labels):
    # n > 32 runs the 64-bit specialisation (n = 64: every bit of the word);
    # vertex labels keep these in the CPU oracle's seconds range
    g, h, go, ho = pair(n, p, seed, directed, labels)
    o = O.solve(go, ho, budget=60)
    assert o.status == 0
    _same(M.solve(g, h, PARITY), o)
    t = M.solve(g, h, THROUGHPUT)
    assert t.size == o.size and M.verify(g, h, t.best)


@pytest.mark.parametrize("n,k,p,directed,seed", [(48, 40, 0.5, False, 21), (64, 36, 0.4, True, 22),
                                                 (64, 60, 0.5, False, 23), (40, 34, 0.7, True, 24)])
def test_more_than_32_classes_parity(n, k, p, directed, seed):
    """Levels of more than 32 label classes: every one of k > 32 vertex labels
    sits on both sides, so the 64-bit policy's second class slot (classes
    32..63 of a level) is live from the root down."""
    rng = np.random.default_rng(seed)
    gr, hr = M.random_graph(n, p, seed, directed), M.random_graph(n, p, seed + 1, directed)
    lg = rng.permutation(np.arange(n) % k).astype(np.int32)
    lh = rng.permutation(np.arange(n) % k).astype(np.int32)
    g, h = M.Graph(n, gr.codes, directed, lg), M.Graph(n, hr.codes, directed, lh)
    go, ho = to_oracle(g), to_oracle(h)
    o = O.solve(go, ho, budget=60)
    assert o.status == 0
    _same(M.solve(g, h, PARITY), o)
    t = M.solve(g, h, THROUGHPUT)
    assert t.size == o.size and M.verify(g, h, t.best)


def test_more_than_32_classes_under_heavy_donation(monkeypatch):
    """The same >32-class levels while every warp donates and takes subtrees
    (16-node polls): donated levels carry the second slot's classes through
    the ring and back into HiSlot."""
    monkeypatch.setenv("MCSG_DEBUG_POLL_INTERVAL", "16")
    for n, k, p, directed, seed in [(48, 40, 0.5, False, 21), (64, 36, 0.4, True, 22), (56, 44, 0.6, False, 25)]:
        rng = np.random.default_rng(seed)
        gr, hr = M.random_graph(n, p, seed, directed), M.random_graph(n, p, seed + 1, directed)
        g = M.Graph(n, gr.codes, directed, rng.permutation(np.arange(n) % k).astype(np.int32))
        h = M.Graph(n, hr.codes, directed, rng.permutation(np.arange(n) % k).astype(np.int32))
        o = O.solve(to_oracle(g), to_oracle(h), budget=60)
        assert o.status == 0
        t = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, max_warps=64))
        assert t.status == M.SolveStatus.optimal and t.size == o.size and M.verify(g, h, t.best)
        assert t.stats.donations > 0


def test_directed_labelled_n40_parity():
    # config 3 shape (directed, vertex-labelled, n=40), easy cells
    for i, (L, p) in enumerate([(4, 0.3), (8, 0.5), (8, 0.3), (4, 0.5)]):
        g, h, go, ho = pair(40, p, 40000 + 2 * i, True, L)
        o = O.solve(go, ho, budget=20)
        assert o.status == 0
        _same(M.solve(g, h, PARITY), o)
        assert M.solve(g, h, THROUGHPUT).size == o.size


@pytest.mark.parametrize("order", [1, 2, 3])
def test_orderings_parity(order):
    for n, d, s in random_pairs(12, 5, 12, 2024):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho, order=order)
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY, order=M.OrderingStrategy(order)))
        _same(r, o)
        assert M.verify(g, h, r.best)


def test_disable_pruning_counts():
    for n, d, s in random_pairs(10, 4, 7, 4321):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho, prune=False)
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY, disable_pruning=True))
        _same(r, o)


def test_batch_both_modes():
    specs = random_pairs(60, 8, 22, 777)
    pairs = [pair(n, d, s) for n, d, s in specs]
    expect = [O.solve(go, ho) for _, _, go, ho in pairs]
    res, st = M.solve_batch([(g, h) for g, h, _, _ in pairs], PARITY)
    for r, o in zip(res, expect):
        _same(r, o)
    assert st.recursions == sum(o.nodes for o in expect)
    res, st = M.solve_batch([(g, h) for g, h, _, _ in pairs], THROUGHPUT)
    for (g, h, _, _), r, o in zip(pairs, res, expect):
        assert r.status == M.SolveStatus.optimal and r.size == o.size and M.verify(g, h, r.best)


def test_empty_and_degenerate():
    e0 = M.from_edge_list(0, [])
    one = M.from_edge_list(1, [])
    iso = M.from_edge_list(5, [])
    for cfg in (PARITY, THROUGHPUT):
        assert M.solve(e0, e0, cfg).size == 0
        assert M.solve(one, one, cfg).size == 1
        assert M.solve(iso, one, cfg).size == 1
        assert M.solve(iso, iso, cfg).size == 5
    # disjoint label sets leave nothing to match
    a = M.from_edge_list(3, [], labels=[0, 0, 0])
    b = M.from_edge_list(3, [], labels=[1, 1, 1])
    r = M.solve(a, b, PARITY)
    assert r.size == 0 and r.stats.recursions == 1


def test_errors_and_statuses():
    und = M.random_graph(5, 0.5, 1)
    dire = M.random_graph(5, 0.5, 1, directed=True)
    with pytest.raises(M.GraphError):
        M.solve(und, dire)
    lab = M.random_graph(5, 0.5, 1, label_count=2)
    with pytest.raises(M.GraphError):
        M.solve(und, lab)
    big = M.random_graph(256, 0.5, 1)  # n <= 255 (test_gpu_wide.py covers 65..255)
    with pytest.raises(M.GraphError):
        M.solve(big, big)
    g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
    r = M.solve(g, h, M.SolveConfig(budget_seconds=0))
    assert r.status == M.SolveStatus.timeout and r.size == 0
    for mode in (M.MODE_PARITY, M.MODE_THROUGHPUT):
        r = M.solve(g, h, M.SolveConfig(budget_seconds=0.2, mode=mode))
        assert r.status == M.SolveStatus.timeout
        assert r.size > 0 and M.verify(g, h, r.best)
    flag = ctypes.c_int32(1)
    r = M.solve(g, h, M.SolveConfig(cancel=flag, mode=M.MODE_THROUGHPUT))
    assert r.status == M.SolveStatus.cancelled and M.verify(g, h, r.best)


def test_goal_directed_and_bound_jump():
    for n, d, s in random_pairs(20, 4, 10, 555):
        g, h, go, ho = pair(n, d, s)
        o = O.solve_goal_directed(go, ho)
        r = M.solve_goal_directed(g, h, PARITY)
        assert r.size == o.size and r.stats.probes == o.probes
        assert r.stats.recursions == o.nodes
        assert M.verify(g, h, r.best)
        for dbl in (0, 1):
            for cb in (0, 2):
                oj = O.bound_jump(go, ho, cb, dbl)
                rj = M.bound_jump_search(g, h, cb, M.JumpMode(dbl), PARITY)
                assert rj.size == oj.size and rj.stats.probes == oj.probes
                assert rj.stats.recursions == oj.nodes
    p3 = M.from_edge_list(3, [(0, 1), (1, 2)])
    k3 = M.from_edge_list(3, [(0, 1), (1, 2), (0, 2)])
    r = M.solve_goal_directed(p3, k3)
    assert r.size == 2 and r.stats.probes == 2
    r = M.bound_jump_search(p3, k3, 1, M.JumpMode.plus_one)
    assert r.size == 2 and r.stats.probes == 2


def test_portfolio_race():
    for n, d, s in random_pairs(10, 10, 20, 7777):
        g, h, go, ho = pair(n, d, s)
        o = O.solve(go, ho)
        pr = M.run_portfolio(g, h, ["recursive", "recursive+order=degree",
                                    "recursive+order=components", "recursive+order=block"])
        assert pr.status == M.SolveStatus.optimal and pr.size == o.size
        assert M.verify(g, h, pr.mapping) and pr.winner


def test_run_engine_dispatch():
    g, h, go, ho = pair(16, 0.5, 31)
    o = O.solve(go, ho)
    for spec in ("recursive", "goal", "parallel:4", "iterative", "jump:plus1", "jump:double",
                 "restarts:11", "gpu", "recursive+order=degree", "parallel+order=block"):
        r = M.run_engine(g, h, M.parse_engine_spec(spec))
        assert r.status == M.SolveStatus.optimal and r.size == o.size, spec
        assert M.verify(g, h, r.best)
