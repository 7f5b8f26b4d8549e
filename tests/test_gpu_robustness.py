"""Launch robustness: the task ring's producer watchdog turns a stall into an
error (never a hang), and the device stays usable afterwards.

The stall is provoked with the library's test hooks: a 4-slot ring
(MCSG_DEBUG_RING_CAP) makes producers wait for slots, and a zero watchdog
(MCSG_DEBUG_RING_WATCHDOG_NS) makes any such wait fatal.
"""
import json
import os

import pytest

import oracle as O
import paper_1908_06418_b200 as M

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def c2_pairs(count):
    out = []
    for i in range(count):
        k, j = i % 3, i // 3
        s = 30000 + 1000 * k + 2 * j
        p = (0.1, 0.3, 0.5)[k]
        out.append((M.random_graph(30, p, s), M.random_graph(30, p, s + 1)))
    return out


def test_ring_stall_is_an_error_and_the_device_recovers(monkeypatch):
    pairs = c2_pairs(6)
    monkeypatch.setenv("MCSG_DEBUG_RING_CAP", "4")
    monkeypatch.setenv("MCSG_DEBUG_RING_WATCHDOG_NS", "0")
    stalled = False
    for _ in range(5):
        try:
            M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
        except M.GraphError as e:
            assert "task ring stalled" in str(e), e
            stalled = True
            break
    assert stalled, "the debug ring never stalled"
    monkeypatch.delenv("MCSG_DEBUG_RING_CAP")
    monkeypatch.delenv("MCSG_DEBUG_RING_WATCHDOG_NS")
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    res, _ = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    assert [r.size for r in res] == [gold[str(i)] for i in range(6)]


def test_small_ring_without_watchdog_is_still_exact(monkeypatch):
    # a 64-slot ring: producers wait for consumers, results stay exact
    pairs = c2_pairs(6)
    monkeypatch.setenv("MCSG_DEBUG_RING_CAP", "64")
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    res, _ = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
    assert [r.size for r in res] == [gold[str(i)] for i in range(6)]


def test_heavy_donation_stress_is_exact(monkeypatch):
    # a 16-node poll interval: ~1M donations per 100-pair batch. This exposed a
    # warp-divergence race (prefetched words read after the next prefetch was
    # issued); the optima must stay exact and the launch must not fault.
    pairs = c2_pairs(100)
    monkeypatch.setenv("MCSG_DEBUG_POLL_INTERVAL", "16")
    gold = json.load(open(os.path.join(HERE, "golden", "c2_sizes.json")))["sizes"]
    for _ in range(2):
        res, st = M.solve_batch(pairs, M.SolveConfig(mode=M.MODE_THROUGHPUT))
        assert [r.size for r in res] == [gold[str(i)] for i in range(100)]
        assert all(r.status == M.SolveStatus.optimal for r in res)
        assert st.donations > 100000


@pytest.mark.parametrize("n,p,labels,directed", [(32, 0.5, 16, False), (32, 0.5, 32, True), (32, 0.3, 8, True)])
def test_full_width_32bit_stacks_exhaustive(n, p, labels, directed):
    """The 32-bit kernel's class stack carries no overflow check (its size,
    m(m+1)/2 + 64, bounds every path: a level at depth k holds at most m - k
    classes). Exhaustive searches on full-width n = 32 pairs with many label
    classes reach the deepest, widest stacks: node counts must equal the
    oracle's in parity mode and the size in throughput mode."""
    from util import to_oracle
    g, h = M.random_graph(n, p, 777, directed, labels), M.random_graph(n, p, 778, directed, labels)
    o = O.solve(to_oracle(g), to_oracle(h), prune=False)
    par = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY, disable_pruning=True))
    assert (par.size, par.stats.recursions) == (o.size, o.nodes)
    thr = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, disable_pruning=True))
    assert thr.status == M.SolveStatus.optimal and thr.size == o.size and M.verify(g, h, thr.best)
