"""GPU parity for wide graphs (64 < n <= 255): the 128- and 256-bit kernels.

Same bar as test_gpu_parity.py: parity mode reproduces the reference's
sequential solve() node for node (size, stats.recursions, mapping), throughput
mode reproduces the optimum with a verified mapping. The instances cover the
word boundaries (n = 65, 100, 128, 129, 130, 200, 254, 255), levels with more
than 32 classes (64 and 128 vertex labels: several lane passes per level),
directed 4-way splits, unequal sizes, and levels that spill to HBM.
Tolerance: none — integer, bit-exact.
"""
import pytest

import oracle as O
import paper_1908_06418_b200 as M
from util import to_oracle

pytestmark = pytest.mark.gpu

PARITY = M.SolveConfig(mode=M.MODE_PARITY)
THROUGHPUT = M.SolveConfig(mode=M.MODE_THROUGHPUT)


def path(n):
    return M.from_edge_list(n, [(i, i + 1) for i in range(n - 1)])


def cycle(n):
    return M.from_edge_list(n, [(i, (i + 1) % n) for i in range(n)])


def complete(n):
    return M.from_edge_list(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def structured():
    return [("P100/P100", path(100), path(100)), ("C100/P100", cycle(100), path(100)),
            ("K254/K254", complete(254), complete(254)), ("K255/K255", complete(255), complete(255)),
            ("K100/K70", complete(100), complete(70)), ("C130/C130", cycle(130), cycle(130)),
            ("K65/P65", complete(65), path(65)), ("P129/C128", path(129), cycle(128))]


# (n_G, n_H, p, directed, labels); G seed 81000 + n_G, H seed 82000 + n_H.
# Each is proven by the CPU oracle in about a second.
RANDOM = [(100, 100, 0.5, False, 32), (70, 70, 0.3, True, 16), (130, 130, 0.5, True, 64),
          (200, 200, 0.5, True, 64), (254, 254, 0.5, True, 128)]


def random_pair(ng, nh, p, directed, labels):
    return (M.random_graph(ng, p, 81000 + ng, directed, labels),
            M.random_graph(nh, p, 82000 + nh, directed, labels))


def _same(r, o):
    assert r.status == M.SolveStatus.optimal
    assert r.size == o.size
    assert r.stats.recursions == o.nodes
    assert [tuple(p) for p in r.best] == [tuple(p) for p in o.pairs]


def _oracle(g, h):
    o = O.solve(to_oracle(g), to_oracle(h), budget=60)
    assert o.status == 0
    return o


def test_structured_parity_and_throughput():
    cases = structured()
    expect = [_oracle(g, h) for _, g, h in cases]
    res, _ = M.solve_batch([(g, h) for _, g, h in cases], PARITY)
    for (name, g, h), r, o in zip(cases, res, expect):
        _same(r, o)
        assert M.verify(g, h, r.best), name
    assert expect[2].size == 254 and expect[3].size == 255  # K254 / K255 self
    res, _ = M.solve_batch([(g, h) for _, g, h in cases], THROUGHPUT)
    for (name, g, h), r, o in zip(cases, res, expect):
        assert r.status == M.SolveStatus.optimal and r.size == o.size, name
        assert M.verify(g, h, r.best), name


@pytest.mark.parametrize("spec", RANDOM, ids=lambda s: "n%d-%d_p%s_%s_L%d" % (s[0], s[1], s[2], "dir" if s[3] else "und", s[4]))
def test_random_wide_parity(spec):
    g, h = random_pair(*spec)
    o = _oracle(g, h)
    _same(M.solve(g, h, PARITY), o)
    t = M.solve(g, h, THROUGHPUT)
    assert t.status == M.SolveStatus.optimal and t.size == o.size and M.verify(g, h, t.best)


def test_mixed_batch_runs_wide_kernel():
    # narrow and wide pairs in one launch: the batch runs the wide flavour and
    # every pair keeps its reference node count
    pairs = [(M.random_graph(20, 0.3, s), M.random_graph(20, 0.3, s + 1)) for s in (1, 3, 5)]
    pairs += [random_pair(130, 130, 0.5, True, 64)]
    pairs += [(M.random_graph(40, 0.5, 40002, True, 8), M.random_graph(40, 0.5, 40003, True, 8))]
    expect = [_oracle(g, h) for g, h in pairs]
    res, st = M.solve_batch(pairs, PARITY)
    for r, o in zip(res, expect):
        _same(r, o)
    assert st.recursions == sum(o.nodes for o in expect)


def test_spill_to_hbm_keeps_parity():
    # the smallest shared-memory stack (one level of n+1 classes): deeper
    # levels live in the per-warp HBM spill area
    g, h = random_pair(200, 200, 0.5, True, 64)
    o = _oracle(g, h)
    r = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY, smem_classes=64))
    _same(r, o)
    assert r.stats.spills > 0
    t = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, smem_classes=64))
    assert t.size == o.size and M.verify(g, h, t.best)


def test_wide_goal_probes():
    g, h = random_pair(130, 130, 0.5, True, 64)
    go, ho = to_oracle(g), to_oracle(h)
    o = O.solve_goal_directed(go, ho)
    r = M.solve_goal_directed(g, h, PARITY)
    assert r.size == o.size and r.stats.probes == o.probes and r.stats.recursions == o.nodes
    oj = O.bound_jump(go, ho, 2, 1)
    rj = M.bound_jump_search(g, h, 2, M.JumpMode.doubling, PARITY)
    assert rj.size == oj.size and rj.stats.probes == oj.probes and rj.stats.recursions == oj.nodes


def test_wide_orderings_parity():
    g, h = random_pair(100, 100, 0.5, False, 32)
    go, ho = to_oracle(g), to_oracle(h)
    for order in (1, 2, 3):
        o = O.solve(go, ho, order=order)
        r = M.solve(g, h, M.SolveConfig(mode=M.MODE_PARITY, order=M.OrderingStrategy(order)))
        _same(r, o)


@pytest.mark.parametrize("devices,frontier", [((0, 0), 0), ((0, 0, 0), 3)])
def test_wide_sharded_over_devices(devices, frontier):
    # one wide instance expanded on the host into wide frozen subtrees dealt to
    # device contexts (repeated ordinals: the multi-GPU path on one B200)
    for spec in RANDOM[:4]:
        g, h = random_pair(*spec)
        o = _oracle(g, h)
        r = M.solve(g, h, M.SolveConfig(devices=devices, frontier=frontier))
        assert r.status == M.SolveStatus.optimal and r.size == o.size, spec
        assert M.verify(g, h, r.best)
    g = complete(200)
    r = M.solve(g, g, M.SolveConfig(devices=devices))
    assert r.size == 200 and M.verify(g, g, r.best)


def test_wide_multi_device_portfolio():
    g, h = random_pair(100, 100, 0.5, False, 32)
    o = _oracle(g, h)
    pr = M.run_portfolio(g, h, ["recursive", "recursive+order=degree", "restarts:3"],
                         M.SolveConfig(devices=(0, 0)))
    assert pr.status == M.SolveStatus.optimal and pr.size == o.size and M.verify(g, h, pr.mapping)
