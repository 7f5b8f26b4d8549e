"""Host-side pieces of the restart engine that need no GPU: VisitedRanges
(heuristics.cpp:187-210; test_heuristics.cpp:214-227) and the RestartConfig
defaults (heuristics.hpp:92-104)."""
import paper_1908_06418_b200 as M


def test_visited_range_normalization_merges_touching_runs():
    vr = M.VisitedRanges()
    vr.add([(0, 0)], [(0, 2)])
    vr.add([(0, 2)], [(0, 5)])
    assert vr.normalize()
    assert vr.size() == 1
    assert vr.covers([(0, 4)])
    assert not vr.covers([(0, 5)])
    bad = M.VisitedRanges()
    bad.add([(0, 0)], [(0, 3)])
    bad.add([(0, 2)], [(0, 4)])
    assert not bad.normalize()  # overlap detected


def test_position_key_order_is_lexicographic():
    vr = M.VisitedRanges()
    vr.add([], [(0, 2**31 - 1)])
    assert vr.normalize() and vr.covers([(0, 0), (1, 7)]) and vr.covers([])
    assert not vr.covers([(0, 2**31 - 1)])


def test_restart_config_defaults_mirror_the_reference():
    c = M.RestartConfig()
    assert (c.seed, c.multiplier, c.disable_pruning, c.ranges_out) == (1, 2.0, False, None)
    assert c.mode == M.MODE_PARITY
    assert M.parse_engine_spec("restarts:7").restart_seed == 7
