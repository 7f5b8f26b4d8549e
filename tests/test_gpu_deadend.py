"""Dead-end handling with the reference's semantics (DeadEndMonitor /
deadend_check, heuristics.hpp:30-60, heuristics.cpp:103-112, checked per node
before the node's offer, search_core.hpp:133-141; forecast-then-jump,
portfolio.cpp:136-155).

Parity mode runs the monitor per node: without a jump it counts suspect
nodes; with one it stops at the reference's node and the bound jump resumes.
recursions, probes, deadend_suspects, size and mapping must equal the
unmodified reference's (tests/golden/deadend.json, make_golden.py deadend).
"""
import json
import os

import pytest

import paper_1908_06418_b200 as M

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "deadend.json")))["cases"]


@pytest.mark.parametrize("spec", sorted({c["spec"] for c in CASES}))
def test_parity_deadend_matches_reference(spec):
    for c in (c for c in CASES if c["spec"] == spec):
        g, h = M.random_graph(c["n"], c["d"], c["seed"]), M.random_graph(c["n"], c["d"], c["seed"] + 1)
        r = M.run_engine(g, h, M.parse_engine_spec(spec), M.SolveConfig(mode=M.MODE_PARITY))
        got = (int(r.status), r.size, r.stats.recursions, r.stats.probes, r.stats.deadend_suspects)
        want = (c["status"], c["size"], c["nodes"], c["probes"], c["suspects"])
        assert got == want, (spec, c["n"], c["d"], c["seed"], got, want)
        assert [list(p) for p in r.best] == c["pairs"], (spec, c["seed"])


def test_throughput_deadend_keeps_the_optimum():
    """The all-warp engine's poll-granular monitor: optimum unchanged."""
    for c in CASES:
        if "jump" not in c["spec"]:
            continue
        g, h = M.random_graph(c["n"], c["d"], c["seed"]), M.random_graph(c["n"], c["d"], c["seed"] + 1)
        r = M.run_engine(g, h, M.parse_engine_spec(c["spec"]))
        assert r.status == M.SolveStatus.optimal and r.size == c["size"] and M.verify(g, h, r.best)
