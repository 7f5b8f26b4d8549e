"""The C4 golden (tests/golden/c4_proof.json) and the decomposition behind it.

C4's "no common subgraph of 17" was proved with the UNMODIFIED reference's
sequential solve() on the pieces of a decomposition at the top of its own
search tree (tools/c4_split_proof.py): branch v->u is the vertex-labelled
pair (G-v, H-u) with label = adjacency to v / u under floor - 1, and
"v unmatched" is (G-v, H), decomposed again. These CPU tests check the
identity behind it on small instances against the C oracle, and that the
committed ledger covers every piece of the decomposition with a proof."""
import json
import os
import sys

import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tools"))
from c4_split_proof import decomposition  # noqa: E402


@pytest.mark.parametrize("n,m,p,seed,depth", [(9, 10, 0.5, 11, 1), (10, 10, 0.3, 12, 2), (10, 11, 0.6, 13, 3),
                                              (11, 10, 0.5, 14, 4), (8, 12, 0.4, 15, 2)])
def test_decomposition_identity(n, m, p, seed, depth):
    """MCS(G, H) = max(1 + MCS of every labelled branch piece, MCS of the
    remainder); and a floor f holds for the pair iff it holds piece by piece."""
    g, h = O.random_graph(n, p, seed), O.random_graph(m, p, seed + 1000)
    opt = O.solve(g, h).size
    tasks, removed = decomposition(depth, g, h, floor=opt)
    assert len(tasks) == 1 + depth * m and len(set(removed)) == depth
    best = 0
    for tag, gs, hs, fl in tasks:
        size = O.solve(gs, hs).size
        assert size <= fl, tag  # the true optimum passes as a floor on every piece
        best = max(best, size + (0 if tag.startswith("unmatched") else 1))
    assert best == opt
    # one below the optimum, some piece must fail its floor
    tasks, _ = decomposition(depth, g, h, floor=opt - 1)
    assert any(O.solve(gs, hs).size > fl for _, gs, hs, fl in tasks)


def test_c4_proof_golden():
    path = os.path.join(HERE, "golden", "c4_proof.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c4_proof.json not produced yet (tools/c4_split_proof.py)")
    proof = json.load(open(path))
    assert proof["status"] == 0 and proof["optimum"] == 16 and proof["witness_reference_verify"] == 1
    g, h = O.random_graph(45, 0.5, 45000), O.random_graph(45, 0.5, 45001)
    wit = [tuple(x) for x in proof["witness"]]
    assert len(wit) == 16 and O.verify(g, h, wit)
    tasks, removed = decomposition(proof["no_17"]["depth"], g, h, floor=16)
    assert removed == proof["no_17"]["removed_vertices"]
    ledger = [json.loads(l) for l in open(os.path.join(HERE, "golden", "c4_pieces.jsonl")) if l.strip()]
    by_tag = {rec["piece"]: rec for rec in ledger}
    assert len(tasks) == proof["no_17"]["pieces"]
    for tag, _, _, fl in tasks:
        rec = by_tag[tag]
        assert rec["floor"] == fl and rec["status"] == 0 and rec["size"] <= fl and rec["proved"], rec
