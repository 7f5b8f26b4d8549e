"""CPU-side checks of the product library (no GPU needed).

The C ABI loads and exports every function include/mcsg.h declares; the
host-side graph core (generator, orderings, verifier, loaders, packer) agrees
with the reference's golden vectors; and without a CUDA device every solve
entry point fails loudly (there is no CPU fallback).
"""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1908_06418_b200 as M

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = json.load(open(os.path.join(HERE, "golden", "small.json")))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mcsg.h")).read()
    return sorted(set(re.findall(r"\b(mcsg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(M.LIB_PATH)
    syms = declared_symbols()
    assert {"mcsg_solve", "mcsg_solve_batch", "mcsg_solve_parallel", "mcsg_solve_goal_directed",
            "mcsg_bound_jump", "mcsg_portfolio", "mcsg_verify", "mcsg_load_graph_file"} <= set(syms)
    for name in syms:
        assert hasattr(lib, name), f"{name} declared in include/mcsg.h but not exported"
    assert M.lib().mcsg_abi_version() == 5


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {M.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_generator_matches_reference():
    for rec in GOLD["generator"]:
        g = M.random_graph(rec["n"], rec["p"], rec["seed"], rec["directed"], rec["labels"])
        assert g.codes.reshape(-1).tobytes().hex() == rec["codes_hex"]
        if rec["vlabels"] is not None:
            assert g.labels.tolist() == rec["vlabels"]


def test_orderings_match_reference():
    names = {M.OrderingStrategy.degree_desc: "degree", M.OrderingStrategy.components_then_degree: "components",
             M.OrderingStrategy.block_triangular: "block"}
    for rec in GOLD["orderings"]:
        g = M.random_graph(rec["n"], 0.4, rec["seed"])
        for o, nm in names.items():
            assert M.make_ordering(g, o).tolist() == rec[f"perm_{nm}"]
    # heuristics tests (test_heuristics.cpp:12-64)
    star = M.from_edge_list(4, [(0, 1), (0, 2), (0, 3)])
    assert M.make_ordering(star, M.OrderingStrategy.degree_desc)[0] == 0
    p4 = M.from_edge_list(4, [(0, 1), (1, 2), (2, 3)])
    assert M.make_ordering(p4, M.OrderingStrategy.block_triangular).tolist() == [2, 0, 1, 3]
    iso = M.from_edge_list(4, [])
    assert M.make_ordering(iso, M.OrderingStrategy.components_then_degree).tolist() == [0, 1, 2, 3]


def test_verify_matches_reference_rules():
    diamond = M.from_edge_list(4, [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3)])
    k4 = M.from_edge_list(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
    assert M.verify(diamond, k4, [(0, 1), (1, 2), (2, 0)])
    p3 = M.from_edge_list(3, [(0, 1), (1, 2)])
    two = M.from_edge_list(3, [(0, 1)])
    assert not M.verify(p3, two, [(1, 1), (2, 2)])
    assert not M.verify(p3, p3, [(0, 0), (1, 0)])
    assert not M.verify(p3, p3, [(0, 0), (0, 1)])
    with pytest.raises(M.GraphError):
        M.verify(p3, p3, [(0, 9)])
    la = M.from_edge_list(2, [], labels=[0, 1])
    assert not M.verify(la, la, [(0, 1)])
    assert M.verify(la, la, [(0, 0), (1, 1)])
    # reference witnesses of the acceptance corpus verify with the product verifier
    for rec in GOLD["acceptance"][:100]:
        g = M.random_graph(rec["n"], rec["d"], rec["seed"])
        h = M.random_graph(rec["n"], rec["d"], rec["seed"] + 1)
        assert M.verify(g, h, rec["pairs"])


def test_from_edge_list_validation():
    with pytest.raises(M.GraphError):
        M.from_edge_list(3, [(0, 3)])
    with pytest.raises(M.GraphError):
        M.from_edge_list(3, [(1, 1)])
    with pytest.raises(M.GraphError):
        M.from_edge_list(3, [(0, 1, 1), (0, 1, 2)], directed=True)
    g = M.from_edge_list(3, [(0, 1), (0, 1)])
    assert g.edge_count() == 1
    d = M.from_edge_list(4, [(0, 1, 1), (0, 2, 2), (0, 3, 1), (1, 2, 1), (2, 3, 3)], directed=True,
                         labels=[0, 1, 0, 1])
    assert d.code(1, 0) == 2 and d.code(2, 0) == 1 and d.code(3, 2) == 3 and d.degree(2) == 4


def test_permute_roundtrip():
    for s in range(1, 8):
        g = M.random_graph(9, 0.4, s)
        p = M.random_permutation(9, s * 7)
        gp = M.permute(g, p)
        inv = np.argsort(p)
        assert M.permute(gp, inv) == g


def test_mivia_and_text_loaders(tmp_path):
    # graph_io.cpp formats; minimal MIVIA instance from test_graph.cpp:122-129
    f = tmp_path / "p2.mivia"
    f.write_bytes(bytes([0x02, 0x00, 0x01, 0x00, 0x01, 0x00, 0x00, 0x00]))
    g = M.load_graph_file(str(f))
    assert g.n() == 2 and g.adjacent(0, 1)
    for bad in ([0x02, 0x00, 0x01, 0x00, 0x05, 0x00, 0x00, 0x00], [0x02, 0x00, 0x01, 0x00],
                [0x01, 0x00, 0x00, 0x00, 0xAB], [0x02, 0x00, 0x01, 0x00, 0x00, 0x00, 0x00, 0x00]):
        f.write_bytes(bytes(bad))
        with pytest.raises(M.ParseError):
            M.load_graph_file(str(f), "mivia")
    for s in range(6):
        g = M.random_graph(3 + 9 * s, 0.4, s)
        path = str(tmp_path / f"g{s}.mivia")
        M.save_graph_file(g, path, "mivia")
        b1 = open(path, "rb").read()
        g2 = M.load_graph_file(path, "mivia")  # auto-detect reads n=48 (byte '0') as text, as the reference does
        assert g2 == g
        M.save_graph_file(g2, path, "mivia")
        assert open(path, "rb").read() == b1
    d = M.random_graph(7, 0.6, 11, directed=True, label_count=2)
    path = str(tmp_path / "d.txt")
    M.save_graph_file(d, path, "text")
    assert M.load_graph_file(path) == d
    t = tmp_path / "t.txt"
    t.write_text("3 directed labeled\n0 5\n1 5\n2 7\n0 1 1\n1 2 3\n")
    g = M.load_graph_file(str(t))
    assert g.directed() and g.label(2) == 7 and g.code(0, 1) == 1 and g.code(2, 1) == 3
    t.write_text("2 labeled\n0 1\n")
    with pytest.raises(M.ParseError):
        M.load_graph_file(str(t))


def test_pack_graph_rows():
    g = M.random_graph(40, 0.3, 40002, directed=True, label_count=4)
    out, inn = M.pack_graph(g)
    for v in range(40):
        for x in range(40):
            c = g.code(v, x)
            assert ((int(out[v]) >> x) & 1) == (c & 1)
            assert ((int(inn[v]) >> x) & 1) == ((c >> 1) & 1)


@pytest.mark.parametrize("n,words", [(65, 2), (128, 2), (129, 3), (200, 4), (255, 4)])
def test_pack_graph_words_rows(n, words):
    # multi-word rows of the wide kernels: bit x%64 of word x//64
    g = M.random_graph(n, 0.3, 50000 + n, directed=True, label_count=3)
    out, inn = M.pack_graph_words(g, words)
    assert out.shape == (n, words) and inn.shape == (n, words)
    codes = g.codes
    for v in range(0, n, 7):
        for x in range(n):
            c = int(codes[v, x])
            assert ((int(out[v, x // 64]) >> (x % 64)) & 1) == (c & 1)
            assert ((int(inn[v, x // 64]) >> (x % 64)) & 1) == ((c >> 1) & 1)
    with pytest.raises(M.GraphError):
        M.pack_graph_words(g, (n + 63) // 64 - 1)  # row too narrow


def test_graph_size_limits():
    # n <= 255 (vertex ids, class counts and bounds are bytes, like the
    # reference's byte-frame engine: K254 accepted / K255 rejected there,
    # test_engine_iterative.cpp:40-59); n = 256 is rejected before any launch
    g = M.random_graph(256, 0.1, 3)
    with pytest.raises(M.GraphError, match="255"):
        M.solve(g, g)
    with pytest.raises(M.GraphError, match="255"):
        M.pack_graph_words(g, 4)


def test_engine_spec_grammar():
    assert M.parse_engine_spec("parallel:4").workers == 4
    assert M.parse_engine_spec("jump:double").jump == M.JumpMode.doubling
    assert M.parse_engine_spec("restarts:7").restart_seed == 7
    s = M.parse_engine_spec("goal+order=block+deadend=rel:2.5")
    assert s.goal_directed and s.order == M.OrderingStrategy.block_triangular and s.deadend == ("rel", 2.5)
    assert s.name() == "goal+order=block+deadend=rel:2.5"
    for bad in ("warp", "recursive+order=random", "recursive+foo=1", "recursive+deadend=x"):
        with pytest.raises(M.GraphError):
            M.parse_engine_spec(bad)


@pytest.mark.skipif(M.device_count() > 0, reason="a CUDA device is present")
def test_no_cpu_fallback_without_device():
    g = M.random_graph(8, 0.5, 1)
    with pytest.raises(M.GraphError):
        M.solve(g, g)
    with pytest.raises(M.GraphError):
        M.solve_batch([(g, g)])
