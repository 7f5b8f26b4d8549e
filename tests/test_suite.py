"""Benchmark-suite layer (bench.hpp / bench.cpp formats), after the
reference's tests/test_bench.cpp."""
import pytest

import paper_1908_06418_b200 as M
from paper_1908_06418_b200 import suite as S


def test_manifest_loading_resolves_the_dataset_root(tmp_path):
    m = tmp_path / "manifest.txt"
    m.write_text("# comment line\na.g b.g mcs30\nc.g d.g\n")
    specs = S.load_manifest(str(m), "/data")
    assert len(specs) == 2
    assert specs[0].g_path == "/data/a.g" and specs[0].h_path == "/data/b.g"
    assert specs[0].category == "mcs30" and specs[0].id == "a__b"
    assert specs[1].category == "uncategorized"
    bad = tmp_path / "bad.txt"
    bad.write_text("only_one.g\n")
    with pytest.raises(M.GraphError):
        S.load_manifest(str(bad))


def test_csv_round_trips_losslessly():
    a = S.InstanceRecord("x__y", "mcs50", 12, 13, "recursive", "optimal", 7, 0.12345678901234567, 0.25,
                         987654321, 17)
    b = S.InstanceRecord(pair_id="p__q", category="bvg", engine="iterative", status="error")
    csv = S.emit_csv([a, b])
    assert csv.startswith("pair_id,category,n_g,n_h,engine,status,size,wall_s,cpu_s,recursions,seed\n")
    parsed = S.parse_csv(csv)
    assert parsed == [a, b]
    assert S.emit_csv(parsed) == csv
    with pytest.raises(M.GraphError):
        S.parse_csv("hdr\n1,2,3\n")


def test_cactus_curves_are_monotone_and_skip_timeouts():
    def rec(engine, status, wall):
        return S.InstanceRecord(engine=engine, status=status, wall_seconds=wall, size=1)
    assert S.emit_cactus([rec("a", "timeout", 1)]) == []
    pts = S.emit_cactus([rec("a", "optimal", 3), rec("a", "optimal", 1), rec("a", "optimal", 2),
                         rec("b", "optimal", 5), rec("b", "timeout", 9)])
    assert [(p.engine, p.threshold_seconds, p.solved) for p in pts] == [
        ("a", 1, 1), ("a", 2, 2), ("a", 3, 3), ("b", 5, 1)]
    assert S.cactus_csv(pts).startswith("engine,threshold_s,solved")


@pytest.mark.gpu
def test_run_suite_records_and_load_errors(tmp_path):
    g, h = M.random_graph(7, 0.5, 1), M.random_graph(7, 0.5, 2)
    M.save_graph_file(g, str(tmp_path / "g.mivia"), "mivia")
    M.save_graph_file(h, str(tmp_path / "h.mivia"), "mivia")
    (tmp_path / "broken.g").write_text("not a graph")
    (tmp_path / "manifest.txt").write_text("g.mivia h.mivia cat\nbroken.g h.mivia cat\n")
    cfg = S.SuiteConfig(engines=["recursive", "gpu", "parallel:4"], budget_seconds=10)
    recs = S.run_suite(S.load_manifest(str(tmp_path / "manifest.txt"), str(tmp_path)), cfg)
    assert len(recs) == 6
    import oracle as O
    expect = O.bruteforce(O.G(7, g.codes.copy()), O.G(7, h.codes.copy()))[0]
    for r in recs[:3]:
        assert r.status == "optimal" and r.size == expect and r.n_g == 7
    assert all(r.status == "error" and r.size == -1 for r in recs[3:])
    assert S.parse_csv(S.emit_csv(recs)) == recs
    zero = S.run_suite(S.load_manifest(str(tmp_path / "manifest.txt"), str(tmp_path)),
                       S.SuiteConfig(engines=["recursive"], budget_seconds=0))
    assert zero[0].status == "timeout"
