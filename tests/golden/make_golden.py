"""Generates tests/golden/*.json from the UNMODIFIED reference solver.

Runs in the dev container only (needs oracle/_ref/libmcs_ref.so, built from
/root/reference/proj/src by oracle/Makefile). The JSON fixtures it writes are
committed; tests on the GPU box read them without the reference.

    python tests/golden/make_golden.py [small|c2|c5|c3|all|c5full|c4|restarts]
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle as O  # noqa: E402

DENS = (0.2, 0.5, 0.8)


def random_pairs(count, n_lo, n_hi, seed0):
    """test_util.hpp:30-40."""
    out = []
    for i in range(count):
        n = n_lo + (i % (n_hi - n_lo + 1) if n_hi > n_lo else 0)
        out.append((n, DENS[i % 3], seed0 + 977 * i))
    return out


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name)


def run(g, h, spec="recursive", budget=1e9):
    r = O.ref_run_engine(g, h, spec, budget)
    return {"status": r.status, "size": r.size, "nodes": r.nodes, "probes": r.probes,
            "pairs": [list(p) for p in r.pairs]}


def small():
    out = {}
    # config-1 seeds: G = random_graph(20,.3,s), H = random_graph(20,.3,s+1)
    out["config1"] = []
    for s in (1, 3, 5, 7, 9):
        g, h = O.ref_random_graph(20, 0.3, s), O.ref_random_graph(20, 0.3, s + 1)
        out["config1"].append({"seed": s, **run(g, h)})
    # acceptance corpus (acceptance_main.cpp:53): brute-force sizes + solve() node counts
    out["acceptance"] = []
    for n, d, s in random_pairs(500, 4, 9, 20260801):
        g, h = O.ref_random_graph(n, d, s), O.ref_random_graph(n, d, s + 1)
        rr = run(g, h)
        out["acceptance"].append({"n": n, "d": d, "seed": s, "bf": O.ref_bruteforce(g, h),
                                  "size": rr["size"], "nodes": rr["nodes"], "pairs": rr["pairs"]})
    # directed / labelled (test_engine_recursive.cpp:41-58 shapes, larger n)
    out["kinds"] = []
    for s in range(1, 21):
        for directed, labels in ((True, 0), (False, 2), (True, 3)):
            n = 9 + s % 6
            g = O.ref_random_graph(n, 0.5, s, directed, labels)
            h = O.ref_random_graph(n, 0.5, s + 500, directed, labels)
            out["kinds"].append({"n": n, "seed": s, "seed_h": s + 500, "directed": directed,
                                 "labels": labels, **run(g, h)})
    # goal-directed / bound jump node + probe counts
    out["probes"] = []
    for n, d, s in random_pairs(30, 4, 11, 555):
        g, h = O.ref_random_graph(n, d, s), O.ref_random_graph(n, d, s + 1)
        rec = {"n": n, "d": d, "seed": s, "goal": run(g, h, "goal")}
        for dbl in (0, 1):
            for cb in (0, 2):
                j = O.ref_bound_jump(g, h, cb, dbl)
                rec[f"jump_{dbl}_{cb}"] = {"size": j.size, "nodes": j.nodes, "probes": j.probes}
        out["probes"].append(rec)
    # orderings (heuristics.cpp:30-101) and ordered solves
    out["orderings"] = []
    for s in range(1, 13):
        g = O.ref_random_graph(9 + s, 0.4, s)
        h = O.ref_random_graph(9 + s, 0.4, s + 77)
        rec = {"n": 9 + s, "seed": s, "seed_h": s + 77}
        for o, nm in ((1, "degree"), (2, "components"), (3, "block")):
            rec[f"perm_{nm}"] = O.ref_ordering(g, o).tolist()
            rec[f"solve_{nm}"] = run(g, h, f"recursive+order={nm}")
        out["orderings"].append(rec)
    # disable_pruning enumeration counts (acceptance criterion 3/4 shape)
    out["exhaustive"] = []
    for n, d, s in random_pairs(20, 4, 7, 4321):
        g, h = O.ref_random_graph(n, d, s), O.ref_random_graph(n, d, s + 1)
        r = O.ref_run_engine(g, h, "recursive", 1e9, disable_pruning=True)
        out["exhaustive"].append({"n": n, "d": d, "seed": s, "size": r.size, "nodes": r.nodes})
    # KATs from the reference's own tests
    diamond = O.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3)])
    k4 = O.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
    k3 = O.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    c4 = O.from_edges(4, [(0, 1), (1, 2), (2, 3), (0, 3)])
    p2 = O.from_edges(2, [(0, 1)])
    p3 = O.from_edges(3, [(0, 1), (1, 2)])
    kat = {}
    kat["diamond_k4"] = run(diamond, k4)
    kat["k3_c4"] = run(k3, c4)
    kat["p2_p3"] = run(p2, p3)
    kat["p3_k3_goal"] = run(p3, k3, "goal")
    j = O.ref_bound_jump(p3, k3, 1, 0)
    kat["p3_k3_jump_plus1_from1"] = {"size": j.size, "probes": j.probes}
    g7 = O.ref_random_graph(7, 0.4, 99)
    kat["rg7_self"] = run(g7, g7)
    chain = []
    for k in range(4):
        cls, b = O.ref_refine_chain(diamond, k4, [(0, 1), (1, 2), (2, 0)][:k])
        chain.append({"classes": [[l, r, a] for l, r, a in cls], "bound": b})
    kat["refine_chain_diamond_k4"] = chain
    dg = O.from_edges(5, [(0, 1, 1), (0, 2, 2), (0, 3, 3)], directed=True)
    cls, b = O.ref_refine_chain(dg, dg, [(0, 0)])
    kat["refine_directed_4way"] = {"classes": [[l, r, a] for l, r, a in cls], "bound": b}
    out["kat"] = kat
    # graph generator fingerprints (graph.cpp:136-161)
    out["generator"] = []
    for (n, p, s, dr, L) in ((20, 0.3, 1, False, 0), (30, 0.5, 32000, False, 0), (40, 0.3, 40002, True, 4),
                             (45, 0.5, 45000, False, 0), (12, 0.5, 9, True, 3), (64, 0.9, 3, False, 0)):
        g = O.ref_random_graph(n, p, s, dr, L)
        out["generator"].append({"n": n, "p": p, "seed": s, "directed": dr, "labels": L,
                                 "codes_hex": bytes(g.codes.reshape(-1).tolist()).hex(),
                                 "vlabels": None if g.labels is None else g.labels.tolist()})
    dump("small.json", out)


def _c2_one(i):
    k, j = i % 3, i // 3
    p = (0.1, 0.3, 0.5)[k]
    s = 30000 + 1000 * k + 2 * j
    g, h = O.ref_random_graph(30, p, s), O.ref_random_graph(30, p, s + 1)
    t0 = time.time()
    r = O.ref_solve_parallel(g, h, workers=2, part_level=5, budget=3600)
    return i, r.status, r.size, r.nodes, time.time() - t0


def c2():
    out = {"sizes": {}, "status": {}, "pool_nodes": {}, "pool_seconds": {},
           "how": "reference solve_parallel(workers=2, part_level=5) per pair, 4 pairs at a time"}
    with ProcessPoolExecutor(4) as ex:
        for i, st, sz, nodes, secs in ex.map(_c2_one, range(100)):
            out["sizes"][i] = sz
            out["status"][i] = st
            out["pool_nodes"][i] = nodes
            out["pool_seconds"][i] = round(secs, 3)
            print(i, st, sz, nodes, round(secs, 2), flush=True)
    dump("c2_sizes.json", out)


def _c5_one(i):
    n = 16 + (i // 3) % 9
    p = (0.1, 0.3, 0.5)[i % 3]
    g, h = O.ref_random_graph(n, p, 50000 + 2 * i), O.ref_random_graph(n, p, 50001 + 2 * i)
    r = O.ref_run_engine(g, h, "recursive", 600)
    return i, n, p, r.status, r.size, r.nodes


def c5(count=300):
    out = {"pairs": []}
    with ProcessPoolExecutor(8) as ex:
        for i, n, p, st, sz, nodes in ex.map(_c5_one, range(count)):
            out["pairs"].append({"i": i, "n": n, "p": p, "status": st, "size": sz, "nodes": nodes})
    dump("c5_sample.json", out)


def floor():
    """Size-floor semantics (SolveConfig::shared_bound, search_core.hpp:21-36):
    sequential solve() with floors below, at and above the optimum."""
    out = []
    for n, d, s in random_pairs(24, 8, 20, 7070):
        g, h = O.ref_random_graph(n, d, s), O.ref_random_graph(n, d, s + 1)
        opt = O.ref_run_engine(g, h, "recursive").size
        for f in sorted({0, max(opt - 2, 0), max(opt - 1, 0), opt, opt + 1}):
            r = O.ref_solve_floor(g, h, f)
            out.append({"n": n, "d": d, "seed": s, "floor": f, "opt": opt, "status": r.status, "size": r.size,
                        "nodes": r.nodes, "pairs": [list(p) for p in r.pairs]})
    dump("floor.json", {"cases": out})


def deadend():
    """Dead-end handling (DeadEndMonitor / deadend_check, heuristics.cpp:103-112;
    forecast-then-jump, portfolio.cpp:136-155): monitored solves with and
    without a jump, absolute and relative policies. recursions, probes and
    deadend_suspects are deterministic (sequential engines)."""
    out = []
    specs = ["recursive+deadend=abs:50", "recursive+deadend=rel:1.5", "jump:plus1+deadend=abs:200",
             "jump:double+deadend=abs:1000", "jump:plus1+deadend=rel:2", "jump:double+deadend=rel:0.5",
             "jump:plus1+deadend=abs:0", "recursive+deadend=abs:0"]
    for n, d, s in random_pairs(16, 8, 22, 6060):
        g, h = O.ref_random_graph(n, d, s), O.ref_random_graph(n, d, s + 1)
        for spec in specs:
            r = O.ref_run_engine(g, h, spec)
            out.append({"n": n, "d": d, "seed": s, "spec": spec, "status": r.status, "size": r.size,
                        "nodes": r.nodes, "probes": r.probes, "suspects": r.extra["deadend_suspects"],
                        "pairs": [list(p) for p in r.pairs]})
    dump("deadend.json", {"cases": out})


def restarts():
    """solve_with_restarts (restarts.cpp:195-246) through the reference's own
    RestartConfig: seeded segment draws, recursions, restarts, visited ranges
    (and the ranges themselves, the VisitedRanges sink, for the smaller runs).
    The cases follow the reference's restart tests (test_heuristics.cpp:
    131-208: random_pairs(40,4,9,454) with seed 1+13i; (10,4,6,999) eager and
    exhaustive; (12,.5,71/72) seed 5 multiplier 1) plus config-1 pairs, orderings,
    directed/labelled pairs and n_H > 32 / n_H > 64 shapes."""
    cases = []
    for i, (n, d, s) in enumerate(random_pairs(40, 4, 9, 454)):
        cases.append(dict(n=n, d=d, seed=s, rseed=1 + 13 * i, mult=2.0, prune=True, order=0))
    for n, d, s in random_pairs(10, 4, 6, 999):
        cases.append(dict(n=n, d=d, seed=s, rseed=s, mult=1.0, prune=False, order=0))
    cases.append(dict(n=12, d=0.5, seed=71, rseed=5, mult=1.0, prune=True, order=0))
    for s in (1, 3, 5, 7, 9):
        cases.append(dict(n=20, d=0.3, seed=s, rseed=7 * s, mult=2.0, prune=True, order=0))
        cases.append(dict(n=20, d=0.3, seed=s, rseed=s, mult=1.0, prune=True, order=1 + s % 3))
        cases.append(dict(n=20, d=0.3, seed=s, rseed=3, mult=0.0, prune=True, order=0))
    for i, (n, d, s) in enumerate(random_pairs(12, 10, 16, 8080)):
        cases.append(dict(n=n, d=d, seed=s, rseed=100 + i, mult=0.5 + 0.5 * (i % 4), prune=True, order=0,
                          directed=i % 2 == 1, labels=(0, 2, 3)[i % 3]))
    for i, (n, nh, d) in enumerate(((11, 36, 0.3), (12, 40, 0.5), (12, 34, 0.8), (11, 70, 0.5))):
        # n_H > 32 / > 64: the 64-bit and 128-bit kernels
        cases.append(dict(n=n, nh=nh, d=d, seed=9000 + i, rseed=17 + i, mult=1.0, prune=True, order=0))
    out = []
    for c in cases:
        dr, lb = c.get("directed", False), c.get("labels", 0)
        g = O.ref_random_graph(c["n"], c["d"], c["seed"], dr, lb)
        h = O.ref_random_graph(c.get("nh", c["n"]), c["d"], c["seed"] + 1, dr, lb)
        r = O.ref_solve_with_restarts(g, h, c["rseed"], c["mult"], c["prune"], c["order"])
        assert r.status == 0, c
        rec = dict(c, size=r.size, nodes=r.nodes, restarts=r.extra["restarts"],
                   visited_ranges=r.extra["visited_ranges"], pairs=[list(p) for p in r.pairs])
        if r.extra["visited_ranges"] <= 400:
            rec["ranges"] = [[[x for _, x in lo], [x for _, x in hi]] for lo, hi in r.extra["ranges"]]
        out.append(rec)
        print("restarts", c["n"], c["d"], c["seed"], r.size, r.nodes, r.extra["restarts"],
              r.extra["visited_ranges"], flush=True)
    dump("restarts.json", {"cases": out, "how": "reference solve_with_restarts (oracle/_ref) with the "
                           "VisitedRanges sink; ranges as iteration lists per key"})


def c3_pairs():
    """C3 (BASELINE configs[2]): directed vertex-labelled ER n=40,
    L in {2,4,8} x p in {.1,.3,.5} x 10 pairs, seeds 40000+2i / 40001+2i."""
    out = []
    i = 0
    for L in (2, 4, 8):
        for p in (0.1, 0.3, 0.5):
            for _ in range(10):
                out.append((i, L, p))
                i += 1
    return out


def _c3_one(args):
    i, L, p = args
    g = O.ref_random_graph(40, p, 40000 + 2 * i, True, L)
    h = O.ref_random_graph(40, p, 40001 + 2 * i, True, L)
    t0 = time.time()
    r = O.ref_solve_parallel(g, h, workers=2, part_level=5, budget=7200)
    return i, L, p, r.status, r.size, r.nodes, time.time() - t0


def c3():
    out = {"pairs": [], "how": "reference solve_parallel(workers=2, part_level=5) per pair, 4 pairs at a time"}
    with ProcessPoolExecutor(4) as ex:
        for i, L, p, st, sz, nodes, secs in ex.map(_c3_one, c3_pairs()):
            out["pairs"].append({"i": i, "labels": L, "p": p, "status": st, "size": sz,
                                 "pool_nodes": nodes, "pool_seconds": round(secs, 3)})
            print("c3", i, L, p, st, sz, nodes, round(secs, 2), flush=True)
    assert all(r["status"] == 0 for r in out["pairs"])
    dump("c3_sizes.json", out)


def _c5_full_one(i):
    n = 16 + (i // 3) % 9
    p = (0.1, 0.3, 0.5)[i % 3]
    g, h = O.ref_random_graph(n, p, 50000 + 2 * i), O.ref_random_graph(n, p, 50001 + 2 * i)
    r = O.ref_run_engine(g, h, "recursive", 120)
    eng = "recursive"
    if r.status != 0:  # the rare long pair: the reference pool proves it
        r = O.ref_solve_parallel(g, h, workers=2, part_level=5, budget=7200)
        eng = "parallel:2"
    return i, r.status, r.size, r.nodes, eng


def c5_full(count=10000):
    """All 10,000 C5 optima; compact form (sizes as one string of bytes)."""
    sizes = [0] * count
    nodes = [0] * count
    eng = {}
    with ProcessPoolExecutor(8) as ex:
        for i, st, sz, nd, e in ex.map(_c5_full_one, range(count), chunksize=16):
            assert st == 0, (i, st)
            sizes[i] = sz
            nodes[i] = nd
            if e != "recursive":
                eng[i] = e
            if i % 500 == 0:
                print("c5", i, sz, nd, flush=True)
    dump("c5_sizes.json", {"count": count, "sizes": "".join(chr(ord("A") + s) for s in sizes),
                           "size_encoding": "chr(ord('A') + size) per pair i",
                           "nodes": nodes, "engine_overrides": eng,
                           "how": "reference solve() (recursive, sequential node counts); "
                                  "pairs it does not prove in 120 s go to solve_parallel"})


def c4():
    """C4 (n=45, p=0.5, seeds 45000/45001). The reference pool with a floor of
    16 timed out after 6 h (its part_level-5 tail ran on one thread), so the
    proof of "no 17" runs the reference's own sequential solve() with a
    SharedBound floor on each of the 541 pieces of a decomposition at the top
    of its search tree, in parallel and resumably (tools/c4_split_proof.py ->
    tests/golden/c4_pieces.jsonl); tools/c4_proof_json.py adds the GPU's
    16-mapping accepted by the reference's oracle::verify and writes
    c4_proof.json (tests/test_c4_proof.py checks the decomposition identity
    and the ledger's coverage)."""
    here = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    subprocess.run([sys.executable, os.path.join(here, "tools", "c4_split_proof.py"), "12"], check=True)
    subprocess.run([sys.executable, os.path.join(here, "tools", "c4_proof_json.py"), "12"], check=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libmcs_ref.so missing: make -C oracle ref")
    if what in ("small", "all"):
        small()
    if what in ("c5", "all"):
        c5()
    if what in ("c2", "all"):
        c2()
    if what in ("c3", "all"):
        c3()
    if what == "c5full":
        c5_full()
    if what in ("floor", "all"):
        floor()
    if what in ("deadend", "all"):
        deadend()
    if what == "c4":
        c4()
    if what in ("restarts", "all"):
        restarts()
