"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two libraries live here:

* ``libmcs_oracle.so`` — the plain-C restatement of the reference solver
  (``mcs_oracle.c``; each function cites the reference file:line it follows).
* ``_ref/libmcs_ref.so`` — the UNMODIFIED reference (``/root/reference/proj/src``)
  compiled by ``oracle/Makefile`` together with the extern "C" shim
  ``ref_shim.cpp``. Built in the dev container; the prebuilt ``.so`` travels to the
  GPU box (``/root/reference`` does not exist there).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package. The product package
``paper_1908_06418_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmcs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmcs_ref.so")
REF_SRC = "/root/reference/proj/src"


def build(ref: bool = True) -> None:
    """Compile the C oracle and, when the reference sources are present, oracle/_ref."""
    subprocess.check_call(["make", "-s", "-C", HERE, "libmcs_oracle.so"])
    if ref and os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


class _OrcGraph(C.Structure):
    _fields_ = [("n", C.c_int32), ("directed", C.c_int32),
                ("codes", C.POINTER(C.c_uint8)), ("labels", C.POINTER(C.c_int32))]


class _OrcOptions(C.Structure):
    _fields_ = [("budget_s", C.c_double), ("goal", C.c_int64), ("prune", C.c_int32),
                ("order", C.c_int32), ("floor_size", C.c_int64),
                ("cancel", C.POINTER(C.c_int32))]


class _OrcResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("size", C.c_int32), ("pairs", C.c_int32 * 512),
                ("nodes", C.c_uint64), ("probes", C.c_uint64), ("wall_s", C.c_double),
                ("sum_classes", C.c_uint64), ("sum_splits", C.c_uint64),
                ("pruned_at_entry", C.c_uint64), ("children_built", C.c_uint64),
                ("max_depth", C.c_int32), ("max_stack_classes", C.c_int32)]


class _RefResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("size", C.c_int32), ("pairs", C.c_int32 * 512),
                ("recursions", C.c_uint64), ("probes", C.c_uint64), ("restarts", C.c_uint64),
                ("visited_ranges", C.c_uint64), ("tasks_published", C.c_uint64),
                ("double_executions", C.c_uint64), ("wall_seconds", C.c_double),
                ("error", C.c_char * 256), ("deadend_suspects", C.c_uint64)]


@dataclass
class G:
    """A graph in the reference's layout: n*n row-major uint8 codes (graph.hpp:60)."""
    n: int
    codes: np.ndarray               # (n, n) uint8
    directed: bool = False
    labels: np.ndarray | None = None  # (n,) int32

    def c_struct(self):
        codes = np.ascontiguousarray(self.codes, dtype=np.uint8).reshape(-1)
        if codes.size == 0:
            codes = np.zeros(1, np.uint8)
        labels = None
        if self.labels is not None:
            labels = np.ascontiguousarray(self.labels, dtype=np.int32)
            if labels.size == 0:
                labels = np.zeros(1, np.int32)
        s = _OrcGraph(self.n, int(self.directed), codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                      labels.ctypes.data_as(C.POINTER(C.c_int32)) if labels is not None
                      else C.POINTER(C.c_int32)())
        s._keep = (codes, labels)
        return s


@dataclass
class Result:
    status: int
    size: int
    pairs: list = field(default_factory=list)
    nodes: int = 0
    probes: int = 0
    wall_s: float = 0.0
    extra: dict = field(default_factory=dict)


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        P = C.POINTER
        lib.orc_random_graph.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                         P(C.c_uint8), P(C.c_int32)]
        lib.orc_random_permutation.argtypes = [C.c_int, C.c_uint64, P(C.c_int32)]
        lib.orc_ordering.argtypes = [P(_OrcGraph), C.c_int, P(C.c_int32)]
        lib.orc_degree.argtypes = [P(_OrcGraph), C.c_int]
        for fn in ("orc_solve", "orc_solve_goal_directed"):
            getattr(lib, fn).argtypes = [P(_OrcGraph), P(_OrcGraph), P(_OrcOptions), P(_OrcResult)]
        lib.orc_bound_jump.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_int, C.c_int,
                                       P(_OrcOptions), P(_OrcResult)]
        lib.orc_verify.argtypes = [P(_OrcGraph), P(_OrcGraph), P(C.c_int32), C.c_int]
        lib.orc_solve_with_restarts.argtypes = [P(_OrcGraph), P(_OrcGraph), P(_OrcOptions), C.c_uint64,
                                                C.c_double, P(_OrcResult), P(C.c_uint64), P(C.c_int32),
                                                C.c_int64, P(C.c_int64)]
        lib.orc_bruteforce.argtypes = [P(_OrcGraph), P(_OrcGraph), P(C.c_int32)]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} not built (make -C oracle ref)")
        lib = C.CDLL(REF_SO)
        P = C.POINTER
        lib.ref_random_graph.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                         P(C.c_uint8), P(C.c_int32)]
        lib.ref_random_permutation.argtypes = [C.c_int, C.c_uint64, P(C.c_int32)]
        lib.ref_run_engine.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_char_p, C.c_double,
                                       C.c_int, P(_RefResult)]
        lib.ref_solve_parallel.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_int, C.c_int,
                                           C.c_double, P(_RefResult)]
        lib.ref_bound_jump.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_int, C.c_int, C.c_double,
                                       P(_RefResult)]
        lib.ref_solve_floor.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_int, C.c_double, P(_RefResult)]
        lib.ref_solve_parallel_floor.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_int, C.c_int,
                                                 C.c_double, C.c_int, P(_RefResult)]
        lib.ref_verify.argtypes = [P(_OrcGraph), P(_OrcGraph), P(C.c_int32), C.c_int]
        lib.ref_solve_with_restarts.argtypes = [P(_OrcGraph), P(_OrcGraph), C.c_uint64, C.c_double, C.c_int,
                                                C.c_int, C.c_double, P(_RefResult), P(C.c_int32), C.c_int64,
                                                P(C.c_int64)]
        lib.ref_bruteforce.argtypes = [P(_OrcGraph), P(_OrcGraph), P(C.c_int32)]
        lib.ref_ordering.argtypes = [P(_OrcGraph), C.c_int, P(C.c_int32)]
        lib.ref_refine_chain.argtypes = [P(_OrcGraph), P(_OrcGraph), P(C.c_int32), C.c_int,
                                         P(C.c_uint64), P(C.c_uint64), P(C.c_int32), C.c_int,
                                         P(C.c_int64)]
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


# ----------------------------------------------------------------- oracle API
def random_graph(n, density, seed, directed=False, label_count=0) -> G:
    """random_graph (graph.cpp:136-161), restated in C (bit-identical mt19937 draws)."""
    codes = np.zeros((max(n, 1), max(n, 1)), np.uint8)
    labels = np.zeros(max(n, 1), np.int32)
    orc_lib().orc_random_graph(n, density, seed, int(directed), label_count,
                               codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                               labels.ctypes.data_as(C.POINTER(C.c_int32)))
    return G(n, codes[:n, :n].copy(), directed, labels[:n].copy() if label_count > 0 else None)


def random_permutation(n, seed):
    f = np.zeros(max(n, 1), np.int32)
    orc_lib().orc_random_permutation(n, seed, f.ctypes.data_as(C.POINTER(C.c_int32)))
    return f[:n].copy()


def from_edges(n, edges, directed=False, labels=None) -> G:
    """from_edge_list (graph.cpp:39-71) for test fixtures: (u, v[, code]) tuples."""
    codes = np.zeros((n, n), np.uint8)
    for e in edges:
        u, v = e[0], e[1]
        c = e[2] if (directed and len(e) > 2) else 1
        if u == v or not (0 <= u < n and 0 <= v < n):
            raise ValueError("bad edge")
        mir = {1: 2, 2: 1, 3: 3}[c] if directed else 1
        codes[u, v] = c
        codes[v, u] = mir
    return G(n, codes, directed, None if labels is None else np.asarray(labels, np.int32))


def _opts(budget=1e9, goal=0, prune=True, order=0, floor_size=0):
    return _OrcOptions(budget, goal, int(prune), order, floor_size, C.POINTER(C.c_int32)())


def _res(r: _OrcResult) -> Result:
    k = r.size
    pairs = [(r.pairs[2 * i], r.pairs[2 * i + 1]) for i in range(k)]
    return Result(r.status, r.size, pairs, r.nodes, r.probes, r.wall_s,
                  dict(sum_classes=r.sum_classes, sum_splits=r.sum_splits,
                       pruned_at_entry=r.pruned_at_entry, children_built=r.children_built,
                       max_depth=r.max_depth, max_stack_classes=r.max_stack_classes))


def solve(g: G, h: G, budget=1e9, prune=True, order=0, floor_size=0) -> Result:
    """Sequential mcs::solve restated (solve.cpp:85-129); nodes == stats.recursions."""
    r = _OrcResult()
    gs, hs = g.c_struct(), h.c_struct()
    if orc_lib().orc_solve(C.byref(gs), C.byref(hs), C.byref(_opts(budget, 0, prune, order, floor_size)),
                           C.byref(r)) != 0:
        raise ValueError("oracle: invalid graph pair")
    return _res(r)


def solve_goal_directed(g: G, h: G, budget=1e9, order=0) -> Result:
    r = _OrcResult()
    gs, hs = g.c_struct(), h.c_struct()
    if orc_lib().orc_solve_goal_directed(C.byref(gs), C.byref(hs), C.byref(_opts(budget, order=order)),
                                         C.byref(r)) != 0:
        raise ValueError("oracle: invalid graph pair")
    return _res(r)


def bound_jump(g: G, h: G, current_best=0, doubling=False, budget=1e9, order=0) -> Result:
    r = _OrcResult()
    gs, hs = g.c_struct(), h.c_struct()
    if orc_lib().orc_bound_jump(C.byref(gs), C.byref(hs), current_best, int(doubling),
                                C.byref(_opts(budget, order=order)), C.byref(r)) != 0:
        raise ValueError("oracle: invalid graph pair")
    return _res(r)


def decode_ranges(words):
    """[len(lo), lo..., len(hi), hi...] runs -> [(lo, hi)] PositionKeys as
    lists of (depth, iteration) pairs (heuristics.hpp:77)."""
    keys, i = [], 0
    while i < len(words):
        k = int(words[i])
        keys.append([(d, int(words[i + 1 + d])) for d in range(k)])
        i += 1 + k
    return [(keys[j], keys[j + 1]) for j in range(0, len(keys), 2)]


def _words(call):
    """Runs call(buf, cap, len_ptr) with a growing buffer; returns the words."""
    cap = 1 << 16
    while True:
        buf = (C.c_int32 * cap)()
        need = C.c_int64(0)
        call(buf, cap, C.byref(need))
        if need.value <= cap:
            return list(buf[:need.value])
        cap = need.value


def solve_with_restarts(g: G, h: G, seed=1, multiplier=2.0, prune=True, order=0, budget=1e9, floor_size=0):
    """solve_with_restarts restated (restarts.cpp:195-246): Result with
    extra restarts / visited_ranges / ranges."""
    gs, hs = g.c_struct(), h.c_struct()
    out = {}

    def call(buf, cap, need):
        r = _OrcResult()
        rs = C.c_uint64(0)
        if orc_lib().orc_solve_with_restarts(C.byref(gs), C.byref(hs), C.byref(_opts(budget, 0, prune, order,
                                                                                      floor_size)),
                                             seed, multiplier, C.byref(r), C.byref(rs), buf, cap, need) != 0:
            raise ValueError("oracle: invalid graph pair")
        out["r"], out["restarts"] = r, rs.value

    words = _words(call)
    r = out["r"]
    res = Result(r.status, r.size, [(r.pairs[2 * i], r.pairs[2 * i + 1]) for i in range(r.size)], r.nodes, 0,
                 r.wall_s)
    res.extra = dict(restarts=out["restarts"], visited_ranges=int(r.probes), ranges=decode_ranges(words))
    return res


def ref_solve_with_restarts(g: G, h: G, seed=1, multiplier=2.0, prune=True, order=0, budget=1e9) -> Result:
    """The unmodified reference's solve_with_restarts (with the VisitedRanges sink)."""
    gs, hs = g.c_struct(), h.c_struct()
    out = {}

    def call(buf, cap, need):
        r = _RefResult()
        ref_lib().ref_solve_with_restarts(C.byref(gs), C.byref(hs), seed, multiplier, int(not prune), order,
                                          budget, C.byref(r), buf, cap, need)
        out["r"] = r

    words = _words(call)
    res = _ref_res(out["r"])
    res.extra["ranges"] = decode_ranges(words)
    return res


def ordering(g: G, strategy: int):
    f = np.zeros(max(g.n, 1), np.int32)
    gs = g.c_struct()
    orc_lib().orc_ordering(C.byref(gs), strategy, f.ctypes.data_as(C.POINTER(C.c_int32)))
    return f[:g.n].copy()


def degree(g: G, v: int) -> int:
    gs = g.c_struct()
    return orc_lib().orc_degree(C.byref(gs), v)


def verify(g: G, h: G, pairs) -> bool:
    flat, p = _i32(np.asarray(pairs, np.int32).reshape(-1) if len(pairs) else np.zeros(1, np.int32))
    gs, hs = g.c_struct(), h.c_struct()
    rc = orc_lib().orc_verify(C.byref(gs), C.byref(hs), p, len(pairs))
    if rc < 0:
        raise ValueError("verify: vertex out of range")
    return rc == 1


def bruteforce(g: G, h: G):
    out = np.zeros(64, np.int32)
    gs, hs = g.c_struct(), h.c_struct()
    k = orc_lib().orc_bruteforce(C.byref(gs), C.byref(hs), out.ctypes.data_as(C.POINTER(C.c_int32)))
    if k < 0:
        raise ValueError("bruteforce: above the practical ceiling")
    return k, [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(k)]


# -------------------------------------------------------------- reference API
def ref_random_graph(n, density, seed, directed=False, label_count=0) -> G:
    codes = np.zeros((max(n, 1), max(n, 1)), np.uint8)
    labels = np.zeros(max(n, 1), np.int32)
    if ref_lib().ref_random_graph(n, density, seed, int(directed), label_count,
                                  codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  labels.ctypes.data_as(C.POINTER(C.c_int32))) != 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return G(n, codes[:n, :n].copy(), directed, labels[:n].copy() if label_count > 0 else None)


def _ref_res(r: _RefResult) -> Result:
    if r.status < 0:
        raise ValueError(r.error.decode())
    pairs = [(r.pairs[2 * i], r.pairs[2 * i + 1]) for i in range(r.size)]
    return Result(r.status, r.size, pairs, r.recursions, r.probes, r.wall_seconds,
                  dict(restarts=r.restarts, visited_ranges=r.visited_ranges,
                       tasks_published=r.tasks_published, double_executions=r.double_executions,
                       deadend_suspects=r.deadend_suspects))


def ref_run_engine(g: G, h: G, spec="recursive", budget=1e9, disable_pruning=False) -> Result:
    r = _RefResult()
    gs, hs = g.c_struct(), h.c_struct()
    ref_lib().ref_run_engine(C.byref(gs), C.byref(hs), spec.encode(), budget, int(disable_pruning),
                             C.byref(r))
    return _ref_res(r)


def ref_solve_parallel(g: G, h: G, workers=0, part_level=5, budget=1e9) -> Result:
    r = _RefResult()
    gs, hs = g.c_struct(), h.c_struct()
    ref_lib().ref_solve_parallel(C.byref(gs), C.byref(hs), workers, part_level, budget, C.byref(r))
    return _ref_res(r)


def ref_solve_floor(g: G, h: G, floor: int, budget=1e9) -> Result:
    """solve() with SolveConfig::shared_bound seeded at `floor` (search_core.hpp:21-36)."""
    r = _RefResult()
    gs, hs = g.c_struct(), h.c_struct()
    ref_lib().ref_solve_floor(C.byref(gs), C.byref(hs), floor, budget, C.byref(r))
    return _ref_res(r)


def ref_solve_parallel_floor(g: G, h: G, floor: int, workers=0, part_level=5, budget=1e9) -> Result:
    """solve_parallel with SolveConfig::shared_bound seeded at `floor` (solve.hpp:70-81)."""
    r = _RefResult()
    gs, hs = g.c_struct(), h.c_struct()
    ref_lib().ref_solve_parallel_floor(C.byref(gs), C.byref(hs), workers, part_level, budget, floor,
                                       C.byref(r))
    return _ref_res(r)


def ref_bound_jump(g: G, h: G, current_best=0, doubling=False, budget=1e9) -> Result:
    r = _RefResult()
    gs, hs = g.c_struct(), h.c_struct()
    ref_lib().ref_bound_jump(C.byref(gs), C.byref(hs), current_best, int(doubling), budget, C.byref(r))
    return _ref_res(r)


def ref_ordering(g: G, strategy: int):
    f = np.zeros(max(g.n, 1), np.int32)
    gs = g.c_struct()
    ref_lib().ref_ordering(C.byref(gs), strategy, f.ctypes.data_as(C.POINTER(C.c_int32)))
    return f[:g.n].copy()


def ref_verify(g: G, h: G, pairs) -> int:
    flat, p = _i32(np.asarray(pairs, np.int32).reshape(-1) if len(pairs) else np.zeros(1, np.int32))
    gs, hs = g.c_struct(), h.c_struct()
    return ref_lib().ref_verify(C.byref(gs), C.byref(hs), p, len(pairs))


def ref_bruteforce(g: G, h: G) -> int:
    out = np.zeros(64, np.int32)
    gs, hs = g.c_struct(), h.c_struct()
    return ref_lib().ref_bruteforce(C.byref(gs), C.byref(hs), out.ctypes.data_as(C.POINTER(C.c_int32)))


def ref_refine_chain(g: G, h: G, pairs):
    """initial_classes + refine(...) chain (label_classes.cpp:8-39,110-142) -> classes, bound."""
    flat, p = _i32(np.asarray(pairs, np.int32).reshape(-1) if len(pairs) else np.zeros(1, np.int32))
    L = np.zeros(64, np.uint64)
    R = np.zeros(64, np.uint64)
    A = np.zeros(64, np.int32)
    b = C.c_int64()
    gs, hs = g.c_struct(), h.c_struct()
    k = ref_lib().ref_refine_chain(C.byref(gs), C.byref(hs), p, len(pairs),
                                   L.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   R.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   A.ctypes.data_as(C.POINTER(C.c_int32)), 64, C.byref(b))
    if k < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return [(int(L[i]), int(R[i]), bool(A[i])) for i in range(k)], int(b.value)
