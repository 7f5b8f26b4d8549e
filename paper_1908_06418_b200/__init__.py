"""B200-native McSplit: Python mirror of the reference solver's public API.

Every call goes through the C ABI of ``libmcsg.so`` (``include/mcsg.h``), whose
solve entry points run the hand-written sm_100a search kernel. There is no CPU
fallback: without the built library or a CUDA device the solve functions raise.

Names, argument meaning and error behaviour follow the reference C++ API
(``/root/reference/proj/include/mcs``):

=========================  ===========================================
this module                reference
=========================  ===========================================
``Graph``                  ``mcs::Graph``            graph.hpp:31-62
``from_edge_list``         ``mcs::from_edge_list``   graph.hpp:66
``random_graph``           ``mcs::random_graph``     graph.hpp:99
``random_permutation``     ``mcs::random_permutation`` graph.hpp:102
``permute``                ``mcs::permute``          graph.hpp:89
``load_graph_file``        ``mcs::load_graph_file``  graph_io.hpp:33
``save_graph_file``        ``mcs::save_graph_file``  graph_io.hpp:34
``SolveConfig``            ``mcs::SolveConfig``      solve.hpp:118-125
``SolveResult``            ``mcs::SolveResult``      solve.hpp:57-66
``solve``                  ``mcs::solve``            solve.hpp:128
``solve_parallel``         ``mcs::solve_parallel``   engine_parallel.hpp:16
``solve_goal_directed``    ``mcs::solve_goal_directed`` solve.hpp:132
``bound_jump_search``      ``mcs::bound_jump_search`` heuristics.hpp:69
``make_ordering``          ``mcs::make_ordering``    heuristics.hpp:26
``parse_engine_spec``      ``mcs::parse_engine_spec`` portfolio.hpp:34
``run_engine``             ``mcs::run_engine``       portfolio.hpp:37
``run_portfolio``          ``mcs::run_portfolio``    portfolio.hpp:100
``verify``                 ``mcs::oracle::verify``   oracle.hpp:16
=========================  ===========================================
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCSG_LIB", os.path.join(HERE, "libmcsg.so"))  # override: dev experiments
MAX_N = 255

__all__ = [
    "Graph", "GraphError", "ParseError", "from_edge_list", "random_graph", "random_permutation",
    "permute", "load_graph_file", "save_graph_file", "SolveStatus", "OrderingStrategy", "JumpMode",
    "SolveConfig", "SearchStats", "SolveResult", "solve", "solve_parallel", "solve_batch",
    "solve_goal_directed", "bound_jump_search", "make_ordering", "EngineSpec", "parse_engine_spec",
    "run_engine", "PortfolioResult", "run_portfolio", "verify", "pack_graph", "lib", "device_count",
    "MODE_THROUGHPUT", "MODE_PARITY", "RestartConfig", "VisitedRanges", "solve_with_restarts",
]


class GraphError(RuntimeError):
    """mcs::GraphError (graph.hpp:25-28): invalid input or unsupported request."""


class ParseError(GraphError):
    """mcs::ParseError (graph_io.hpp:11)."""


MODE_THROUGHPUT = 0
MODE_PARITY = 1
DIRECTED = 1
LABELED = 2


class SolveStatus(enum.IntEnum):
    optimal = 0
    timeout = 2
    cancelled = 4


class OrderingStrategy(enum.IntEnum):
    none = 0
    degree_desc = 1
    components_then_degree = 2
    block_triangular = 3


class JumpMode(enum.IntEnum):
    plus_one = 0
    doubling = 1


# ------------------------------------------------------------------ C ABI --
class _Graph(C.Structure):
    _fields_ = [("n", C.c_int32), ("flags", C.c_uint32), ("codes", C.POINTER(C.c_uint8)),
                ("labels", C.POINTER(C.c_int32))]


class _Options(C.Structure):
    _fields_ = [("budget_s", C.c_double), ("order", C.c_int32), ("mode", C.c_int32),
                ("goal", C.c_int32), ("disable_pruning", C.c_int32), ("floor_size", C.c_int32),
                ("device", C.c_int32), ("max_warps", C.c_int32), ("smem_classes", C.c_int32),
                ("seed", C.c_uint64), ("cancel", C.POINTER(C.c_int32)),
                ("n_devices", C.c_int32), ("devices", C.c_int32 * 16), ("frontier", C.c_int32),
                ("deadend_abs", C.c_uint64), ("deadend_rel", C.c_double), ("deadend_jump", C.c_int32),
                ("restart_multiplier", C.c_double), ("shared_bound", C.POINTER(C.c_int32)),
                ("warp_share", C.c_int32), ("deadend_kind", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [("nodes", C.c_uint64), ("sum_classes", C.c_uint64), ("splits", C.c_uint64),
                ("split_classes", C.c_uint64), ("donations", C.c_uint64), ("tasks", C.c_uint64),
                ("spills", C.c_uint64), ("probes", C.c_uint64), ("wall_s", C.c_double),
                ("kernel_s", C.c_double), ("h2d_s", C.c_double), ("warps", C.c_int32),
                ("ctas", C.c_int32), ("smem_per_cta", C.c_int32), ("smem_classes", C.c_int32),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("launches", C.c_uint64),
                ("busy_cycles", C.c_uint64), ("idle_cycles", C.c_uint64),
                ("restarts", C.c_uint64), ("frozen", C.c_uint64), ("idle_s", C.c_double),
                ("busy_s", C.c_double), ("peer_pushes", C.c_uint64), ("visited_ranges", C.c_uint64)]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("size", C.c_int32), ("pairs", C.c_int32 * (2 * MAX_N)),
                ("nodes", C.c_uint64), ("solve_s", C.c_double), ("flags", C.c_int32),
                ("probes", C.c_int32), ("deadend_suspects", C.c_uint64)]


_lib = None


def lib():
    """Load libmcsg.so (fails loudly when it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_1908_06418_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        G, O, R, S = P(_Graph), P(_Options), P(_Result), P(_Stats)
        L.mcsg_solve.argtypes = [G, G, O, R, S]
        L.mcsg_solve_parallel.argtypes = [G, G, O, R, S]
        L.mcsg_solve_batch.argtypes = [C.c_int32, G, G, O, R, S]
        L.mcsg_solve_goal_directed.argtypes = [G, G, O, R, S]
        L.mcsg_bound_jump.argtypes = [G, G, C.c_int32, C.c_int32, O, R, S]
        L.mcsg_portfolio.argtypes = [G, G, C.c_int32, P(C.c_int32), P(C.c_uint64), O, R, P(C.c_int32), S]
        L.mcsg_probe_parallel.argtypes = [G, G, C.c_int32, C.c_int32, O, R, S]
        L.mcsg_solve_with_restarts.argtypes = [G, G, O, R, S, P(C.c_int32), C.c_int64, P(C.c_int64)]
        L.mcsg_verify.argtypes = [G, G, P(C.c_int32), C.c_int32]
        L.mcsg_random_graph.argtypes = [C.c_int32, C.c_double, C.c_uint64, C.c_uint32, C.c_int32,
                                        P(C.c_uint8), P(C.c_int32)]
        L.mcsg_random_permutation.argtypes = [C.c_int32, C.c_uint64, P(C.c_int32)]
        L.mcsg_ordering.argtypes = [G, C.c_int32, P(C.c_int32)]
        L.mcsg_load_graph_file.argtypes = [C.c_char_p, C.c_int32, P(C.c_int32), P(C.c_uint32),
                                           P(C.c_uint8), P(C.c_int32)]
        L.mcsg_save_graph_file.argtypes = [G, C.c_char_p, C.c_int32]
        L.mcsg_pack_graph.argtypes = [G, P(C.c_uint64), P(C.c_uint64)]
        L.mcsg_pack_graph_words.argtypes = [G, C.c_int32, P(C.c_uint64), P(C.c_uint64)]
        L.mcsg_last_error.restype = C.c_char_p
        L.mcsg_last_error_kind.restype = C.c_int32
        L.mcsg_abi_version.restype = C.c_int32
        L.mcsg_device_count.restype = C.c_int32
        _lib = L
    return _lib


def _err():
    msg = lib().mcsg_last_error().decode()
    if lib().mcsg_last_error_kind() == 2:  # MCSG_ERR_PARSE
        return ParseError(msg)
    return GraphError(msg)


def device_count() -> int:
    return int(lib().mcsg_device_count())


# ------------------------------------------------------------------ graphs --
class Graph:
    """Immutable graph: n*n row-major uint8 adjacency codes (graph.hpp:31-62)."""

    __slots__ = ("_n", "_codes", "_directed", "_labels", "_cs")

    def __init__(self, n: int, codes, directed: bool = False, labels=None):
        self._n = int(n)
        self._codes = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8).reshape(self._n, self._n))
        self._codes.setflags(write=False)
        self._directed = bool(directed)
        self._labels = None
        if labels is not None:
            lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
            if lab.shape != (self._n,):
                raise GraphError("label vector size does not match vertex count")
            lab.setflags(write=False)
            self._labels = lab
        self._cs = None

    def n(self) -> int:
        return self._n

    def directed(self) -> bool:
        return self._directed

    def labeled(self) -> bool:
        return self._labels is not None

    def code(self, u: int, v: int) -> int:
        return int(self._codes[u, v])

    def adjacent(self, u: int, v: int) -> bool:
        return self._codes[u, v] != 0

    def label(self, v: int) -> int:
        return int(self._labels[v])

    @property
    def codes(self) -> np.ndarray:
        return self._codes

    @property
    def labels(self):
        return self._labels

    def degree(self, v: int) -> int:
        row = self._codes[v]
        if not self._directed:
            return int(np.count_nonzero(row))
        return int(np.count_nonzero(row & 1) + np.count_nonzero(row & 2))

    def edge_count(self) -> int:
        return int(np.count_nonzero(np.triu(self._codes, 1)))

    def __eq__(self, other) -> bool:
        return (isinstance(other, Graph) and self._n == other._n and self._directed == other._directed
                and np.array_equal(self._codes, other._codes)
                and ((self._labels is None and other._labels is None)
                     or (self._labels is not None and other._labels is not None
                         and np.array_equal(self._labels, other._labels))))

    def __repr__(self) -> str:
        return (f"Graph(n={self._n}, edges={self.edge_count()}, directed={self._directed}, "
                f"labeled={self.labeled()})")

    def _c(self) -> _Graph:
        if self._cs is None:
            codes = self._codes.reshape(-1) if self._n else np.zeros(1, np.uint8)
            flags = (DIRECTED if self._directed else 0) | (LABELED if self._labels is not None else 0)
            lab = self._labels if (self._labels is not None and self._n) else (
                np.zeros(1, np.int32) if self._labels is not None else None)
            s = _Graph(self._n, flags, codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                       lab.ctypes.data_as(C.POINTER(C.c_int32)) if lab is not None
                       else C.POINTER(C.c_int32)())
            s._keep = (codes, lab)
            self._cs = s
        return self._cs


def from_edge_list(n: int, edges, directed: bool = False, labels=None) -> Graph:
    """from_edge_list (graph.hpp:66, graph.cpp:39-71): (u, v[, code]) tuples.

    Duplicates collapse; a conflicting duplicate, a self-loop, an out-of-range
    endpoint or a directed code of 0 raise GraphError.
    """
    if n < 0:
        raise GraphError("negative vertex count")
    if labels is not None and len(labels) != n:
        raise GraphError("label vector size does not match vertex count")
    codes = np.zeros((n, n), np.uint8)
    for e in edges:
        u, v = int(e[0]), int(e[1])
        c = int(e[2]) if len(e) > 2 else 1
        if not (0 <= u < n and 0 <= v < n):
            raise GraphError(f"edge endpoint out of range: ({u},{v})")
        if u == v:
            raise GraphError(f"self-loop on vertex {u}")
        if directed:
            if c == 0:
                raise GraphError("directed edge with code none")
            fwd, bwd = c, {1: 2, 2: 1, 3: 3}[c]
        else:
            fwd = bwd = 1
        if codes[u, v] not in (0, fwd):
            raise GraphError(f"conflicting duplicate edge ({u},{v})")
        codes[u, v] = fwd
        codes[v, u] = bwd
    return Graph(n, codes, directed, labels)


def random_graph(n: int, density: float, seed: int, directed: bool = False,
                 label_count: int = 0) -> Graph:
    """random_graph (graph.cpp:136-161): bit-identical mt19937 draws."""
    codes = np.zeros(max(n * n, 1), np.uint8)
    labels = np.zeros(max(n, 1), np.int32)
    rc = lib().mcsg_random_graph(n, density, seed, DIRECTED if directed else 0, label_count,
                                 codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                                 labels.ctypes.data_as(C.POINTER(C.c_int32)))
    if rc != 0:
        raise _err()
    return Graph(n, codes[: n * n], directed, labels[:n] if label_count > 0 else None)


def random_permutation(n: int, seed: int) -> np.ndarray:
    f = np.zeros(max(n, 1), np.int32)
    lib().mcsg_random_permutation(n, seed, f.ctypes.data_as(C.POINTER(C.c_int32)))
    return f[:n].copy()


def permute(g: Graph, p) -> Graph:
    """permute (graph.cpp:94-109): adjacency(p(u), p(v)) of the result = adjacency(u, v) of g."""
    p = np.asarray(p, dtype=np.int64)
    if p.shape != (g.n(),) or sorted(p.tolist()) != list(range(g.n())):
        raise GraphError("permutation size does not match graph" if p.shape != (g.n(),)
                         else "permutation is not a bijection")
    codes = np.zeros_like(g.codes)
    codes[np.ix_(p, p)] = g.codes
    labels = None
    if g.labeled():
        labels = np.zeros(g.n(), np.int32)
        labels[p] = g.labels
    return Graph(g.n(), codes, g.directed(), labels)


def load_graph_file(path: str, format: str = "auto") -> Graph:
    """load_graph_file (graph_io.cpp:139-151): MIVIA binary or text, auto-detected."""
    fmt = {"mivia": 0, "text": 1, "auto": 2}[format]
    n = C.c_int32()
    flags = C.c_uint32()
    if lib().mcsg_load_graph_file(path.encode(), fmt, C.byref(n), C.byref(flags), None, None) != 0:
        raise _err()
    nn = n.value
    codes = np.zeros(max(nn * nn, 1), np.uint8)
    labels = np.zeros(max(nn, 1), np.int32)
    if lib().mcsg_load_graph_file(path.encode(), fmt, C.byref(n), C.byref(flags),
                                  codes.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  labels.ctypes.data_as(C.POINTER(C.c_int32))) != 0:
        raise _err()
    return Graph(nn, codes[: nn * nn], bool(flags.value & DIRECTED),
                 labels[:nn] if flags.value & LABELED else None)


def save_graph_file(g: Graph, path: str, format: str = "mivia") -> None:
    fmt = {"mivia": 0, "text": 1}[format]
    if lib().mcsg_save_graph_file(C.byref(g._c()), path.encode(), fmt) != 0:
        raise _err()


def pack_graph(g: Graph):
    """The loader's device form: per-vertex 64-bit adjacency rows (out, in)."""
    out = np.zeros(max(g.n(), 1), np.uint64)
    inn = np.zeros(max(g.n(), 1), np.uint64)
    if lib().mcsg_pack_graph(C.byref(g._c()), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                             inn.ctypes.data_as(C.POINTER(C.c_uint64))) != 0:
        raise _err()
    return out[: g.n()].copy(), inn[: g.n()].copy()


def pack_graph_words(g: Graph, words: int | None = None):
    """Multi-word device rows (n <= 255): arrays of shape (n, words), bit x%64
    of word x//64 (the wide kernels' form)."""
    w = words if words is not None else max(1, (g.n() + 63) // 64)
    out = np.zeros((max(g.n(), 1), w), np.uint64)
    inn = np.zeros((max(g.n(), 1), w), np.uint64)
    if lib().mcsg_pack_graph_words(C.byref(g._c()), w, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   inn.ctypes.data_as(C.POINTER(C.c_uint64))) != 0:
        raise _err()
    return out[: g.n()].copy(), inn[: g.n()].copy()


def make_ordering(g: Graph, strategy: OrderingStrategy) -> np.ndarray:
    f = np.zeros(max(g.n(), 1), np.int32)
    if lib().mcsg_ordering(C.byref(g._c()), int(strategy), f.ctypes.data_as(C.POINTER(C.c_int32))) != 0:
        raise _err()
    return f[: g.n()].copy()


def verify(g: Graph, h: Graph, mapping) -> bool:
    """oracle::verify (oracle.cpp:8-24); out-of-range vertices raise GraphError."""
    flat = np.asarray(mapping, np.int32).reshape(-1) if len(mapping) else np.zeros(1, np.int32)
    rc = lib().mcsg_verify(C.byref(g._c()), C.byref(h._c()), flat.ctypes.data_as(C.POINTER(C.c_int32)),
                           len(mapping))
    if rc < 0:
        raise _err()
    return rc == 1


# ------------------------------------------------------------------ solving --
class SharedBound:
    """SharedBound (solve.hpp:70-81): a monotone size shared between engines.
    Passed as SolveConfig.shared_bound, the running kernel reads it as a live
    size floor and raises it to the size of every mapping it stores."""

    def __init__(self, size: int = 0):
        self._v = C.c_int32(int(size))

    def get(self) -> int:
        return int(self._v.value)

    def bump(self, size: int) -> None:
        if size > self._v.value:
            self._v.value = int(size)


@dataclass
class SolveConfig:
    """SolveConfig (solve.hpp:118-125) plus the GPU engine knobs."""
    budget_seconds: float = 1e9
    order: OrderingStrategy = OrderingStrategy.none
    cancel: object = None              # a ctypes c_int32 (or anything with .value) polled while running
    disable_pruning: bool = False
    shared_bound: "int | SharedBound" = 0  # size floor, or a live SharedBound shared with other engines
    mode: int = MODE_THROUGHPUT        # MODE_PARITY: reference node order and counts
    device: int = -1
    max_warps: int = 0
    smem_classes: int = 0
    seed: int = 0
    devices: tuple = ()                # > 1 entry: shard one instance over these GPUs
    frontier: int = 0                  # host-expanded subtrees per device (0 = 256)
    deadend: tuple | None = None       # ("abs", n) | ("rel", mult): DeadEndPolicy
    deadend_jump: "JumpMode | None" = None  # jump that resumes after a suspect verdict
    restart_multiplier: float = 0.0    # RestartConfig::multiplier (throughput mode); 0 = no restarts
    warp_share: int = 0                # > 1: use 1/warp_share of the GPU (concurrent engines on one GPU)


@dataclass
class SearchStats:
    """SearchStats (solve.hpp:27-55): the reference's fields first, mapped to
    what the GPU engine measures; then the engine's own counters."""
    recursions: int = 0
    deadend_suspects: int = 0
    # reference fields of the other engines (solve.hpp:35-52)
    per_worker_recursions: list = field(default_factory=list)  # not kept per warp (thousands of warps)
    idle_seconds: float = 0.0          # Σ over warps of the time spent waiting for a subtree
    tasks_published: int = 0           # = donations (subtrees handed to idle warps)
    iterations_total: int = 0          # parallel-engine iteration ledger: not applicable
    iterations_executed: int = 0
    iterations_pruned: int = 0
    iteration_double_executions: int = 0
    restore_checks: int = 0            # iterative-engine frame checks: not applicable
    restore_violations: int = 0
    peak_frames: int = 0
    peak_frame_bytes: int = 0
    restarts: int = 0                  # restart events (restart_multiplier > 0; restarts.cpp:35-246)
    frozen: int = 0                    # open-path subtrees frozen into the ring by those restarts
    visited_ranges: int = 0            # 1 for a completed search: the whole tree, exactly once
    wall_seconds: float = 0.0
    kernel_seconds: float = 0.0
    solve_seconds: float = 0.0
    probes: int = 0
    seed: int = 0
    sum_classes: int = 0
    splits: int = 0
    split_classes: int = 0
    donations: int = 0
    tasks: int = 0
    spills: int = 0
    warps: int = 0
    ctas: int = 0
    smem_per_cta: int = 0
    smem_classes: int = 0
    h2d_seconds: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    launches: int = 0
    busy_cycles: int = 0
    idle_cycles: int = 0
    peer_pushes: int = 0               # incumbent sizes pushed to peer GPUs (NVLink P2P)


@dataclass
class SolveResult:
    status: SolveStatus = SolveStatus.optimal
    best: list = field(default_factory=list)   # [(v in G, u in H)] original ids
    size: int = 0
    stats: SearchStats = field(default_factory=SearchStats)

    def canonical_bytes(self) -> str:
        """solve.cpp:40-47 without the fields this engine does not produce."""
        m = "".join(f"{v}->{u}," for v, u in self.best)
        return f"{self.status.name}|{self.size}|{m}|{self.stats.recursions}|{self.stats.seed}|{self.stats.probes}"


def _options(cfg: SolveConfig | None, **over) -> _Options:
    cfg = cfg or SolveConfig()
    o = _Options()
    o.budget_s = cfg.budget_seconds
    o.order = int(cfg.order)
    o.mode = cfg.mode
    o.goal = 0
    o.disable_pruning = int(cfg.disable_pruning)
    if isinstance(cfg.shared_bound, SharedBound):
        o.floor_size = cfg.shared_bound.get()
        o.shared_bound = C.pointer(cfg.shared_bound._v)
    else:
        o.floor_size = int(cfg.shared_bound)
    o.device = cfg.device
    o.max_warps = cfg.max_warps
    o.smem_classes = cfg.smem_classes
    o.seed = cfg.seed
    if cfg.cancel is not None:
        o.cancel = C.cast(C.pointer(cfg.cancel), C.POINTER(C.c_int32))
    if len(cfg.devices) > 16:
        raise GraphError("at most 16 devices")
    o.n_devices = len(cfg.devices)
    for i, dv in enumerate(cfg.devices):
        o.devices[i] = int(dv)
    o.frontier = cfg.frontier
    if cfg.deadend is not None:
        kind, val = cfg.deadend
        if kind == "abs":
            o.deadend_abs = int(val)
            o.deadend_kind = 1
        elif kind == "rel":
            o.deadend_rel = float(val)
            o.deadend_kind = 2
        else:
            raise GraphError(f"unknown deadend policy '{kind}'")
        if cfg.deadend_jump is not None:
            o.deadend_jump = 2 if cfg.deadend_jump == JumpMode.doubling else 1
    o.restart_multiplier = float(cfg.restart_multiplier)
    o.warp_share = int(cfg.warp_share)
    for k, v in over.items():
        setattr(o, k, v)
    return o


def _result(r: _Result, st: _Stats | None = None, seed: int = 0) -> SolveResult:
    pairs = [(int(r.pairs[2 * i]), int(r.pairs[2 * i + 1])) for i in range(r.size)]
    s = SearchStats(recursions=int(r.nodes), solve_seconds=r.solve_s, seed=seed, probes=int(r.probes),
                    deadend_suspects=int(r.deadend_suspects))
    if st is not None:
        s.wall_seconds = st.wall_s
        s.kernel_seconds = st.kernel_s
        s.h2d_seconds = st.h2d_s
        s.probes = int(st.probes)
        s.sum_classes, s.splits, s.split_classes = int(st.sum_classes), int(st.splits), int(st.split_classes)
        s.donations, s.tasks, s.spills = int(st.donations), int(st.tasks), int(st.spills)
        s.warps, s.ctas, s.smem_per_cta, s.smem_classes = st.warps, st.ctas, st.smem_per_cta, st.smem_classes
        s.h2d_bytes, s.d2h_bytes, s.launches = int(st.h2d_bytes), int(st.d2h_bytes), int(st.launches)
        s.busy_cycles, s.idle_cycles = int(st.busy_cycles), int(st.idle_cycles)
        s.tasks_published = s.donations
        s.restarts, s.frozen = int(st.restarts), int(st.frozen)
        s.peer_pushes = int(st.peer_pushes)
        s.idle_seconds = float(st.idle_s)
    if r.status == 0:
        s.visited_ranges = 1
    return SolveResult(SolveStatus(r.status), pairs, int(r.size), s)



def _check(rc: int):
    if rc == 3:
        raise _err()


def solve(g: Graph, h: Graph, config: SolveConfig | None = None) -> SolveResult:
    """mcs::solve (solve.hpp:128). status optimal guarantees the exact MCS size."""
    r, st = _Result(), _Stats()
    o = _options(config)
    _check(lib().mcsg_solve(C.byref(g._c()), C.byref(h._c()), C.byref(o), C.byref(r), C.byref(st)))
    return _result(r, st, (config or SolveConfig()).seed)


def solve_parallel(g: Graph, h: Graph, config: SolveConfig | None = None, workers: int = 0,
                   part_level: int = 5) -> SolveResult:
    """mcs::solve_parallel (engine_parallel.hpp:16): the GPU work-sharing engine.

    ``workers`` caps the resident warps (0 = all); ``part_level`` is accepted for
    signature parity (donation depth is adaptive on the GPU).
    """
    if workers < 0 or part_level < 0:
        raise GraphError("solve_parallel: workers and part_level must be non-negative")
    cfg = config or SolveConfig()
    r, st = _Result(), _Stats()
    o = _options(cfg, mode=MODE_THROUGHPUT, max_warps=workers or cfg.max_warps)
    _check(lib().mcsg_solve_parallel(C.byref(g._c()), C.byref(h._c()), C.byref(o), C.byref(r), C.byref(st)))
    return _result(r, st, cfg.seed)


def solve_batch(pairs, config: SolveConfig | None = None):
    """Many pairs in one persistent launch (run_suite's loop, bench.cpp:74-122)."""
    n = len(pairs)
    G = (_Graph * max(n, 1))()
    H = (_Graph * max(n, 1))()
    for i, (g, h) in enumerate(pairs):
        G[i] = g._c()
        H[i] = h._c()
    R = (_Result * max(n, 1))()
    st = _Stats()
    o = _options(config)
    _check(lib().mcsg_solve_batch(n, G, H, C.byref(o), R, C.byref(st)))
    seed = (config or SolveConfig()).seed
    out = [_result(R[i], None, seed) for i in range(n)]
    stats = _result(_Result(), st, seed).stats
    stats.recursions = int(st.nodes)
    return out, stats


def solve_goal_directed(g: Graph, h: Graph, config: SolveConfig | None = None) -> SolveResult:
    """mcs::solve_goal_directed (solve.cpp:131-168): goal probes run on the GPU."""
    r, st = _Result(), _Stats()
    _check(lib().mcsg_solve_goal_directed(C.byref(g._c()), C.byref(h._c()), C.byref(_options(config)),
                                          C.byref(r), C.byref(st)))
    return _result(r, st)


def bound_jump_search(g: Graph, h: Graph, current_best: int, mode: JumpMode,
                      config: SolveConfig | None = None) -> SolveResult:
    """mcs::bound_jump_search (heuristics.cpp:114-185) over GPU goal probes."""
    r, st = _Result(), _Stats()
    _check(lib().mcsg_bound_jump(C.byref(g._c()), C.byref(h._c()), int(current_best), int(mode),
                                 C.byref(_options(config)), C.byref(r), C.byref(st)))
    return _result(r, st)


# ---------------------------------------------------------------- restarts --
_KEY_MAX = 2**31 - 1


class VisitedRanges:
    """VisitedRanges (heuristics.hpp:79-89, heuristics.cpp:187-210): half-open
    lexicographic intervals of PositionKeys — a key is the list of
    (depth, iteration) pairs along a node's path from the root."""

    def __init__(self):
        self.runs = []

    def add(self, lo, hi):
        self.runs.append((list(lo), list(hi)))

    def normalize(self) -> bool:
        """Sorts and merges touching runs; False if any two overlap."""
        self.runs.sort()
        disjoint = True
        merged = []
        for lo, hi in self.runs:
            if merged and lo < merged[-1][1]:
                disjoint = False
            if merged and lo == merged[-1][1]:
                merged[-1] = (merged[-1][0], hi)
            else:
                merged.append((lo, hi))
        self.runs = merged
        return disjoint

    def covers(self, key) -> bool:
        key = list(key)
        return any(not (key < lo) and key < hi for lo, hi in self.runs)

    def size(self) -> int:
        return len(self.runs)


@dataclass
class RestartConfig:
    """RestartConfig (heuristics.hpp:92-104) plus the GPU engine knobs.

    mode MODE_PARITY (default) reproduces the reference's RestartDriver
    exactly — seeded mt19937_64 segment draws, recursions, restarts, visited
    ranges — one GPU warp per segment; MODE_THROUGHPUT runs the all-warp
    engine's restart epochs (open paths frozen into the task ring)."""
    seed: int = 1
    multiplier: float = 2.0            # <= 0: restarts off
    budget_seconds: float = 1e9
    order: OrderingStrategy = OrderingStrategy.none
    cancel: object = None
    disable_pruning: bool = False
    shared_bound: "int | SharedBound" = 0
    ranges_out: "VisitedRanges | None" = None  # instrumentation sink
    mode: int = MODE_PARITY
    device: int = -1


def solve_with_restarts(g: Graph, h: Graph, config: RestartConfig | None = None) -> SolveResult:
    """mcs::solve_with_restarts (heuristics.hpp:107, restarts.cpp:195-246)."""
    cfg = config or RestartConfig()
    sc = SolveConfig(budget_seconds=cfg.budget_seconds, order=cfg.order, cancel=cfg.cancel,
                     disable_pruning=cfg.disable_pruning, shared_bound=cfg.shared_bound, mode=cfg.mode,
                     device=cfg.device, seed=cfg.seed, restart_multiplier=cfg.multiplier)
    o = _options(sc)
    want = cfg.ranges_out is not None and cfg.mode == MODE_PARITY
    cap = 1 << 16 if want else 0
    while True:
        r, st = _Result(), _Stats()
        need = C.c_int64(0)
        words = (C.c_int32 * cap)() if cap else None
        _check(lib().mcsg_solve_with_restarts(C.byref(g._c()), C.byref(h._c()), C.byref(o), C.byref(r),
                                              C.byref(st), words, cap, C.byref(need)))
        if not want or need.value <= cap:
            break
        cap = need.value  # the run is deterministic: again with room for every range
    if words is not None:
        words = words[:need.value]
    res = _result(r, st, cfg.seed)
    res.stats.restarts = int(st.restarts)
    res.stats.visited_ranges = int(st.visited_ranges)
    if cfg.mode == MODE_PARITY:
        res.stats.recursions = int(st.nodes)
    if words is not None:
        w, i = words, 0
        keys = []
        while i < len(w):
            k = w[i]
            keys.append([(d, w[i + 1 + d]) for d in range(k)])
            i += 1 + k
        for j in range(0, len(keys), 2):
            cfg.ranges_out.add(keys[j], keys[j + 1])
    return res


# ----------------------------------------------------------------- engines --
_ORDER_NAMES = {"degree": OrderingStrategy.degree_desc,
                "components": OrderingStrategy.components_then_degree,
                "block": OrderingStrategy.block_triangular}


@dataclass
class EngineSpec:
    """EngineSpec (portfolio.hpp:16-31); base in recursive|parallel|iterative|gpu."""
    base: str = "recursive"
    order: OrderingStrategy = OrderingStrategy.none
    goal_directed: bool = False
    jump: JumpMode | None = None
    deadend: tuple | None = None        # ("abs", n) | ("rel", mult)
    restart_seed: int | None = None
    workers: int = 0
    part_level: int = 5
    budget_seconds: float = -1.0
    stage: int = 1

    def name(self) -> str:
        if self.base == "recursive":
            if self.goal_directed:
                s = "goal"
            elif self.jump is not None:
                s = "jump:plus1" if self.jump == JumpMode.plus_one else "jump:double"
            elif self.restart_seed is not None:
                s = f"restarts:{self.restart_seed}"
            else:
                s = "recursive"
        elif self.base == "parallel":
            s = f"parallel:{self.workers}"
        else:
            s = self.base
        if self.order != OrderingStrategy.none:
            s += "+order=" + {v: k for k, v in _ORDER_NAMES.items()}[self.order]
        if self.deadend is not None:
            s += f"+deadend={self.deadend[0]}:{self.deadend[1]}"
        return s


def parse_engine_spec(text: str) -> EngineSpec:
    """parse_engine_spec (portfolio.cpp:51-99): "recursive", "goal", "parallel:4",
    "iterative", "jump:plus1", "jump:double", "restarts:7", "gpu", each optionally
    suffixed with "+order=degree|components|block" and "+deadend=abs:N|rel:X"."""
    spec = EngineSpec()
    head, _, rest = text.partition("+")
    name, _, arg = head.partition(":")
    if name == "recursive":
        pass
    elif name == "goal":
        spec.goal_directed = True
    elif name == "parallel":
        spec.base = "parallel"
        if arg:
            spec.workers = int(arg)
    elif name == "iterative":
        spec.base = "iterative"
    elif name == "gpu":
        spec.base = "gpu"
    elif name == "jump":
        spec.jump = JumpMode.doubling if arg == "double" else JumpMode.plus_one
    elif name == "restarts":
        spec.restart_seed = int(arg) if arg else 1
    else:
        raise GraphError(f"unknown engine '{name}'")
    for flag in filter(None, rest.split("+")):
        key, _, val = flag.partition("=")
        if key == "order":
            if val not in _ORDER_NAMES:
                raise GraphError(f"unknown ordering '{val}'")
            spec.order = _ORDER_NAMES[val]
        elif key == "deadend":
            if val.startswith("abs:"):
                spec.deadend = ("abs", int(val[4:]))
            elif val.startswith("rel:"):
                spec.deadend = ("rel", float(val[4:]))
            else:
                raise GraphError(f"unknown deadend policy '{val}'")
        else:
            raise GraphError(f"unknown engine flag '{key}'")
    return spec


def run_engine(g: Graph, h: Graph, spec: EngineSpec, config: SolveConfig | None = None) -> SolveResult:
    """run_engine (portfolio.cpp:101-157) dispatch onto the GPU engines.

    recursive / iterative -> parity mode (reference node order);
    parallel / gpu       -> throughput mode (all warps, donation);
    goal / jump          -> GPU goal probes; restarts:<seed> -> solve_with_restarts
    (RestartConfig::multiplier = 2): with a parity-mode config the reference's
    RestartDriver exactly; otherwise throughput mode with that seed's search
    order, every warp freezing its open path into the ring when the nodes
    since the last improvement reach twice the nodes at it. Orderings are
    applied host-side around every engine.
    """
    import dataclasses
    cfg = dataclasses.replace(config or SolveConfig(), order=spec.order)
    if spec.base not in ("recursive",) and (spec.goal_directed or spec.jump is not None
                                            or spec.restart_seed is not None):
        raise GraphError("goal/jump/restart variants run on the recursive engine only")
    if spec.base == "parallel":
        return solve_parallel(g, h, cfg, spec.workers, spec.part_level)
    if spec.base == "gpu":
        return solve(g, h, dataclasses.replace(cfg, mode=MODE_THROUGHPUT))
    if spec.base == "iterative":
        return solve(g, h, dataclasses.replace(cfg, mode=MODE_PARITY))
    if spec.goal_directed:
        return solve_goal_directed(g, h, cfg)
    if spec.restart_seed is not None:
        # RestartConfig from the solve config (portfolio.cpp:123-133); an
        # explicit parity-mode config runs the reference's RestartDriver
        # exactly, otherwise the all-warp engine's restart epochs
        return solve_with_restarts(g, h, RestartConfig(
            seed=spec.restart_seed, budget_seconds=cfg.budget_seconds, order=cfg.order, cancel=cfg.cancel,
            disable_pruning=cfg.disable_pruning, shared_bound=cfg.shared_bound,
            mode=MODE_PARITY if cfg.mode == MODE_PARITY else MODE_THROUGHPUT, device=cfg.device))
    if spec.deadend is not None:
        # forecast-then-mitigate (portfolio.cpp:136-155): a monitored solve;
        # with a jump configured, a suspect verdict hands the incumbent to the
        # bound jump (without one the monitor never stops the search). An
        # explicit parity-mode config runs the reference's per-node monitor
        # (its recursions, probes and suspects); otherwise the all-warp engine
        # monitors at its polls.
        mode = MODE_PARITY if cfg.mode == MODE_PARITY else MODE_THROUGHPUT
        return solve(g, h, dataclasses.replace(cfg, mode=mode, deadend=spec.deadend, deadend_jump=spec.jump))
    if spec.jump is not None:
        return bound_jump_search(g, h, 0, spec.jump, cfg)
    return solve(g, h, dataclasses.replace(cfg, mode=MODE_PARITY))


def probe_parallel(g: Graph, h: Graph, current_best: int = 0, width: int = 0,
                   config: SolveConfig | None = None) -> SolveResult:
    """Parallel binary search over goal probes (bound_jump_search's bracket,
    heuristics.cpp:114-185, `width` targets per round, over config.devices):
    a reached target implies every lower one, an exhausted one every higher
    one, across GPUs over NVLink P2P. Throughput mode."""
    import dataclasses
    cfg = dataclasses.replace(config or SolveConfig(), mode=MODE_THROUGHPUT)
    r, st = _Result(), _Stats()
    _check(lib().mcsg_probe_parallel(C.byref(g._c()), C.byref(h._c()), int(current_best), int(width),
                                     C.byref(_options(cfg)), C.byref(r), C.byref(st)))
    return _result(r, st)


@dataclass
class PortfolioConfig:
    """PortfolioConfig (portfolio.hpp:78-84)."""
    mode: str = "race_all"              # "race_all" | "staged"
    budget_seconds: float = 1e9
    stage1_budget_seconds: float = 5.0
    grace_seconds: float = 1.0          # cancellation acknowledgment watchdog
    share_incumbent: bool = False       # monotone size broadcasts between engines (SharedBound)


@dataclass
class EngineReport:
    """EngineReport (portfolio.hpp:68-75)."""
    spec_name: str = ""
    outcome: str = "finished"           # finished | cancelled | error | timeout
    size: int = 0
    wall_seconds: float = 0.0
    cancel_ack_seconds: float = -1.0
    error: str = ""


@dataclass
class PortfolioResult:
    """PortfolioResult (portfolio.hpp:86-98)."""
    status: SolveStatus = SolveStatus.optimal
    winner: str = ""
    size: int = 0
    mapping: list = field(default_factory=list)
    wall_seconds: float = 0.0
    stats: SearchStats = field(default_factory=SearchStats)
    engines: list = field(default_factory=list)   # EngineReport per member run
    grace_violations: int = 0
    overhead_seconds: float = 0.0


def _is_searcher(s: EngineSpec) -> bool:
    """Plain searches (any ordering) race inside ONE GPU launch with a shared
    incumbent size; every other member is an engine of its own."""
    return (s.base in ("recursive", "iterative", "parallel", "gpu") and not s.goal_directed
            and s.jump is None and s.deadend is None and s.restart_seed is None)


def _race_group(g: Graph, h: Graph, specs, config: SolveConfig):
    """The searchers of a portfolio in one launch (mcsg_portfolio): members are
    orderings of the pair sharing the incumbent size; the first to prove wins."""
    orders = (C.c_int32 * len(specs))(*[int(s.order) for s in specs])
    seeds = (C.c_uint64 * len(specs))(*[0 for _ in specs])
    r, st = _Result(), _Stats()
    win = C.c_int32(-1)
    _check(lib().mcsg_portfolio(C.byref(g._c()), C.byref(h._c()), len(specs), orders, seeds,
                                C.byref(_options(config)), C.byref(r), C.byref(win), C.byref(st)))
    res = _result(r, st)
    return res, (specs[win.value].name() if win.value >= 0 else "")


def _race(g, h, specs, cfg: SolveConfig, budget: float, bound, grace: float):
    """race() (portfolio.cpp:249-292) over GPU engines: one host thread per
    unit — the plain searchers together as one launch, every goal / jump /
    dead-end / restarts member as its own engine (run_engine, GPU probes and
    searches). Units are dealt over the configured devices; units sharing a
    GPU split its warps (warp_share) and run concurrently. The first unit to
    finish optimal wins and the others are cancelled (their cancel flag is
    polled by the running kernels)."""
    import dataclasses
    import threading
    searchers = [s for s in specs if _is_searcher(s)]
    units = ([("group", searchers)] if searchers else []) + [("engine", s) for s in specs if not _is_searcher(s)]
    devices = list(cfg.devices) if cfg.devices else [cfg.device]
    # device placement: with a GPU per unit to spare, the searchers' launch
    # spreads over every GPU the engines leave (P2P incumbent, first to prove
    # stops all); otherwise units are dealt round-robin and share GPUs
    n_eng = len(units) - (1 if searchers else 0)
    if searchers and len(devices) >= len(units):
        place = [devices[:len(devices) - n_eng]] + [[d] for d in devices[len(devices) - n_eng:]]
    else:
        place = [[devices[i % len(devices)]] for i in range(len(units))]
    per_dev = {}
    for pl in place:
        for d in pl:
            per_dev[d] = per_dev.get(d, 0) + 1
    cancel = C.c_int32(0)
    out = [None] * len(units)

    def run(i):
        kind, what = units[i]
        dev = place[i][0]
        ucfg = dataclasses.replace(cfg, device=dev, devices=tuple(place[i]) if len(place[i]) > 1 else (),
                                   cancel=cancel, warp_share=per_dev[dev],
                                   shared_bound=bound if bound is not None else cfg.shared_bound)
        t0 = time.perf_counter()
        try:
            if kind == "group":
                res, name = _race_group(g, h, what, dataclasses.replace(
                    ucfg, budget_seconds=budget, mode=MODE_THROUGHPUT))
            else:
                b = min(what.budget_seconds, budget) if what.budget_seconds >= 0 else budget
                res, name = run_engine(g, h, what, dataclasses.replace(ucfg, budget_seconds=b)), what.name()
            out[i] = (res, name or (what.name() if kind == "engine" else ",".join(s.name() for s in what)),
                      None, time.perf_counter())
        except GraphError as e:
            out[i] = (None, what.name() if kind == "engine" else "group", str(e), time.perf_counter())

    t_start = time.perf_counter()
    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(units))]
    for t in threads:
        t.start()
    reports, seen = [], [False] * len(units)
    winner = None
    t_cancel = None
    best = None
    while not all(seen):
        for i, t in enumerate(threads):
            if seen[i] or t.is_alive():
                continue
            seen[i] = True
            res, name, err, t_end = out[i]
            rep = EngineReport(spec_name=name or (units[i][1].name() if units[i][0] == "engine" else ""),
                               wall_seconds=t_end - t_start)
            if err is not None:
                rep.outcome, rep.error = "error", err
            else:
                rep.size = res.size
                rep.outcome = {SolveStatus.optimal: "finished", SolveStatus.timeout: "timeout",
                               SolveStatus.cancelled: "cancelled"}[res.status]
                if res.status == SolveStatus.optimal and winner is None:
                    winner = (name, res, rep.wall_seconds)
                    cancel.value = 1
                    t_cancel = time.perf_counter()
                if best is None or res.size > best.size:
                    best = res
            if t_cancel is not None and (winner is None or winner[0] != rep.spec_name):
                rep.cancel_ack_seconds = max(0.0, t_end - t_cancel)
            reports.append(rep)
        if not all(seen):
            time.sleep(0.001)
    grace_violations = sum(1 for r in reports if r.cancel_ack_seconds > grace)
    return winner, best, reports, grace_violations


def run_portfolio(g: Graph, h: Graph, specs, config: SolveConfig | None = None,
                  portfolio: PortfolioConfig | None = None) -> PortfolioResult:
    """run_portfolio (portfolio.cpp:310-365) on GPU engines. Every member
    runs with its own semantics — plain searches race in one launch with a
    shared incumbent size; goal-directed, bound-jump, dead-end and restarts
    members run as their own GPU engines next to them — and the first member
    to finish optimal wins (portfolio.cpp:271-279). Staged mode runs the
    stage-1 members under stage1_budget_seconds, then stage 2 (everything
    again when nothing is staged) with the rest of the budget, carrying the
    best incumbent over. share_incumbent broadcasts sizes between the units
    (SharedBound, solve.hpp:68-81)."""
    specs = [parse_engine_spec(s) if isinstance(s, str) else s for s in specs]
    if not specs:
        raise GraphError("portfolio needs at least one engine spec")
    for s in specs:
        if s.base not in ("recursive",) and (s.goal_directed or s.jump is not None or s.restart_seed is not None):
            raise GraphError("goal/jump/restart variants run on the recursive engine only")
    cfg = config or SolveConfig()
    pc = portfolio or PortfolioConfig(budget_seconds=cfg.budget_seconds)
    t0 = time.perf_counter()
    bound = SharedBound(0) if pc.share_incumbent else None
    remaining = lambda: pc.budget_seconds - (time.perf_counter() - t0)  # noqa: E731
    if pc.mode == "staged":
        stage1 = [s for s in specs if s.stage <= 1]
        stage2 = [s for s in specs if s.stage > 1]
        winner, best, reports, gv = None, None, [], 0
        if stage1 and pc.stage1_budget_seconds > 0:
            winner, best, reports, gv = _race(g, h, stage1, cfg, min(pc.stage1_budget_seconds, pc.budget_seconds),
                                              bound, pc.grace_seconds)
        if winner is None:
            w2, b2, r2, gv2 = _race(g, h, stage2 or stage1, cfg, max(0.0, remaining()), bound, pc.grace_seconds)
            winner, reports, gv = w2, reports + r2, gv + gv2
            if best is None or (b2 is not None and b2.size > best.size):
                best = b2
    elif pc.mode == "race_all":
        winner, best, reports, gv = _race(g, h, specs, cfg, pc.budget_seconds, bound, pc.grace_seconds)
    else:
        raise GraphError(f"unknown portfolio mode '{pc.mode}'")
    wall = time.perf_counter() - t0
    res = PortfolioResult(engines=reports, grace_violations=gv, wall_seconds=wall)
    if winner is not None:
        name, r, w_wall = winner
        res.status, res.winner, res.size, res.mapping, res.stats = SolveStatus.optimal, name, r.size, r.best, r.stats
        res.overhead_seconds = wall - w_wall
    else:
        if all(r.outcome == "error" for r in reports):
            raise GraphError("portfolio: every engine failed")
        res.status = SolveStatus.timeout
        if best is not None:
            res.size, res.mapping, res.stats = best.size, best.best, best.stats
    return res
