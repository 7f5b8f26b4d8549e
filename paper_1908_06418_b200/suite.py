"""Benchmark-suite runner: manifests, per-instance records, CSV and cactus
curves for the GPU engines, in the reference's formats (include/mcs/bench.hpp,
src/bench.cpp:48-182), so GPU runs line up with the reference's CPU records
and the paper's cactus plots.

Extension over the reference: the ``gpu`` engine solves every loaded instance
of the manifest in ONE persistent launch (``solve_batch``); its record's
``wall_s`` is then the instance's own time to proven optimum inside that
launch (device clock), which is what a cactus curve counts.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

from . import (GraphError, SolveConfig, SolveStatus, load_graph_file, parse_engine_spec, run_engine,
               solve_batch, verify, MODE_THROUGHPUT)


@dataclass
class InstanceSpec:
    id: str
    category: str
    g_path: str
    h_path: str


@dataclass
class InstanceRecord:
    """bench.hpp:24-38."""
    pair_id: str = ""
    category: str = ""
    n_g: int = 0
    n_h: int = 0
    engine: str = ""
    status: str = ""     # optimal | timeout | cancelled | error
    size: int = -1       # present iff status != error
    wall_seconds: float = 0.0
    cpu_seconds: float = 0.0
    recursions: int = 0
    seed: int = 0


@dataclass
class SuiteConfig:
    engines: list = field(default_factory=list)  # EngineSpec or spec strings
    budget_seconds: float = 10.0
    verify_results: bool = True


def _stem(path: str) -> str:
    name = path.rsplit("/", 1)[-1]
    return name.rsplit(".", 1)[0] if "." in name else name


def _join(root: str, rel: str) -> str:
    if not root or not rel or rel.startswith("/"):
        return rel
    return root + rel if root.endswith("/") else root + "/" + rel


def load_manifest(path: str, dataset_root: str = ""):
    """Manifest lines `g_file h_file [category]`, '#' comments; relative paths
    resolve against dataset_root or $MCS_DATASET_ROOT (bench.cpp:48-72)."""
    root = dataset_root or os.environ.get("MCS_DATASET_ROOT", "")
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise GraphError(f"cannot open manifest '{path}'")
    specs = []
    for line in lines:
        fields = line.split()
        if not fields or fields[0].startswith("#"):
            continue
        if len(fields) < 2:
            raise GraphError(f"manifest line needs two files: '{line}'")
        cat = fields[2] if len(fields) > 2 else "uncategorized"
        specs.append(InstanceSpec(f"{_stem(fields[0])}__{_stem(fields[1])}", cat,
                                  _join(root, fields[0]), _join(root, fields[1])))
    return specs


def _status_name(s: SolveStatus) -> str:
    return {SolveStatus.optimal: "optimal", SolveStatus.timeout: "timeout",
            SolveStatus.cancelled: "cancelled"}[SolveStatus(s)]


def run_suite(instances, config: SuiteConfig):
    """One record per (instance, engine); unloadable instances give an error
    record and the suite continues (bench.cpp:74-122)."""
    engines = [parse_engine_spec(e) if isinstance(e, str) else e for e in config.engines]
    loaded = []
    for inst in instances:
        try:
            loaded.append((load_graph_file(inst.g_path), load_graph_file(inst.h_path)))
        except Exception:
            loaded.append(None)
    out = {}
    for ei, spec in enumerate(engines):
        if spec.base == "gpu":  # the whole manifest in one persistent launch
            idx = [k for k, pair in enumerate(loaded) if pair is not None]
            if idx and config.budget_seconds > 0:
                c0 = time.process_time()
                res, _ = solve_batch([loaded[k] for k in idx],
                                     SolveConfig(mode=MODE_THROUGHPUT, budget_seconds=config.budget_seconds,
                                                 order=spec.order))
                cpu = (time.process_time() - c0) / max(len(idx), 1)
                for k, r in zip(idx, res):
                    out[(k, ei)] = (r, cpu)
            continue
        for k, pair in enumerate(loaded):
            if pair is None:
                continue
            c0 = time.process_time()
            try:
                r = run_engine(pair[0], pair[1], spec, SolveConfig(budget_seconds=config.budget_seconds))
            except Exception:
                r = None
            out[(k, ei)] = (r, time.process_time() - c0)
    records = []
    for k, inst in enumerate(instances):
        for ei, spec in enumerate(engines):
            rec = InstanceRecord(pair_id=inst.id, category=inst.category, engine=spec.name())
            if loaded[k] is None:
                rec.status = "error"
                records.append(rec)
                continue
            g, h = loaded[k]
            rec.n_g, rec.n_h = g.n(), h.n()
            if spec.restart_seed is not None:
                rec.seed = spec.restart_seed
            if config.budget_seconds <= 0:  # solve.cpp:95
                rec.status, rec.size = "timeout", 0
                records.append(rec)
                continue
            r, cpu = out.get((k, ei), (None, 0.0))
            rec.cpu_seconds = cpu
            if r is None or (config.verify_results and not verify(g, h, r.best)):
                rec.status = "error"
            else:
                rec.status = _status_name(r.status)
                rec.size = r.size
                rec.wall_seconds = r.stats.solve_seconds if spec.base == "gpu" else r.stats.wall_seconds
                rec.recursions = r.stats.recursions
            records.append(rec)
    return records


def _fmt(x: float) -> str:
    return "%.17g" % x  # std::setprecision(17), bench.cpp:31-35


def emit_csv(records) -> str:
    """bench.cpp:124-135."""
    lines = ["pair_id,category,n_g,n_h,engine,status,size,wall_s,cpu_s,recursions,seed"]
    for r in records:
        size = "" if r.status == "error" else str(r.size)
        lines.append(f"{r.pair_id},{r.category},{r.n_g},{r.n_h},{r.engine},{r.status},{size},"
                     f"{_fmt(r.wall_seconds)},{_fmt(r.cpu_seconds)},{r.recursions},{r.seed}")
    return "\n".join(lines) + "\n"


def parse_csv(csv: str):
    """bench.cpp:137-161."""
    lines = csv.split("\n")
    if not lines or not lines[0]:
        raise GraphError("empty CSV")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 11:
            raise GraphError(f"malformed CSV row: '{line}'")
        out.append(InstanceRecord(f[0], f[1], int(f[2]), int(f[3]), f[4], f[5], int(f[6]) if f[6] else -1,
                                  float(f[7]), float(f[8]), int(f[9]), int(f[10])))
    return out


@dataclass
class CactusPoint:
    engine: str
    threshold_seconds: float
    solved: int


def emit_cactus(records):
    """Per engine: sorted solve times with cumulative counts; timeouts excluded
    (bench.cpp:163-174)."""
    times = {}
    for r in records:
        if r.status == "optimal":
            times.setdefault(r.engine, []).append(r.wall_seconds)
    points = []
    for engine in sorted(times):
        for i, t in enumerate(sorted(times[engine])):
            points.append(CactusPoint(engine, t, i + 1))
    return points


def cactus_csv(points) -> str:
    lines = ["engine,threshold_s,solved"] + [f"{p.engine},{_fmt(p.threshold_seconds)},{p.solved}" for p in points]
    return "\n".join(lines) + "\n"
