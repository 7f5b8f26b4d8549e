// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference solver (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).
// It exists so that tests/ (golden-vector generation, parity pinning of the
// C restatement in oracle/mcs_oracle.c) and bench.py's reference arm can drive
// the reference's own public API:
//   mcs::random_graph            proj/include/mcs/graph.hpp:99
//   mcs::parse_engine_spec       proj/include/mcs/portfolio.hpp:34
//   mcs::run_engine              proj/include/mcs/portfolio.hpp:37
//   mcs::solve_parallel          proj/include/mcs/engine_parallel.hpp:16 (optionally with a SharedBound floor)
//   mcs::solve_with_restarts     proj/include/mcs/heuristics.hpp:107 (with the VisitedRanges sink)
//   mcs::oracle::verify          proj/include/mcs/oracle.hpp:16
//   mcs::oracle::mcs_bruteforce  proj/include/mcs/oracle.hpp:26
//   mcs::make_ordering           proj/include/mcs/heuristics.hpp:26
//   mcs::load_graph_file         proj/include/mcs/graph_io.hpp:33
// No reference source is copied here; the reference headers are included
// from /root/reference at build time only.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "mcs/engine_parallel.hpp"
#include "mcs/graph.hpp"
#include "mcs/graph_io.hpp"
#include "mcs/heuristics.hpp"
#include "mcs/label_classes.hpp"
#include "mcs/oracle.hpp"
#include "mcs/portfolio.hpp"
#include "mcs/solve.hpp"

extern "C" {

struct ref_graph {
    int32_t n;
    int32_t directed;
    const uint8_t* codes;   // n*n row-major, graph.hpp:60 layout
    const int32_t* labels;  // n entries or NULL
};

struct ref_result {
    int32_t status;  // 0 optimal, 1 timeout, 2 cancelled, -1 error
    int32_t size;
    int32_t pairs[2 * 256];
    uint64_t recursions;
    uint64_t probes;
    uint64_t restarts;
    uint64_t visited_ranges;
    uint64_t tasks_published;
    uint64_t double_executions;
    double wall_seconds;
    char error[256];
    uint64_t deadend_suspects;
};
}

namespace {

thread_local std::string g_err;

mcs::Graph to_graph(const ref_graph* rg) {
    std::vector<mcs::Edge> edges;
    const int n = rg->n;
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v) {
            uint8_t c = rg->codes[(size_t)u * n + v];
            if (c) edges.push_back({u, v, static_cast<mcs::EdgeCode>(c)});
        }
    std::optional<std::vector<int>> labels;
    if (rg->labels) labels.emplace(rg->labels, rg->labels + n);
    return mcs::from_edge_list(n, edges,
                               rg->directed ? mcs::GraphKind::directed : mcs::GraphKind::undirected,
                               std::move(labels));
}

void fill(const mcs::SolveResult& r, ref_result* out) {
    out->status = static_cast<int32_t>(r.status);
    out->size = r.size;
    int k = 0;
    for (const auto& p : r.best) {
        if (k >= 256) break;
        out->pairs[2 * k] = p.v;
        out->pairs[2 * k + 1] = p.u;
        ++k;
    }
    out->recursions = r.stats.recursions;
    out->probes = r.stats.probes;
    out->restarts = r.stats.restarts;
    out->visited_ranges = r.stats.visited_ranges;
    out->tasks_published = r.stats.tasks_published;
    out->double_executions = r.stats.iteration_double_executions;
    out->wall_seconds = r.stats.wall_seconds;
    out->error[0] = 0;
    out->deadend_suspects = r.stats.deadend_suspects;
}

void fail(ref_result* out, const char* what) {
    std::memset(out, 0, sizeof(*out));
    out->status = -1;
    std::strncpy(out->error, what, sizeof(out->error) - 1);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_hardware_concurrency(void) { return (int)std::thread::hardware_concurrency(); }

// Returns 0 on success; codes_out must hold n*n bytes, labels_out n ints
// (written only when label_count > 0).
int ref_random_graph(int n, double density, uint64_t seed, int directed, int label_count,
                     uint8_t* codes_out, int32_t* labels_out) {
    try {
        mcs::RandomGraphOptions o;
        o.kind = directed ? mcs::GraphKind::directed : mcs::GraphKind::undirected;
        o.label_count = label_count;
        mcs::Graph g = mcs::random_graph(n, density, seed, o);
        for (int u = 0; u < n; ++u)
            for (int v = 0; v < n; ++v) codes_out[(size_t)u * n + v] = g.code(u, v);
        if (label_count > 0 && labels_out)
            for (int v = 0; v < n; ++v) labels_out[v] = g.label(v);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_random_permutation(int n, uint64_t seed, int32_t* fwd_out) {
    auto p = mcs::random_permutation(n, seed);
    for (int i = 0; i < n; ++i) fwd_out[i] = p(i);
    return 0;
}

// Runs one engine spec (portfolio.cpp grammar) through mcs::run_engine.
int ref_run_engine(const ref_graph* g, const ref_graph* h, const char* spec, double budget,
                   int disable_pruning, ref_result* out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::SolveConfig cfg;
        cfg.budget_seconds = budget;
        cfg.disable_pruning = disable_pruning != 0;
        mcs::SolveResult r = mcs::run_engine(gg, hh, mcs::parse_engine_spec(spec), cfg);
        fill(r, out);
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// mcs::solve_with_restarts (heuristics.hpp:107) with the VisitedRanges sink:
// ranges_out receives each run as [len(lo), lo iterations..., len(hi), hi
// iterations...] (a PositionKey's depth field equals its index, so only the
// iterations travel); *ranges_len = the words needed.
int ref_solve_with_restarts(const ref_graph* g, const ref_graph* h, uint64_t seed, double multiplier,
                            int disable_pruning, int order, double budget, ref_result* out, int32_t* ranges_out,
                            int64_t ranges_cap, int64_t* ranges_len) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::RestartConfig rc;
        rc.seed = seed;
        rc.multiplier = multiplier;
        rc.disable_pruning = disable_pruning != 0;
        rc.order = static_cast<mcs::OrderingStrategy>(order);
        rc.budget_seconds = budget;
        mcs::VisitedRanges vr;
        rc.ranges_out = &vr;
        fill(mcs::solve_with_restarts(gg, hh, rc), out);
        int64_t w = 0;
        auto put = [&](int32_t x) {
            if (ranges_out && w < ranges_cap) ranges_out[w] = x;
            ++w;
        };
        for (const auto& run : vr.runs)
            for (const mcs::PositionKey* k : {&run.first, &run.second}) {
                put(int32_t(k->size()));
                for (size_t d = 0; d < k->size(); ++d) {
                    if ((*k)[d].first != int(d)) throw std::runtime_error("position key depth != index");
                    put((*k)[d].second);
                }
            }
        if (ranges_len) *ranges_len = w;
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// Thread-pool engine with explicit workers (0 = hardware_concurrency) and part_level.
int ref_solve_parallel(const ref_graph* g, const ref_graph* h, int workers, int part_level,
                       double budget, ref_result* out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::ParallelConfig pc;
        pc.workers = workers;
        pc.part_level = part_level;
        pc.base.budget_seconds = budget;
        fill(mcs::solve_parallel(gg, hh, pc), out);
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// Thread-pool engine seeded with an external size floor: SolveConfig::shared_bound
// (solve.hpp:70-81,124) starts at `floor`, and the pool prunes every node whose
// bound is <= max(incumbent, floor) (engine_parallel.cpp:75-78). Status optimal
// with floor k therefore proves that no common subgraph larger than k exists.
int ref_solve_parallel_floor(const ref_graph* g, const ref_graph* h, int workers, int part_level,
                             double budget, int floor, ref_result* out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::SharedBound sb;
        sb.bump(floor);
        mcs::ParallelConfig pc;
        pc.workers = workers;
        pc.part_level = part_level;
        pc.base.budget_seconds = budget;
        pc.base.shared_bound = &sb;
        fill(mcs::solve_parallel(gg, hh, pc), out);
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// Sequential solve (solve.hpp:128) with SolveConfig::shared_bound seeded at
// `floor`: the size-floor semantics of LocalIncumbent (search_core.hpp:21-36).
int ref_solve_floor(const ref_graph* g, const ref_graph* h, int floor, double budget, ref_result* out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::SharedBound sb;
        sb.bump(floor);
        mcs::SolveConfig cfg;
        cfg.budget_seconds = budget;
        cfg.shared_bound = &sb;
        fill(mcs::solve(gg, hh, cfg), out);
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// Bound-jump from a caller-supplied lower bound (heuristics.hpp:69).
int ref_bound_jump(const ref_graph* g, const ref_graph* h, int current_best, int doubling,
                   double budget, ref_result* out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::SolveConfig cfg;
        cfg.budget_seconds = budget;
        fill(mcs::bound_jump_search(gg, hh, current_best,
                                    doubling ? mcs::JumpMode::doubling : mcs::JumpMode::plus_one,
                                    cfg),
             out);
        return 0;
    } catch (const std::exception& e) {
        fail(out, e.what());
        return -1;
    }
}

// 1 valid, 0 invalid, -1 error (out of range).
int ref_verify(const ref_graph* g, const ref_graph* h, const int32_t* pairs, int k) {
    try {
        mcs::Mapping m;
        for (int i = 0; i < k; ++i) m.push_back({pairs[2 * i], pairs[2 * i + 1]});
        return mcs::oracle::verify(to_graph(g), to_graph(h), m) ? 1 : 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_bruteforce(const ref_graph* g, const ref_graph* h, int32_t* pairs_out) {
    try {
        auto r = mcs::oracle::mcs_bruteforce(to_graph(g), to_graph(h));
        for (size_t i = 0; i < r.witness.size(); ++i) {
            pairs_out[2 * i] = r.witness[i].v;
            pairs_out[2 * i + 1] = r.witness[i].u;
        }
        return r.size;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// strategy: 0 none, 1 degree, 2 components, 3 block-triangular.
int ref_ordering(const ref_graph* g, int strategy, int32_t* fwd_out) {
    try {
        auto p = mcs::make_ordering(to_graph(g), static_cast<mcs::OrderingStrategy>(strategy));
        for (int i = 0; i < p.size(); ++i) fwd_out[i] = p(i);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Loads a graph file; first call with codes_out == NULL to learn n/flags.
int ref_load_graph_file(const char* path, int format, int32_t* n_out, int32_t* directed_out,
                        int32_t* labeled_out, uint8_t* codes_out, int32_t* labels_out) {
    try {
        mcs::Graph g = mcs::load_graph_file(path, static_cast<mcs::FileFormat>(format));
        *n_out = g.n();
        *directed_out = g.directed();
        *labeled_out = g.labeled();
        if (codes_out)
            for (int u = 0; u < g.n(); ++u)
                for (int v = 0; v < g.n(); ++v) codes_out[(size_t)u * g.n() + v] = g.code(u, v);
        if (labels_out && g.labeled())
            for (int v = 0; v < g.n(); ++v) labels_out[v] = g.label(v);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Serialises through the reference writers (format 0 mivia, 1 text).
int ref_save_graph_file(const ref_graph* g, const char* path, int format) {
    try {
        mcs::save_graph_file(to_graph(g), path, static_cast<mcs::FileFormat>(format));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Label-class refinement KAT hook: refines the initial classes of (g,h) by
// the pairs given in order and reports the final classes as (left set, right
// set) bitmasks (n <= 64) plus compute_bound(k, classes).
int ref_refine_chain(const ref_graph* g, const ref_graph* h, const int32_t* pairs, int k,
                     uint64_t* left_masks, uint64_t* right_masks, int32_t* adjacent,
                     int max_classes, int64_t* bound_out) {
    try {
        mcs::Graph gg = to_graph(g), hh = to_graph(h);
        mcs::ClassState st = mcs::initial_classes(gg, hh);
        for (int i = 0; i < k; ++i) st = mcs::refine(st, pairs[2 * i], pairs[2 * i + 1], gg, hh);
        int c = 0;
        for (const auto& cl : st.classes) {
            if (c >= max_classes) break;
            uint64_t lm = 0, rm = 0;
            for (int j = 0; j < cl.left_len; ++j) lm |= 1ull << st.left[cl.left_start + j];
            for (int j = 0; j < cl.right_len; ++j) rm |= 1ull << st.right[cl.right_start + j];
            left_masks[c] = lm;
            right_masks[c] = rm;
            adjacent[c] = cl.adjacent;
            ++c;
        }
        *bound_out = mcs::compute_bound(k, st.classes);
        return c;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
