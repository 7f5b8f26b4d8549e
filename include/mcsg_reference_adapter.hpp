// Drop-in adapter: the reference's C++ entry points on top of the mcsg C ABI.
//
// A maintainer of the reference (proj/, C++20) includes this header and links
// libmcsg.so; nothing else in the reference changes. It converts the
// reference's types at the boundary:
//
//   mcs::Graph (graph.hpp:31-62)         -> mcsg_graph (n*n codes, labels)
//   mcs::SolveConfig (solve.hpp:118-125) -> mcsg_options
//   mcsg_result                          -> mcs::SolveResult (solve.hpp:57-66)
//
// and raises mcs::GraphError where the C ABI reports MCSG_ERROR, as the
// reference does (solve.cpp:94, portfolio.cpp:75). Timeout and cancellation
// stay statuses. SolveConfig::visitor has no GPU counterpart (per-node host
// callbacks cannot run inside the kernel) and is rejected.
#pragma once

#include <atomic>
#include <chrono>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mcs/graph.hpp"
#include "mcs/heuristics.hpp"
#include "mcs/solve.hpp"
#include "mcsg.h"

namespace mcs::gpu {

struct GraphBuffer {
    std::vector<uint8_t> codes;
    std::vector<int32_t> labels;
    mcsg_graph view{};

    explicit GraphBuffer(const Graph& g) {
        const int n = g.n();
        codes.resize(size_t(n) * size_t(n));
        for (int u = 0; u < n; ++u)
            for (int v = 0; v < n; ++v) codes[size_t(u) * n + v] = g.code(u, v);
        view.n = n;
        view.flags = (g.directed() ? MCSG_DIRECTED : 0u) | (g.labeled() ? MCSG_LABELED : 0u);
        view.codes = codes.data();
        if (g.labeled()) {
            labels.assign(g.labels()->begin(), g.labels()->end());
            view.labels = labels.data();
        }
    }
};

inline mcsg_options to_options(const SolveConfig& cfg, int mode) {
    if (cfg.visitor) throw GraphError("mcs::gpu: NodeVisitor hooks are not supported on the GPU engine");
    mcsg_options o{};
    o.budget_s = cfg.budget_seconds;
    o.order = static_cast<int32_t>(cfg.order);
    o.mode = mode;
    o.disable_pruning = cfg.disable_pruning ? 1 : 0;
    o.floor_size = cfg.shared_bound ? static_cast<int32_t>(cfg.shared_bound->get()) : 0;
    o.shared_bound = nullptr;  // set by CancelBridge when cfg.shared_bound is given
    o.device = -1;
    o.cancel = nullptr;  // set by CancelBridge when cfg.cancel is given
    return o;
}

// SolveConfig::cancel is a std::atomic<bool> and SolveConfig::shared_bound a
// SharedBound (atomic long long); the ABI polls int32s. A small watcher thread
// mirrors them for the duration of a call: the cancel flag and the bound's
// rises in, the kernel's stored improvements out (SharedBound::bump), so a
// GPU member of a CPU portfolio sees and feeds mid-run improvements.
class CancelBridge {
public:
    CancelBridge(const std::atomic<bool>* src, mcsg_options& o, SharedBound* bound = nullptr)
        : src_(src), bound_(bound) {
        if (!src_ && !bound_) return;
        if (src_) o.cancel = &flag_;
        if (bound_) {
            shared_ = static_cast<int32_t>(bound_->get());
            o.shared_bound = &shared_;
        }
        watcher_ = std::thread([this] {
            while (!done_.load()) {
                sync();
                std::this_thread::sleep_for(std::chrono::microseconds(200));
            }
            sync();
        });
    }
    ~CancelBridge() {
        done_.store(true);
        if (watcher_.joinable()) watcher_.join();
    }

private:
    void sync() {
        if (src_ && src_->load()) flag_ = 1;
        if (!bound_) return;
        const int32_t mine = __atomic_load_n(&shared_, __ATOMIC_ACQUIRE);
        bound_->bump(mine);  // the kernel's improvements out
        const long long ext = bound_->get();
        int32_t cur = mine;  // other engines' rises in (atomic max: the library writes too)
        while (ext > cur && !__atomic_compare_exchange_n(&shared_, &cur, static_cast<int32_t>(ext), true,
                                                         __ATOMIC_RELEASE, __ATOMIC_ACQUIRE)) {
        }
    }

    const std::atomic<bool>* src_;
    SharedBound* bound_;
    volatile int32_t flag_ = 0;
    volatile int32_t shared_ = 0;
    std::atomic<bool> done_{false};
    std::thread watcher_;
};

inline SolveResult to_result(const mcsg_result& r, const mcsg_stats& st) {
    SolveResult out;
    out.status = r.status == MCSG_TIMEOUT     ? SolveStatus::timeout
                 : r.status == MCSG_CANCELLED ? SolveStatus::cancelled
                                              : SolveStatus::optimal;
    out.size = r.size;
    for (int k = 0; k < r.size; ++k) out.best.push_back({r.pairs[2 * k], r.pairs[2 * k + 1]});
    out.stats.recursions = r.nodes;
    out.stats.wall_seconds = st.wall_s;
    out.stats.probes = st.probes;
    out.stats.tasks_published = st.donations;                    // subtrees handed to idle warps
    out.stats.idle_seconds = st.idle_s;  // Σ warps' wait for work (cycles / the device's SM clock)
    out.stats.deadend_suspects = (r.flags & MCSG_RESULT_SUSPECT) ? 1 : 0;
    if (out.status == SolveStatus::optimal) out.stats.visited_ranges = 1;  // the whole tree, exactly once
    return out;
}

inline void check(int32_t rc) {
    if (rc == MCSG_ERROR) throw GraphError(std::string("mcs::gpu: ") + mcsg_last_error());
}

// mcs::solve (solve.hpp:128). MCSG_MODE_PARITY reproduces the reference's
// node order and stats.recursions; the default is the all-warp engine.
inline SolveResult solve(const Graph& g, const Graph& h, const SolveConfig& cfg = {},
                         int mode = MCSG_MODE_THROUGHPUT) {
    GraphBuffer gb(g), hb(h);
    mcsg_options o = to_options(cfg, mode);
    CancelBridge bridge(cfg.cancel, o, cfg.shared_bound);
    mcsg_result r{};
    mcsg_stats st{};
    check(mcsg_solve(&gb.view, &hb.view, &o, &r, &st));
    return to_result(r, st);
}

// mcs::solve_goal_directed (solve.hpp:132).
inline SolveResult solve_goal_directed(const Graph& g, const Graph& h, const SolveConfig& cfg = {}) {
    GraphBuffer gb(g), hb(h);
    mcsg_options o = to_options(cfg, MCSG_MODE_THROUGHPUT);
    CancelBridge bridge(cfg.cancel, o, cfg.shared_bound);
    mcsg_result r{};
    mcsg_stats st{};
    check(mcsg_solve_goal_directed(&gb.view, &hb.view, &o, &r, &st));
    return to_result(r, st);
}

// mcs::bound_jump_search (heuristics.hpp:69).
inline SolveResult bound_jump_search(const Graph& g, const Graph& h, int current_best, JumpMode mode,
                                     const SolveConfig& cfg = {}) {
    GraphBuffer gb(g), hb(h);
    mcsg_options o = to_options(cfg, MCSG_MODE_THROUGHPUT);
    CancelBridge bridge(cfg.cancel, o, cfg.shared_bound);
    mcsg_result r{};
    mcsg_stats st{};
    check(mcsg_bound_jump(&gb.view, &hb.view, current_best, mode == JumpMode::doubling ? 1 : 0, &o,
                          &r, &st));
    return to_result(r, st);
}

// mcs::solve_with_restarts (heuristics.hpp:107). MCSG_MODE_PARITY (the
// default here) is the reference's RestartDriver exactly: the same seeded
// segment draws, recursions, restarts and visited ranges; with
// config.ranges_out the VisitedRanges runs are filled in the reference's order.
inline SolveResult solve_with_restarts(const Graph& g, const Graph& h, const RestartConfig& config,
                                       int mode = MCSG_MODE_PARITY) {
    if (config.visitor) throw GraphError("mcs::gpu: NodeVisitor hooks are not supported on the GPU engine");
    GraphBuffer gb(g), hb(h);
    SolveConfig base;
    base.budget_seconds = config.budget_seconds;
    base.order = config.order;
    base.disable_pruning = config.disable_pruning;
    base.shared_bound = config.shared_bound;
    mcsg_options o = to_options(base, mode);
    o.seed = config.seed;
    o.restart_multiplier = config.multiplier;
    CancelBridge bridge(config.cancel, o, config.shared_bound);
    mcsg_result r{};
    mcsg_stats st{};
    std::vector<int32_t> words(config.ranges_out ? size_t(1) << 16 : 0);
    int64_t need = 0;
    check(mcsg_solve_with_restarts(&gb.view, &hb.view, &o, &r, &st, words.data(), int64_t(words.size()), &need));
    if (config.ranges_out && need > int64_t(words.size())) {  // deterministic: again with room
        words.resize(size_t(need));
        check(mcsg_solve_with_restarts(&gb.view, &hb.view, &o, &r, &st, words.data(), need, &need));
    }
    SolveResult out = to_result(r, st);
    out.stats.recursions = st.nodes;
    out.stats.restarts = st.restarts;
    out.stats.visited_ranges = st.visited_ranges;
    out.stats.seed = config.seed;
    if (config.ranges_out) {
        auto key = [&](size_t& i) {
            PositionKey k;
            const int32_t len = words[i++];
            for (int32_t d = 0; d < len; ++d) k.emplace_back(d, words[i++]);
            return k;
        };
        for (size_t i = 0; i < size_t(need);) {
            PositionKey lo = key(i);
            PositionKey hi = key(i);
            config.ranges_out->add(std::move(lo), std::move(hi));
        }
    }
    return out;
}

// oracle::verify (oracle.hpp:16) through the library's host verifier.
inline bool verify(const Graph& g, const Graph& h, const Mapping& m) {
    GraphBuffer gb(g), hb(h);
    std::vector<int32_t> pairs;
    for (const VtxPair& p : m) {
        pairs.push_back(p.v);
        pairs.push_back(p.u);
    }
    const int32_t rc = mcsg_verify(&gb.view, &hb.view, pairs.data(), int32_t(m.size()));
    if (rc < 0) throw GraphError(std::string("verify: ") + mcsg_last_error());
    return rc == 1;
}

}  // namespace mcs::gpu
