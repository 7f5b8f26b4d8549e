// Integration example: the reference's own types driven through the mcsg
// drop-in adapter (include/mcsg_reference_adapter.hpp). Built against the
// reference headers + oracle/_ref/libmcs_ref.so (for mcs::Graph and friends)
// and libmcsg.so. Prints one line per check; exit code 0 = all checks passed.
#include <cstdio>

#include "mcs/graph.hpp"
#include "mcs/heuristics.hpp"
#include "mcs/solve.hpp"
#include "mcsg_reference_adapter.hpp"

int main() {
    using namespace mcs;
    Graph g = random_graph(20, 0.3, 1), h = random_graph(20, 0.3, 2);
    Graph diamond = from_edge_list(4, {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {2, 3}});
    Graph k4 = from_edge_list(4, {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}});
    int fails = 0;
    bool ok = gpu::verify(diamond, k4, {{0, 1}, {1, 2}, {2, 0}});
    std::printf("verify worked pair: %s\n", ok ? "ok" : "FAIL");
    fails += !ok;
    const bool have_gpu = mcsg_device_count() > 0;
    try {
        SolveResult ref = solve(g, h);  // the reference's sequential engine
        SolveResult par = gpu::solve(g, h, {}, MCSG_MODE_PARITY);
        SolveResult thr = gpu::solve(g, h);
        ok = have_gpu && par.size == ref.size && par.stats.recursions == ref.stats.recursions &&
             par.best == ref.best && thr.size == ref.size && gpu::verify(g, h, thr.best);
        std::printf("gpu solve parity: %s (size %d, nodes %llu vs %llu)\n", ok ? "ok" : "FAIL", par.size,
                    (unsigned long long)par.stats.recursions, (unsigned long long)ref.stats.recursions);
        fails += !ok;
        // the reference's RestartDriver through the adapter: identical stats and ranges
        RestartConfig rc;
        rc.seed = 7;
        rc.multiplier = 1.0;
        VisitedRanges vr_ref, vr_gpu;
        rc.ranges_out = &vr_ref;
        SolveResult rref = solve_with_restarts(g, h, rc);
        rc.ranges_out = &vr_gpu;
        SolveResult rgpu = gpu::solve_with_restarts(g, h, rc);
        ok = rgpu.size == rref.size && rgpu.best == rref.best && rgpu.stats.recursions == rref.stats.recursions &&
             rgpu.stats.restarts == rref.stats.restarts && rgpu.stats.visited_ranges == rref.stats.visited_ranges &&
             vr_gpu.runs == vr_ref.runs;
        std::printf("gpu restarts parity: %s (restarts %llu, ranges %llu)\n", ok ? "ok" : "FAIL",
                    (unsigned long long)rgpu.stats.restarts, (unsigned long long)rgpu.stats.visited_ranges);
        fails += !ok;
    } catch (const GraphError& e) {
        // without a device the adapter must raise, never fall back to the CPU
        ok = !have_gpu;
        std::printf("no device -> GraphError: %s (%s)\n", ok ? "ok" : "FAIL", e.what());
        fails += !ok;
    }
    return fails ? 1 : 0;
}
