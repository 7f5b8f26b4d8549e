/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the McSplit search path.
 *
 * A plain-C restatement of the reference solver's sequential algorithm
 * (/root/reference/proj, see mcs_oracle.c for per-function file:line
 * citations). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker or
 * the timed CPU baseline — never as part of the product path.
 *
 * Parity status: PINNED. tests/test_oracle.py checks this restatement against
 * golden vectors produced by the unmodified reference (oracle/_ref, see
 * tests/golden/make_golden.py): optimum sizes, exact node counts
 * (stats.recursions), mappings, orderings and the reference's own KATs.
 */
#ifndef MCS_ORACLE_H
#define MCS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t n;
    int32_t directed;       /* 0 undirected (codes 0/1), 1 directed (codes 0..3) */
    const uint8_t* codes;   /* n*n row-major: code(u,v) = codes[u*n+v] */
    const int32_t* labels;  /* n labels or NULL (unlabelled) */
} orc_graph;

typedef struct {
    double budget_s;        /* <= 0: immediate timeout; >= 1e8: unlimited */
    int64_t goal;           /* 0 off */
    int32_t prune;          /* 1 normal, 0 exhaustive (disable_pruning) */
    int32_t order;          /* 0 none, 1 degree, 2 components, 3 block-triangular */
    int64_t floor_size;     /* external shared bound (SharedBound), 0 = none */
    const volatile int32_t* cancel;
} orc_options;

typedef struct {
    int32_t status;         /* 0 optimal, 1 timeout, 2 cancelled, -1 error */
    int32_t size;
    int32_t pairs[2 * 256]; /* (v in G, u in H) in original ids */
    uint64_t nodes;         /* == reference stats.recursions */
    uint64_t probes;
    double wall_s;
    /* instrumentation (design data, not reference fields) */
    uint64_t sum_classes;   /* sum over counted nodes of live classes */
    uint64_t sum_splits;    /* sum over children built of parent classes split */
    uint64_t pruned_at_entry;
    uint64_t children_built;
    int32_t max_depth;
    int32_t max_stack_classes;
} orc_result;

void orc_random_graph(int n, double density, uint64_t seed, int directed, int label_count,
                      uint8_t* codes_out, int32_t* labels_out);
void orc_random_permutation(int n, uint64_t seed, int32_t* fwd_out);
int orc_degree(const orc_graph* g, int v);
int orc_ordering(const orc_graph* g, int strategy, int32_t* fwd_out);

/* mcs::solve (proj/src/solve.cpp:85-129). Returns 0, or -1 on input error. */
int orc_solve(const orc_graph* g, const orc_graph* h, const orc_options* o, orc_result* r);
/* mcs::solve_goal_directed (proj/src/solve.cpp:131-168). */
int orc_solve_goal_directed(const orc_graph* g, const orc_graph* h, const orc_options* o,
                            orc_result* r);
/* mcs::bound_jump_search (proj/src/heuristics.cpp:114-185); doubling 0 = plus_one. */
int orc_bound_jump(const orc_graph* g, const orc_graph* h, int current_best, int doubling,
                   const orc_options* o, orc_result* r);
/* mcs::solve_with_restarts (proj/src/restarts.cpp:195-246): seeded segment
 * draws (mt19937_64), restart rule, visited ranges. r->probes carries
 * stats.visited_ranges; ranges_out (may be NULL) receives each run as
 * [len(lo), lo..., len(hi), hi...] (iterations per depth), *ranges_len the
 * words needed. */
int orc_solve_with_restarts(const orc_graph* g, const orc_graph* h, const orc_options* o, uint64_t seed,
                            double multiplier, orc_result* r, uint64_t* restarts, int32_t* ranges_out,
                            int64_t ranges_cap, int64_t* ranges_len);
/* mcs::oracle::verify (proj/src/oracle.cpp:8-24): 1 valid, 0 invalid, -1 out of range. */
int orc_verify(const orc_graph* g, const orc_graph* h, const int32_t* pairs, int k);
/* mcs::oracle::mcs_bruteforce (proj/src/oracle.cpp:76-86): size, or -1 above n=10. */
int orc_bruteforce(const orc_graph* g, const orc_graph* h, int32_t* pairs_out);

#ifdef __cplusplus
}
#endif
#endif
