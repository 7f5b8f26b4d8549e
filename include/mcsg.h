/* mcsg — B200-native McSplit (maximum common induced subgraph) solver.
 *
 * C ABI of the drop-in boundary. Plain pointers and sizes, caller-owned
 * buffers, no allocation across the ABI, integer status codes. Each entry
 * point replaces one public entry of the reference C++ solver
 * (/root/reference/proj/include/mcs/...):
 *
 *   mcsg_solve                 mcs::solve(g, h, SolveConfig)              solve.hpp:128
 *                              (mode MCSG_MODE_PARITY reproduces it node-for-node;
 *                               MCSG_MODE_THROUGHPUT is the GPU work-sharing engine)
 *   mcsg_solve_parallel        mcs::solve_parallel(g, h, ParallelConfig)  engine_parallel.hpp:16
 *   mcsg_solve_batch           run_suite's per-instance loop              bench.cpp:74-122
 *                              (many pairs in one persistent launch)
 *   mcsg_solve_goal_directed   mcs::solve_goal_directed                   solve.hpp:132
 *   mcsg_bound_jump            mcs::bound_jump_search                     heuristics.hpp:69
 *   mcsg_probe_parallel        bound_jump_search's bracket, probed in parallel (many targets
 *                              per round, over GPUs)                      heuristics.cpp:114-185
 *   mcsg_solve_with_restarts   mcs::solve_with_restarts                   heuristics.hpp:107
 *                              (parity mode: the reference's RestartDriver exactly — seeded
 *                               segment draws, recursions, restarts, visited ranges)
 *   mcsg_portfolio             mcs::run_portfolio (race semantics)        portfolio.hpp:100
 *   mcsg_verify                mcs::oracle::verify                        oracle.hpp:16
 *   mcsg_random_graph          mcs::random_graph                          graph.hpp:99
 *   mcsg_random_permutation    mcs::random_permutation                    graph.hpp:102
 *   mcsg_ordering              mcs::make_ordering                         heuristics.hpp:26
 *   mcsg_load_graph_file       mcs::load_graph_file                       graph_io.hpp:33
 *   mcsg_save_graph_file       mcs::save_graph_file                       graph_io.hpp:34
 *   mcsg_pack_graph            (the loader's bitset packing; no reference counterpart)
 *   mcsg_pack_graph_words      (the same, multi-word rows for 64 < n <= 255)
 *
 * Graphs use the reference's storage: an n*n row-major byte matrix of
 * adjacency codes (graph.hpp:40,60): 0 none; undirected 1 = edge; directed
 * 1 forward (u->v), 2 backward, 3 both, mirror-consistent.
 *
 * Errors: functions return MCSG_ERROR (and mcsg_last_error() explains) where
 * the reference throws GraphError / ParseError; timeouts and cancellation are
 * statuses, not errors (solve.hpp:23). No CPU fallback: without a usable CUDA
 * device every solve returns MCSG_ERROR.
 */
#ifndef MCSG_H
#define MCSG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCSG_ABI_VERSION 5

/* status codes (mirror mcs_main.cpp:22-24 exit codes; SolveStatus solve.hpp:23) */
#define MCSG_OPTIMAL 0
#define MCSG_TIMEOUT 2
#define MCSG_ERROR 3
#define MCSG_CANCELLED 4

/* mcsg_graph.flags */
#define MCSG_DIRECTED 1u
#define MCSG_LABELED 2u

/* mcsg_options.mode */
#define MCSG_MODE_THROUGHPUT 0 /* all warps, subtree donation, shared incumbent */
#define MCSG_MODE_PARITY 1     /* one warp per instance: reference node order and counts */

/* mcsg_options.order — OrderingStrategy (solve.hpp:116) */
#define MCSG_ORDER_NONE 0
#define MCSG_ORDER_DEGREE 1
#define MCSG_ORDER_COMPONENTS 2
#define MCSG_ORDER_BLOCK 3

#define MCSG_MAX_N 255

typedef struct mcsg_graph {
    int32_t n;
    uint32_t flags;         /* MCSG_DIRECTED | MCSG_LABELED */
    const uint8_t* codes;   /* n*n row-major codes (graph.hpp:60) */
    const int32_t* labels;  /* n vertex labels when MCSG_LABELED, else NULL */
} mcsg_graph;

typedef struct mcsg_options {
    double budget_s;                /* SolveConfig::budget_seconds; <= 0 immediate timeout */
    int32_t order;                  /* MCSG_ORDER_* */
    int32_t mode;                   /* MCSG_MODE_* */
    int32_t goal;                   /* 0 off; > 0: stop at |M| >= goal, prune below it */
    int32_t disable_pruning;        /* SolveConfig::disable_pruning */
    int32_t floor_size;             /* SolveConfig::shared_bound value (size floor) */
    int32_t device;                 /* CUDA ordinal, -1 = current */
    int32_t max_warps;              /* 0 = every resident warp */
    int32_t smem_classes;           /* 0 = auto: class-stack entries per warp in smem */
    uint64_t seed;                  /* restarts:<seed> portfolio member: donation order */
    const volatile int32_t* cancel; /* SolveConfig::cancel; polled by the kernel */
    /* Multi-GPU (one process drives every device; incumbent sizes travel over
     * NVLink P2P). n_devices > 1: mcsg_solve shards ONE instance — the host
     * expands the top of the tree into `frontier` subtrees per device, dealt
     * round-robin — and mcsg_portfolio spreads its members over the devices
     * (first member to finish proves for all). Repeated ordinals are allowed
     * (shards then run one after another on that device). */
    int32_t n_devices;
    int32_t devices[16];
    int32_t frontier;               /* subtrees per device, 0 = 256 */
    /* Dead-end handling (DeadEndPolicy heuristics.hpp:30-38, run_engine's
     * forecast-then-jump composition portfolio.cpp:136-155): with a jump mode
     * set, the search stops once the nodes since the last improvement reach
     * deadend_abs (or deadend_rel x the nodes at that improvement) and a bound
     * jump (MCSG_JUMP_*) resumes from the incumbent. */
    uint64_t deadend_abs;           /* 0 = off */
    double deadend_rel;             /* 0 = off */
    int32_t deadend_jump;           /* 0 none, 1 plus_one, 2 doubling */
    /* Restarts (RestartConfig::multiplier, heuristics.hpp:90-102; throughput
     * mode): when the nodes since the last improvement reach multiplier x
     * max(1, nodes at that improvement), every warp freezes its open path
     * into the task ring and resumes with the oldest queued subtree — the
     * search stays complete. 0 = off. */
    double restart_multiplier;
    /* SolveConfig::shared_bound (SharedBound, solve.hpp:70-81), live: may be
     * NULL. While the call runs the host mirrors *shared_bound into the
     * kernel, which folds it into its prune threshold at every poll (a size
     * floor raised by other engines mid-run), and raises *shared_bound
     * (atomic max) to the size of every mapping the search stores. floor_size
     * is the same floor fixed at call start. */
    volatile int32_t* shared_bound;
    /* > 1: use 1/warp_share of the resident warps, so that several engines
     * (one host thread each) can run concurrently on one GPU — concurrent
     * calls on one device take separate device contexts. 0/1 = every warp. */
    int32_t warp_share;
    /* DeadEndPolicy::Kind (heuristics.hpp:30-38): 0 = from the fields above
     * (deadend_abs > 0 absolute, deadend_rel > 0 relative), 1 absolute
     * (deadend_abs may then be 0: every node is suspect), 2 relative. Parity
     * mode runs the reference's monitor per node (note_recursion /
     * deadend_check before the node's offer, search_core.hpp:133-141): with a
     * jump it stops at the reference's node, without one it counts suspect
     * nodes (result.deadend_suspects). Throughput mode checks at polls and
     * only stops when a jump follows. */
    int32_t deadend_kind;
} mcsg_options;

#define MCSG_JUMP_PLUS_ONE 1
#define MCSG_JUMP_DOUBLING 2

typedef struct mcsg_stats {
    uint64_t nodes;          /* stats.recursions: counted search nodes */
    uint64_t sum_classes;    /* reserved (0) */
    uint64_t splits;         /* children materialised (filter_classes writing a class level) */
    uint64_t split_classes;  /* Σ classes moved through shared memory by those splits: the
                              * child's written + the parent's reloaded at the pop back
                              * (the shared-memory roofline's per-node bytes) */
    uint64_t donations;      /* subtrees handed to idle warps */
    uint64_t tasks;          /* tasks executed (roots + donated) */
    uint64_t spills;         /* class levels placed in the HBM spill area */
    uint64_t probes;         /* goal-directed / bound-jump probes */
    double wall_s;           /* host wall time of the call */
    double kernel_s;         /* device time of the search kernel(s) (CUDA events) */
    double h2d_s;            /* host->device staging time */
    int32_t warps;           /* resident warps launched */
    int32_t ctas;
    int32_t smem_per_cta;
    int32_t smem_classes;
    uint64_t h2d_bytes;      /* bytes copied host->device by the call */
    uint64_t d2h_bytes;      /* bytes copied device->host by the call */
    uint64_t launches;       /* kernels launched by the call */
    uint64_t busy_cycles;    /* Σ over warps of SM cycles running tasks */
    uint64_t idle_cycles;    /* Σ over warps of SM cycles waiting for a task */
    uint64_t restarts;       /* restart events (group 0 of the call) */
    uint64_t frozen;         /* subtrees frozen into the ring by restarts */
    double idle_s;           /* idle_cycles / the device's SM clock (SearchStats::idle_seconds) */
    double busy_s;           /* busy_cycles / the device's SM clock */
    uint64_t peer_pushes;    /* incumbent improvements pushed to peer GPUs over NVLink P2P */
    uint64_t visited_ranges; /* SearchStats::visited_ranges (mcsg_solve_with_restarts) */
} mcsg_stats;

typedef struct mcsg_result {
    int32_t status;          /* MCSG_OPTIMAL / MCSG_TIMEOUT / MCSG_CANCELLED / MCSG_ERROR */
    int32_t size;
    int32_t pairs[2 * MCSG_MAX_N]; /* (v in G, u in H) in ORIGINAL ids */
    uint64_t nodes;          /* nodes of this instance */
    double solve_s;          /* device time from launch to this instance's proof */
    int32_t flags;           /* MCSG_RESULT_SUSPECT: stopped by the dead-end policy */
    int32_t probes;          /* goal / jump probes run for this result */
    uint64_t deadend_suspects; /* SearchStats::deadend_suspects (parity mode: suspect nodes) */
} mcsg_result;

#define MCSG_RESULT_SUSPECT 1

/* ---- solving ---------------------------------------------------------- */
int32_t mcsg_solve(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                   mcsg_result* out, mcsg_stats* stats);
int32_t mcsg_solve_parallel(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                            mcsg_result* out, mcsg_stats* stats);
/* count pairs solved in one launch; outs[count] */
int32_t mcsg_solve_batch(int32_t count, const mcsg_graph* gs, const mcsg_graph* hs,
                         const mcsg_options* opt, mcsg_result* outs, mcsg_stats* stats);
int32_t mcsg_solve_goal_directed(const mcsg_graph* g, const mcsg_graph* h,
                                 const mcsg_options* opt, mcsg_result* out, mcsg_stats* stats);
int32_t mcsg_bound_jump(const mcsg_graph* g, const mcsg_graph* h, int32_t current_best,
                        int32_t doubling, const mcsg_options* opt, mcsg_result* out,
                        mcsg_stats* stats);
/* Parallel binary search over goal probes (bound_jump_search's bracket,
 * heuristics.cpp:114-185, probed `width` targets at a time): each round
 * probes up to width (<= 32; 0 = max(8, devices)) targets of the open bracket
 * (lower, upper] concurrently — dealt over opt->n_devices GPUs (one GPU when
 * 0) as independent groups of one launch per device. A reached target implies
 * every lower target, an exhausted one every higher target, across devices
 * over NVLink P2P, so each probe stops once its answer is implied. Starts from
 * current_best (a size known reachable); result.probes = targets probed.
 * Throughput mode only. */
int32_t mcsg_probe_parallel(const mcsg_graph* g, const mcsg_graph* h, int32_t current_best, int32_t width,
                            const mcsg_options* opt, mcsg_result* out, mcsg_stats* stats);
/* mcs::solve_with_restarts (heuristics.hpp:107, restarts.cpp:195-246).
 * opt->restart_multiplier is RestartConfig::multiplier (<= 0: no restarts) and
 * opt->seed RestartConfig::seed. MCSG_MODE_PARITY reproduces the reference's
 * RestartDriver exactly: the segment pool is drawn with the reference's seeded
 * mt19937_64, each segment runs on the GPU with the per-node restart check,
 * and result/stats carry the reference's recursions, restarts and
 * visited_ranges; ranges_out (may be NULL; ranges_cap int32 words) receives
 * the VisitedRanges runs in insertion order, each run as [len(lo), lo...,
 * len(hi), hi...] — a PositionKey is the iteration taken at each depth
 * (heuristics.hpp:77), INT32_MAX for successor({}) — and *ranges_len the words
 * needed. MCSG_MODE_THROUGHPUT runs the work-sharing engine's restart epochs
 * (every warp freezes its open path into the ring); visited_ranges = 1 for a
 * completed search. */
int32_t mcsg_solve_with_restarts(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                                 mcsg_result* out, mcsg_stats* stats, int32_t* ranges_out, int64_t ranges_cap,
                                 int64_t* ranges_len);
/* Races `count` member strategies of ONE pair in one launch with a shared
 * incumbent size; first member to prove wins (portfolio.cpp:249-292).
 * orders[i] in MCSG_ORDER_*; seeds[i] != 0 gives member i a seeded search
 * order (the restarts:<seed> member); either array may be NULL; winner_out may
 * be NULL. */
int32_t mcsg_portfolio(const mcsg_graph* g, const mcsg_graph* h, int32_t count,
                       const int32_t* orders, const uint64_t* seeds, const mcsg_options* opt,
                       mcsg_result* out, int32_t* winner_out, mcsg_stats* stats);

/* ---- graph core / loader ---------------------------------------------- */
/* 1 valid, 0 invalid, MCSG_ERROR-style -1 on out-of-range vertices */
int32_t mcsg_verify(const mcsg_graph* g, const mcsg_graph* h, const int32_t* pairs, int32_t k);
int32_t mcsg_random_graph(int32_t n, double density, uint64_t seed, uint32_t flags,
                          int32_t label_count, uint8_t* codes_out, int32_t* labels_out);
int32_t mcsg_random_permutation(int32_t n, uint64_t seed, int32_t* fwd_out);
int32_t mcsg_ordering(const mcsg_graph* g, int32_t strategy, int32_t* fwd_out);
/* format: 0 mivia, 1 text, 2 auto-detect (FileFormat, graph_io.hpp:31).
 * Two-phase: call with codes_out == NULL to learn n and flags, then again with
 * buffers of n*n bytes (and n labels when MCSG_LABELED). */
int32_t mcsg_load_graph_file(const char* path, int32_t format, int32_t* n_out,
                             uint32_t* flags_out, uint8_t* codes_out, int32_t* labels_out);
int32_t mcsg_save_graph_file(const mcsg_graph* g, const char* path, int32_t format);
/* The loader's device form: 64-bit adjacency rows. out_rows[n] gets the
 * undirected adjacency / directed forward bits; in_rows[n] (may be NULL)
 * the directed backward bits. */
int32_t mcsg_pack_graph(const mcsg_graph* g, uint64_t* out_rows, uint64_t* in_rows);
/* The same for any n <= MCSG_MAX_N: row v is words[v*words .. v*words+words),
 * bit x%64 of word x/64 (the wide kernels' form). words >= ceil(n/64). */
int32_t mcsg_pack_graph_words(const mcsg_graph* g, int32_t words, uint64_t* out_rows, uint64_t* in_rows);

/* ---- runtime ------------------------------------------------------------ */
const char* mcsg_last_error(void);
/* class of the last error: GraphError, ParseError (graph_io.hpp:11) or CUDA runtime */
#define MCSG_ERR_GRAPH 1
#define MCSG_ERR_PARSE 2
#define MCSG_ERR_CUDA 3
int32_t mcsg_last_error_kind(void);
int32_t mcsg_abi_version(void);
/* number of usable CUDA devices (0 when none) */
int32_t mcsg_device_count(void);
/* release every device context this process created */
void mcsg_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* MCSG_H */
