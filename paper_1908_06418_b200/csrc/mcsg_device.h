// Device-side data layout shared by the host runtime (mcsg_host.cpp) and the
// search kernel (mcsg_kernel.cu). Everything here lives in HBM; the kernel
// stages the hot parts (adjacency rows, vertex keys, the class stack, the
// DFS frames) in shared memory per warp.
//
// Terminology follows the reference (/root/reference/proj):
//   instance  = one (G, H) pair to solve                    (solve.hpp:128)
//   class     = one label class / bidomain (L ⊆ V_G, R ⊆ V_H) (label_classes.hpp:12-20)
//   node      = one counted entry into search_node          (search_core.hpp:130)
//   task      = a frozen subtree (node state + remaining branch plan), the
//               GPU counterpart of SearchTask               (task_queue.hpp:27-48)
//   group     = instances sharing one incumbent size (portfolio members of one
//               pair: SharedBound semantics, solve.hpp:68-81)
#pragma once
#include <cstdint>

namespace mcsg {

constexpr int kMaxN = 64;        // one 64-bit word per bitset row (all configs n <= 45)
constexpr int kMaxDepth = kMaxN + 1;
constexpr int kWarpsPerCta = 4;
// Wide graphs (64 < n <= 255): bitset rows of kWideWords 64-bit words. Vertex
// ids, class counts and bounds still fit one byte (the frame/mapping layout of
// the 64-bit kernel), like the reference's byte-frame engine (K254 accepted,
// K255 rejected: engine_iterative.hpp:9, test_engine_iterative.cpp:40-59).
constexpr int kMaxWideN = 255;
constexpr int kWideWords = 4;

// Per-instance read-only description, packed by the host loader
// (graph.hpp:31-62 codes -> bitsets). 64-bit storage even when the kernel
// runs the 32-bit specialisation (n <= 32); the kernel truncates.
struct InstanceDesc {
    int32_t n_g, n_h;
    int32_t maxp;      // min(n_g, n_h)            (search_core.hpp:105)
    int32_t goal;      // 0 = off                  (search_core.hpp:93)
    int32_t n_init;    // initial classes          (label_classes.cpp:8-39)
    int32_t group;     // incumbent group id
    int32_t prune;     // 0 = disable_pruning      (solve.hpp:122)
    int32_t floor;     // external size floor      (search_core.hpp:25-28)
    uint64_t out_g[kMaxN];  // undirected: adjacency; directed: code bit0 (v -> x)
    uint64_t out_h[kMaxN];
    uint64_t in_g[kMaxN];   // directed only: code bit1 (x -> v)
    uint64_t in_h[kMaxN];
    uint64_t init_l[kMaxN];
    uint64_t init_r[kMaxN];
    uint16_t vkey[kMaxN];   // (255 - deg) << 6 | id: min == select_vertex (label_classes.cpp:69-78)
};

// Per-instance mutable state (results). 16-byte aligned: polls prefetch its
// first 16 bytes with cp.async (which faults on a misaligned source).
struct alignas(16) InstanceState {
    uint32_t map_size;      // size of the mapping stored in map_v/map_u
    int32_t lock;           // spin lock guarding map_* on improvement
    int32_t open_tasks;     // tasks of this instance not yet finished
    int32_t workers;        // warps currently running a task of this instance (fairness)
    unsigned long long nodes;
    unsigned long long t_done_ns;  // %globaltimer when the last task finished
    unsigned long long suspects;   // parity mode: nodes the dead-end monitor found suspect
    uint8_t map_v[kMaxWideN + 1];
    uint8_t map_u[kMaxWideN + 1];
};
static_assert(sizeof(InstanceState) % 16 == 0, "InstanceState rows must stay 16-byte aligned");

// Wide instance description (n <= 255): same header fields as InstanceDesc,
// rows of kWideWords words (the 128-vertex kernel reads the first two).
struct WideDesc {
    int32_t n_g, n_h;
    int32_t maxp;
    int32_t goal;
    int32_t n_init;
    int32_t group;
    int32_t prune;
    int32_t floor;
    uint64_t out_g[kMaxWideN + 1][kWideWords];
    uint64_t out_h[kMaxWideN + 1][kWideWords];
    uint64_t in_g[kMaxWideN + 1][kWideWords];
    uint64_t in_h[kMaxWideN + 1][kWideWords];
    uint64_t init_l[kMaxWideN + 1][kWideWords];
    uint64_t init_r[kMaxWideN + 1][kWideWords];
    uint32_t vkey[kMaxWideN + 1];  // (1023 - deg) << 8 | id  (degree <= 2 * 254 when directed)
};

// Incumbent group (one per solved pair; several instances when a portfolio
// races orderings/strategies on one GPU and shares the size).
struct alignas(16) GroupState {
    uint32_t best;          // monotone size, only raised after a mapping of that size is stored
    uint32_t done;          // 1: max reached, goal reached, suspect, or one member proved optimality
    int32_t winner;         // instance that proved / reached first (-1 none)
    int32_t reached;        // goal probes: 1 when |M| >= goal was found
    // dead-end monitor (heuristics.hpp:30-60), only when a policy is set
    uint32_t suspect;       // 1: the policy fired and stopped the search
    uint32_t epoch;         // restarts so far (RestartDriver, restarts.cpp:35-246)
    unsigned long long nodes;       // nodes counted so far (per poll interval)
    unsigned long long at_improve;  // `nodes` when the incumbent last improved
};

// A frozen subtree: the node's classes and mapping, the selected class and
// vertex, the u candidates not yet tried and whether the "v unmatched"
// continuation still belongs to it (search_core.hpp:183-212).
enum : uint8_t { kTaskRoot = 0, kTaskBranch = 1 };

struct TaskHeader {
    int32_t inst;
    uint8_t kind;
    uint8_t depth;
    uint8_t nc;
    uint8_t sel;
    uint8_t v;
    uint8_t bound;
    uint8_t cont;
    uint8_t fanout;         // 1: donated while many warps waited (the receiver polls early)
    uint64_t cand;          // remaining u candidates (bitset over V_H)
    uint64_t pad1;
};

struct alignas(128) TaskSlot {
    unsigned long long seq;  // Vyukov ring sequence word
    unsigned long long pad[1];
    TaskHeader hdr;          // 32 B
    uint8_t map_v[kMaxN];
    uint8_t map_u[kMaxN];
    uint64_t cls_l[kMaxN];
    uint64_t cls_r[kMaxN];
};

// Wide frozen subtree (n <= 255): the remaining u set and the classes are
// kWideWords words per bitset; hdr.cand is unused.
struct alignas(128) WideSlot {
    unsigned long long seq;
    unsigned long long pad[1];
    TaskHeader hdr;
    uint64_t cand[kWideWords];
    uint8_t map_v[kMaxWideN + 1];
    uint8_t map_u[kMaxWideN + 1];
    uint64_t cls[kMaxWideN][2][kWideWords];  // [class][L, R][word]
};

// Global counters (one set per launch), for the roofline / stats.
struct Counters {
    unsigned long long nodes;
    unsigned long long sum_classes;  // reserved (0)
    unsigned long long splits;       // children materialised (filter_classes writes a level)
    unsigned long long split_classes;// Σ classes moved through shared memory by those
                                     // splits: the child's written + the parent's
                                     // reloaded at the pop back
    unsigned long long donations;
    unsigned long long tasks;
    unsigned long long spills;       // levels placed in the HBM spill area
    unsigned long long t_start_ns;   // min %globaltimer over warps at kernel start
    unsigned long long overflow;     // class-stack overflow (must stay 0)
    unsigned long long ring_stall;   // a producer waited > 2 s for a ring slot (must stay 0)
    unsigned long long bad_task;     // a consumed subtree had an impossible header (must stay 0)
    unsigned long long frozen;       // subtrees frozen into the ring by restarts
    unsigned long long nests_smem, nests_hbm;  // compacted subtrees (64-bit kernel; nests_hbm stays 0: shared-memory nests only)
    unsigned long long stall_pos, stall_head, stall_tail, stall_seq;  // its ticket and the ring state
    unsigned long long idle_cycles;  // Σ over warps of SM cycles spent waiting for a task
    unsigned long long busy_cycles;  // Σ over warps of SM cycles spent running tasks
    unsigned long long peer_pushes;  // improvements pushed to peer devices over NVLink P2P
};

// Control words of one launch, one 128-byte line each so that idle warps
// polling the ring do not contend with busy warps' counters.
struct alignas(128) Line64 {
    unsigned long long v;
};
struct alignas(128) Line32 {
    int32_t v;
};
// The stop line also carries the live external size floor (SharedBound,
// solve.hpp:70-81): every poll prefetches the line, so the floor reaches every
// warp with the stop word at no extra load.
struct alignas(128) StopLine {
    int32_t v;
    int32_t floor;  // raised by warp 0 from the host-mapped shared bound
};
struct Ctl {
    Line64 head;       // ring consumer ticket
    Line64 tail;       // ring producer ticket
    Line32 pending;    // tasks queued + tasks in flight (termination)
    Line32 idle;       // warps waiting for work (donation trigger)
    StopLine stop;     // 0 run, 1 timeout, 2 cancelled, 3 internal error; + live floor
    Line32 next_root;  // root tasks are implicit: instance ids handed out by atomicAdd
    Line32 live;       // instances with unfinished tasks (fairness share)
};

// One segment of the exact restart engine (parity mode; RestartDriver,
// restarts.cpp:35-191). The host keeps the segment pool as position keys —
// the iteration taken at each step from the root, a step being a u child
// (iteration = rank of u in the selected class's R, ascending) or the "v
// unmatched" continuation (iteration = |R|) — and draws the next segment with
// the reference's mt19937_64. The kernel (one warp) replays the key from the
// root classes to the segment's node, enters it (counted, restart check,
// offer, bound, select), resumes its branch loop at `from_iter`, and runs the
// subtree with the reference's per-node restart check: when nodes since the
// last improvement reach mult x max(1, nodes at that improvement) it stops at
// that node's entry and reports the path to it (the iterations below the
// segment's node), from which the host freezes the path into segments and
// records the visited ranges exactly as the reference does.
struct RxState {
    // in
    double mult;                   // RestartConfig::multiplier (<= 0: no restart check)
    unsigned long long nodes0;     // nodes counted before this segment (RestartDriver::nodes)
    unsigned long long at0;        // RestartDriver::at_improvement
    int32_t script_len;            // steps from the root to the segment's node
    int32_t from_iter;             // first iteration still to run at the segment's node
    uint8_t script[kMaxWideN + 1]; // the iterations of those steps
    // out
    int32_t fired;                 // 1: a restart fired at the entry of the path's last node
    int32_t log_len;               // steps below the segment's node to that node (0: the segment's node)
    unsigned long long nodes;      // nodes counted after this segment
    unsigned long long at;         // at_improvement after this segment (before the rearm of a restart)
    uint8_t log[kMaxWideN + 1];    // the iterations of those steps
    uint8_t lp_at[kMaxWideN + 2];  // kernel scratch: path length at each open level
};

constexpr int kMaxPeers = 16;
constexpr int kMaxLadder = 32;  // probe targets of one parallel binary-search round

struct KernelParams {
    const InstanceDesc* inst;   // n <= 64 kernels
    const WideDesc* winst;      // wide kernels
    InstanceState* ist;
    GroupState* grp;
    TaskSlot* slots;            // n <= 64 kernels
    WideSlot* wslots;           // wide kernels
    Ctl* ctl;
    uint32_t cap_mask;       // ring capacity - 1 (power of two)
    unsigned long long ring_watchdog_ns;  // a producer waiting longer for a slot aborts the launch
    int32_t n_inst;
    int32_t n_roots;         // instances handed out as root tasks (0: the ring was pre-seeded)
    // Cross-device incumbent of group 0 (one instance sharded over devices, or
    // portfolio members on different devices): other devices' GroupState,
    // reachable over NVLink P2P. Sizes are pushed with system-scope atomicMax.
    GroupState* peer_grp[kMaxPeers];
    int32_t n_peers;
    int32_t peer_done_on_complete;  // portfolio: the first device to finish proves for all
    const volatile int32_t* cancel;  // host-mapped cancel flag (may be null)
    // Live SharedBound (solve.hpp:70-81; may be null): warp 0 reads the
    // host-mapped size at its polls and raises ctl->stop.floor, which every
    // warp folds into its prune threshold (never into offers); every stored
    // improvement is pushed back to the host with a system-scope atomicMax.
    const volatile int32_t* ext_floor;
    int32_t* ext_best;
    unsigned long long budget_ns;    // per-warp deadline = warp start + budget, 0 = none
    uint64_t* spill;         // per-warp HBM spill area for class levels (64-bit and wide kernels)
    int32_t spill_classes;   // classes per warp in the spill area
    int32_t smem_classes;    // classes per warp in shared memory
    int32_t donate;          // 0 = parity mode (no donation: exact sequential semantics)
    int32_t poll_interval;   // poll global state every poll_interval nodes
    Counters* counters;
    // dead-end policy (DeadEndPolicy, heuristics.hpp:30-38; deadend_check,
    // heuristics.cpp:103-112): suspect when nodes since the last improvement
    // reach deadend_abs, or deadend_rel * max(1, nodes at the improvement)
    int32_t deadend_kind;            // 0 off, 1 absolute, 2 relative
    int32_t deadend_stop;            // 1: a suspect node stops the search (a jump follows)
    unsigned long long deadend_abs;  // absolute threshold
    double deadend_rel;              // relative multiplier
    // Restarts (RestartConfig::multiplier, heuristics.hpp:90-102): a restart
    // is due when the group's nodes since its last improvement reach
    // restart_mult x max(1, nodes at that improvement); every warp of the
    // group then freezes its open path into the ring (exactly-once segments)
    // and resumes with the oldest queued subtree. 0 = off.
    double restart_mult;
    // 64-bit kernel: run subtrees whose live vertex sets fit 32 bits with
    // the 32-bit policy (CompactSearch, nested in the task): a level is
    // compacted when its bound exceeds the prune threshold by at least
    // `compact` (a small slack means a small subtree, where the compaction
    // costs more than it saves); 0 = off
    int32_t compact;
    // test knob: nest only when the compact stack needs at most this many
    // 32-bit entries (0 = no limit); larger subtrees run in the 64-bit policy
    int32_t compact_room_cap;
    // Probe ladder (parallel binary search over goal probes):
    // every group of the launch is a probe of the same pair with its own goal,
    // and the ladder spans every device of the round. Entry k (ascending goal)
    // is ladder_grp[k], local or a peer's GroupState over NVLink P2P. A probe
    // that reaches its goal marks every entry with a goal <= its own reached
    // (and done); a probe that exhausts its tree without reaching marks every
    // entry with a goal >= its own done (failed). ladder_n = 0: no ladder.
    int32_t ladder_n;
    int32_t ladder_goal[kMaxLadder];
    GroupState* ladder_grp[kMaxLadder];
    // Exact restart engine (parity mode, one instance): the segment to run;
    // null otherwise.
    RxState* rx;
};

}  // namespace mcsg
