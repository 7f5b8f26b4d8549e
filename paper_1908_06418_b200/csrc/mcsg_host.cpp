// Host runtime and C ABI of the B200 McSplit solver.
//
// One device context per GPU owns the HBM working set of the persistent search
// kernel (instance table, results, the subtree ring, per-warp spill areas)
// and a pinned staging area. A call packs its pairs (loader -> bitsets),
// stages them with one async H2D copy, launches the kernel once, mirrors the
// caller's cancel flag into host-mapped memory while it runs, and copies the
// per-instance results back. Orderings are applied host-side before packing
// and undone on the returned mapping (with_ordering, search_core.hpp:72-81);
// every returned mapping is re-verified on the host (oracle.cpp:8-24 rules)
// before it leaves the library.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <thread>

#include "../../include/mcsg.h"
#include "mcsg_device.h"
#include "mcsg_frontier.hpp"
#include "mcsg_graph.hpp"

namespace mcsg {

// kernel flavours by bitset width (mcsg_kernel.cu): 32, 64, 128, 256
int kernel_occupancy(int bits, bool directed, int smem_classes);
int kernel_smem_per_warp(int bits, bool directed, int smem_classes);
int kernel_smem_fixed(int bits, bool directed);
int kernel_class_bytes(int bits);
cudaError_t kernel_launch(int bits, bool directed, bool parity, const KernelParams& p, int ctas, cudaStream_t st);
cudaError_t ring_reset(TaskSlot* slots, uint32_t cap, Counters* c, cudaStream_t st);
cudaError_t ring_reset_wide(WideSlot* slots, uint32_t cap, Counters* c, cudaStream_t st);

namespace {

thread_local std::string t_err;
thread_local int t_err_kind = 0;

struct CudaErr : Error {
    explicit CudaErr(const std::string& w) : Error(w) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaErr(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr uint32_t kRingCap = 16384;                      // power of two
constexpr uint32_t kWideRingCap = 4096;                   // wide slots are 17 KB
constexpr int kSpillClasses = kMaxDepth * kMaxN;          // 64-bit kernel: worst-case stack, no overflow possible
constexpr int kMaxSlots = 4;                              // contexts per device for concurrent host threads

// Bitset width of the kernel flavour that fits n vertices.
int bits_for(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }
// Vertex capacity of a flavour (the wide 256-bit flavour stops at 255).
int capacity_of(int bits) { return bits == 256 ? kMaxWideN : bits; }

struct Context {
    int device = 0;
    int sms = 0;
    int smem_per_sm = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    InstanceDesc* d_inst = nullptr;
    WideDesc* d_winst = nullptr;    // wide instances (n > 64), allocated on first use
    WideDesc* h_winst = nullptr;
    size_t winst_cap = 0;
    WideSlot* d_wslots = nullptr;   // wide ring, allocated on first use
    InstanceState* d_ist = nullptr;
    GroupState* d_grp = nullptr;
    InstanceDesc* h_inst = nullptr;
    InstanceState* h_ist = nullptr;
    GroupState* h_grp = nullptr;
    size_t inst_cap = 0, grp_cap = 0;
    TaskSlot* d_slots = nullptr;
    Ctl* d_ctl = nullptr;
    Counters* d_cnt = nullptr;
    Counters* h_cnt = nullptr;
    Ctl* h_ctl = nullptr;  // pinned
    uint64_t* d_spill = nullptr;
    size_t spill_bytes = 0;
    int32_t* h_cancel = nullptr;  // pinned, mapped
    int32_t* d_cancel = nullptr;
    int32_t* h_xfloor = nullptr;  // live SharedBound: host -> kernel (pinned, mapped)
    int32_t* d_xfloor = nullptr;
    int32_t* h_xbest = nullptr;   // stored improvements: kernel -> host (pinned, mapped)
    int32_t* d_xbest = nullptr;
    int clock_khz = 0;            // SM clock (cycle counters -> seconds)
    RxState* d_rx = nullptr;      // exact restart engine: the segment in flight
    RxState* h_rx = nullptr;      // (pinned)
    std::mutex mu;

    explicit Context(int dev) : device(dev) {
        ck(cudaSetDevice(dev), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
        if (prop.major < 10)
            throw Error("mcsg kernels are built for sm_100a; device " + std::to_string(dev) +
                        " is sm_" + std::to_string(prop.major * 10 + prop.minor));
        sms = prop.multiProcessorCount;
        smem_per_sm = int(prop.sharedMemPerMultiprocessor);
        ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreate(&ev0), "event");
        ck(cudaEventCreate(&ev1), "event");
        ck(cudaMalloc(&d_slots, sizeof(TaskSlot) * kRingCap), "ring");
        ck(cudaMalloc(&d_ctl, sizeof(Ctl)), "ctl");
        ck(cudaMalloc(&d_cnt, sizeof(Counters)), "counters");
        ck(cudaMallocHost(&h_cnt, sizeof(Counters)), "counters host");
        ck(cudaMallocHost(&h_ctl, sizeof(Ctl)), "ctl host");
        ck(cudaHostAlloc(&h_cancel, sizeof(int32_t), cudaHostAllocMapped), "cancel flag");
        ck(cudaHostGetDevicePointer(&d_cancel, h_cancel, 0), "cancel flag map");
        *h_cancel = 0;
        ck(cudaHostAlloc(&h_xfloor, sizeof(int32_t), cudaHostAllocMapped), "shared bound");
        ck(cudaHostGetDevicePointer(&d_xfloor, h_xfloor, 0), "shared bound map");
        ck(cudaHostAlloc(&h_xbest, sizeof(int32_t), cudaHostAllocMapped), "shared bound");
        ck(cudaHostGetDevicePointer(&d_xbest, h_xbest, 0), "shared bound map");
        *h_xfloor = *h_xbest = 0;
        ck(cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, dev), "clock rate");
    }

    void reserve(size_t n_inst, size_t n_grp, size_t spill) {
        if (n_inst > inst_cap) {
            size_t cap = std::max<size_t>(n_inst, inst_cap * 2);
            cudaFree(d_inst);
            cudaFree(d_ist);
            cudaFreeHost(h_inst);
            cudaFreeHost(h_ist);
            ck(cudaMalloc(&d_inst, sizeof(InstanceDesc) * cap), "instances");
            ck(cudaMalloc(&d_ist, sizeof(InstanceState) * cap), "instance state");
            ck(cudaMallocHost(&h_inst, sizeof(InstanceDesc) * cap), "instances host");
            ck(cudaMallocHost(&h_ist, sizeof(InstanceState) * cap), "instance state host");
            inst_cap = cap;
        }
        if (n_grp > grp_cap) {
            size_t cap = std::max<size_t>(n_grp, grp_cap * 2);
            cudaFree(d_grp);
            cudaFreeHost(h_grp);
            ck(cudaMalloc(&d_grp, sizeof(GroupState) * cap), "groups");
            ck(cudaMallocHost(&h_grp, sizeof(GroupState) * cap), "groups host");
            grp_cap = cap;
        }
        if (spill > spill_bytes) {
            cudaFree(d_spill);
            d_spill = nullptr;
            ck(cudaMalloc(&d_spill, spill), "spill");
            spill_bytes = spill;
        }
    }

    void ensure_rx() {
        if (d_rx) return;
        ck(cudaMalloc(&d_rx, sizeof(RxState)), "restart segment");
        ck(cudaMallocHost(&h_rx, sizeof(RxState)), "restart segment host");
    }

    void reserve_wide(size_t n_inst) {
        if (!d_wslots) {
            ck(cudaMalloc(&d_wslots, sizeof(WideSlot) * kWideRingCap), "wide ring");
        }
        if (n_inst > winst_cap) {
            size_t cap = std::max<size_t>(n_inst, winst_cap * 2);
            cudaFree(d_winst);
            cudaFreeHost(h_winst);
            ck(cudaMalloc(&d_winst, sizeof(WideDesc) * cap), "wide instances");
            ck(cudaMallocHost(&h_winst, sizeof(WideDesc) * cap), "wide instances host");
            winst_cap = cap;
        }
    }
};

std::mutex g_ctx_mu;
std::map<std::pair<int, int>, std::unique_ptr<Context>> g_ctx;

// Device context `slot` of a CUDA device. Slot > 0 only appears when several
// shards of one multi-device solve are placed on the same physical device
// (each shard needs its own ring and instance state).
Context& context(int device, int slot = 0) {
    int dev = device;
    if (dev < 0) {
        ck(cudaGetDevice(&dev), "cudaGetDevice");
    }
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    auto it = g_ctx.find({dev, slot});
    if (it != g_ctx.end()) return *it->second;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw Error("no CUDA device available (mcsg has no CPU fallback)");
    if (dev >= count) throw Error("CUDA device " + std::to_string(dev) + " does not exist");
    auto ctx = std::make_unique<Context>(dev);
    Context& ref = *ctx;
    g_ctx[{dev, slot}] = std::move(ctx);
    return ref;
}

// One instance of a launch: a (possibly permuted) pair plus how to undo the
// permutation on its mapping.
struct Job {
    HostGraph g, h;            // as searched (permuted when ordered)
    std::vector<int> inv_g;    // searched id -> original id (empty = identity)
    std::vector<int> inv_h;
    int group = 0;
    int goal = 0;
    int floor_size = 0;
    uint64_t seed = 0;         // throughput mode: seeded search order (restarts:<seed>)
};

struct JobResult {
    int status = MCSG_OPTIMAL;
    int size = 0;
    std::vector<int32_t> pairs;  // original ids
    uint64_t nodes = 0;
    double solve_s = 0;
    bool completed = false;
    bool suspect = false;  // the dead-end policy stopped it
    uint64_t suspects = 0;  // parity mode: suspect nodes (deadend_suspects)
};

struct GroupResult {
    bool done = false;
    int winner = -1;
    bool reached = false;
    bool suspect = false;
    uint32_t restarts = 0;
};

struct LaunchOut {
    std::vector<JobResult> jobs;
    std::vector<GroupResult> groups;
    Counters counters{};
    double kernel_s = 0, h2d_s = 0;
    int warps = 0, ctas = 0, smem_per_cta = 0, smem_classes = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0, launches = 0;
    int clock_khz = 0;
    RxState rx{};  // exact restart engine: the segment's outcome
};

Job make_job(const HostGraph& g, const HostGraph& h, int order) {
    Job j;
    if (order == MCSG_ORDER_NONE) {
        j.g = g;
        j.h = h;
        return j;
    }
    const auto pg = make_ordering(g, order);
    const auto ph = make_ordering(h, order);
    j.g = g.permuted(pg);
    j.h = h.permuted(ph);
    j.inv_g.assign(g.n, 0);
    j.inv_h.assign(h.n, 0);
    for (int v = 0; v < g.n; ++v) j.inv_g[pg[v]] = v;
    for (int u = 0; u < h.n; ++u) j.inv_h[ph[u]] = u;
    return j;
}

// Throughput mode: relabel G so that its ids follow select_vertex's order
// (degree desc, id asc; label_classes.cpp:69-78) REVERSED: the first vertex
// of that order gets the highest id. The kernel then picks v with one FLO
// (highest set bit); the composed permutation is undone on the returned
// mapping.
//
// A nonzero seed is the GPU counterpart of the "restarts:<seed>" portfolio
// member (restarts.cpp:213-228 draws the next segment with mt19937_64): it
// diversifies the search order instead — equal-degree G vertices are ordered
// by a seeded permutation and H is relabelled by random_permutation(n_H, seed),
// so u candidates are tried in a seeded order. Optima are unaffected.
void relabel_for_throughput(Job& j, uint64_t seed = 0) {
    const int n = j.g.n;
    std::vector<int> order(n);
    for (int v = 0; v < n; ++v) order[v] = v;
    std::vector<int> deg(n);
    for (int v = 0; v < n; ++v) deg[v] = j.g.degree(v);
    std::vector<int> tie(n);
    for (int v = 0; v < n; ++v) tie[v] = v;
    if (seed) tie = random_permutation(n, seed * 0x9e3779b97f4a7c15ull);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return deg[a] != deg[b] ? deg[a] > deg[b] : tie[a] < tie[b]; });
    std::vector<int> fwd(n);
    for (int pos = 0; pos < n; ++pos) fwd[order[pos]] = n - 1 - pos;
    std::vector<int> inv(n);
    for (int v = 0; v < n; ++v) inv[fwd[v]] = j.inv_g.empty() ? v : j.inv_g[v];
    j.g = j.g.permuted(fwd);
    j.inv_g = std::move(inv);
    if (seed) {
        const int m = j.h.n;
        const std::vector<int> ph = random_permutation(m, seed);
        std::vector<int> ih(m);
        for (int u = 0; u < m; ++u) ih[ph[u]] = j.inv_h.empty() ? u : j.inv_h[u];
        j.h = j.h.permuted(ph);
        j.inv_h = std::move(ih);
    }
}

// SharedBound::bump (solve.hpp:73-77) on the caller's int32
void bump_shared(volatile int32_t* sb, int32_t size) {
    int32_t cur = __atomic_load_n(sb, __ATOMIC_ACQUIRE);
    while (size > cur && !__atomic_compare_exchange_n(sb, &cur, size, true, __ATOMIC_RELEASE, __ATOMIC_ACQUIRE)) {
    }
}

// Effective DeadEndPolicy kind of the options (0 = no policy).
int deadend_kind(const mcsg_options& o) {
    if (o.deadend_kind == 1 || o.deadend_kind == 2) return o.deadend_kind;
    return o.deadend_abs ? 1 : o.deadend_rel > 0 ? 2 : 0;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// What a launch does beyond "every instance is a root task".
struct LaunchExtras {
    std::vector<TaskSlot> seeded;    // subtrees published in the ring before the launch
    std::vector<WideSlot> wseeded;   // the same for a wide (n > 64) launch
    bool roots = true;               // hand out every instance as a root task
    std::vector<GroupState*> peers;  // group 0's incumbent on the other devices (P2P)
    bool peer_done_on_complete = false;
    bool relabeled = false;          // jobs already in the kernel's vertex order
    int seed_best = 0;               // host incumbent of instance 0 (frontier expansion)
    std::vector<uint8_t> seed_v, seed_u;
    std::vector<int> ladder_goal;            // probe ladder of the round (ascending goals)
    std::vector<GroupState*> ladder_grp;     // its groups: local or peer GroupState
    const RxState* rx = nullptr;             // exact restart engine: the segment to run (parity mode)
};

// A launch in flight on one context (ctx.mu held by the caller until finish()).
struct InFlight {
    Context* ctx = nullptr;
    std::vector<Job>* jobs = nullptr;
    mcsg_options o{};
    int n = 0, n_groups = 0, ctas = 0, warps = 0, smem_classes = 0;
    int bits = 32;          // kernel flavour (bitset width)
    bool directed = false;
    int spill_classes = 0;  // per warp, in HBM
    size_t spill_bytes = 0;
    size_t seeded = 0;
    std::chrono::steady_clock::time_point t_stage;
    double h2d_s = 0;
    bool rx = false;
};

// Kernel shape for a batch: specialisation, shared-memory class stack, grid.
void plan(Context& ctx, const std::vector<Job>& jobs, const mcsg_options& o, InFlight* f) {
    int maxn = 0, maxm = 0;
    f->directed = false;
    for (const Job& j : jobs) {
        maxn = std::max(maxn, std::max(j.g.n, j.h.n));
        maxm = std::max(maxm, std::min(j.g.n, j.h.n));
        f->directed |= j.g.directed;
    }
    f->bits = bits_for(maxn);
    const bool parity = o.mode == MCSG_MODE_PARITY;
    // Shared-memory class stack. A search level at depth d holds at most
    // min(n_G, n_H) - d classes, so m(m+1)/2 (+ slack for one child's worst
    // case) bounds the whole path: the 32-bit kernel never spills. The other
    // flavours take what the register-limited occupancy leaves and spill
    // whole levels beyond it to HBM. Level 0 (a root or a donated subtree)
    // always sits in shared memory.
    const int path_bound = maxm * (maxm + 1) / 2 + 2 * capacity_of(f->bits);
    const int cls_bytes = kernel_class_bytes(f->bits);
    const int min_smem = f->bits <= 64 ? 64 : std::max(64, maxm + 1);
    int smem_classes = o.smem_classes;
    int blocks = kernel_occupancy(f->bits, f->directed, min_smem);
    if (blocks <= 0) throw Error("search kernel cannot be resident on this device");
    if (smem_classes <= 0) {
        const int per_cta = ctx.smem_per_sm / blocks - 1024;
        const int per_warp = per_cta / kWarpsPerCta;
        const int fixed = kernel_smem_fixed(f->bits, f->directed);
        smem_classes = std::clamp((per_warp - fixed) / cls_bytes, min_smem, 2048);
        smem_classes = std::max(std::min(smem_classes, path_bound), min_smem);
        while (smem_classes > min_smem && kernel_occupancy(f->bits, f->directed, smem_classes) < blocks)
            smem_classes -= 16;
    }
    smem_classes = std::max(smem_classes, min_smem);
    if (f->bits == 32) smem_classes = std::max(smem_classes, path_bound);  // 32-bit kernel: no spill path
    blocks = kernel_occupancy(f->bits, f->directed, smem_classes);
    if (blocks <= 0) throw Error("requested shared-memory class stack does not fit");
    int ctas = blocks * ctx.sms;
    if (o.max_warps > 0) ctas = std::min(ctas, (o.max_warps + kWarpsPerCta - 1) / kWarpsPerCta);
    if (o.warp_share > 1) ctas = std::max(1, ctas / o.warp_share);  // concurrent engines on one GPU
    if (parity) ctas = std::min(ctas, (int(jobs.size()) + kWarpsPerCta - 1) / kWarpsPerCta);
    f->ctas = std::max(ctas, 1);
    f->warps = f->ctas * kWarpsPerCta;
    f->smem_classes = smem_classes;
    f->spill_classes = f->bits == 32 ? 0 : f->bits == 64 ? kSpillClasses : path_bound;
    f->spill_bytes = size_t(f->spill_classes) * size_t(cls_bytes) * size_t(f->warps);
}

// Packs, stages and launches; returns without waiting.
InFlight start(Context& ctx, std::vector<Job>& jobs, int n_groups, const mcsg_options& o,
               const LaunchExtras& ex) {
    ck(cudaSetDevice(ctx.device), "cudaSetDevice");
    InFlight f;
    f.ctx = &ctx;
    f.jobs = &jobs;
    f.o = o;
    f.n = int(jobs.size());
    f.n_groups = n_groups;
    const bool parity = o.mode == MCSG_MODE_PARITY;
    if (!parity && !ex.relabeled)
        for (Job& j : jobs) relabel_for_throughput(j, j.seed ? j.seed : o.seed);
    plan(ctx, jobs, o, &f);
    const int n = f.n;
    const bool wide = f.bits > 64;
    ctx.reserve(size_t(n), size_t(n_groups), f.spill_bytes);
    if (wide) ctx.reserve_wide(size_t(n));
    const uint32_t ring_cap = wide ? kWideRingCap : kRingCap;
    const size_t n_seeded = wide ? ex.wseeded.size() : ex.seeded.size();
    if (n_seeded + size_t(f.warps) > ring_cap) throw Error("too many seeded subtrees for the ring");
    if (wide ? !ex.seeded.empty() : !ex.wseeded.empty()) throw Error("seeded subtrees of the wrong width");

    f.t_stage = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) {
        if (wide)
            pack_wide(jobs[i].g, jobs[i].h, jobs[i].goal, o.disable_pruning == 0, jobs[i].floor_size,
                      jobs[i].group, &ctx.h_winst[i]);
        else
            pack_instance(jobs[i].g, jobs[i].h, jobs[i].goal, o.disable_pruning == 0, jobs[i].floor_size,
                          jobs[i].group, &ctx.h_inst[i]);
        std::memset(&ctx.h_ist[i], 0, sizeof(InstanceState));
        ctx.h_ist[i].open_tasks = ex.roots ? 1 : 0;
    }
    for (int gi = 0; gi < n_groups; ++gi) {
        ctx.h_grp[gi] = GroupState{};
        ctx.h_grp[gi].winner = -1;
    }
    if (n > 0 && ex.seed_best > 0) {  // the host's incumbent travels with the shard
        InstanceState& s0 = ctx.h_ist[0];
        s0.map_size = unsigned(ex.seed_best);
        for (int k = 0; k < ex.seed_best; ++k) s0.map_v[k] = ex.seed_v[k], s0.map_u[k] = ex.seed_u[k];
        ctx.h_grp[0].best = unsigned(ex.seed_best);
    }
    for (const TaskSlot& t : ex.seeded) ctx.h_ist[t.hdr.inst].open_tasks += 1;
    for (const WideSlot& t : ex.wseeded) ctx.h_ist[t.hdr.inst].open_tasks += 1;
    if (wide)
        ck(cudaMemcpyAsync(ctx.d_winst, ctx.h_winst, sizeof(WideDesc) * n, cudaMemcpyHostToDevice, ctx.stream), "h2d");
    else
        ck(cudaMemcpyAsync(ctx.d_inst, ctx.h_inst, sizeof(InstanceDesc) * n, cudaMemcpyHostToDevice, ctx.stream), "h2d");
    ck(cudaMemcpyAsync(ctx.d_ist, ctx.h_ist, sizeof(InstanceState) * n, cudaMemcpyHostToDevice, ctx.stream), "h2d");
    ck(cudaMemcpyAsync(ctx.d_grp, ctx.h_grp, sizeof(GroupState) * n_groups, cudaMemcpyHostToDevice, ctx.stream), "h2d");
    *ctx.h_ctl = Ctl{};
    ctx.h_ctl->pending.v = (ex.roots ? n : 0) + int(n_seeded);
    ctx.h_ctl->tail.v = n_seeded;
    ctx.h_ctl->live.v = n;
    ck(cudaMemcpyAsync(ctx.d_ctl, ctx.h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, ctx.stream), "h2d");
    if (wide)
        ck(ring_reset_wide(ctx.d_wslots, kWideRingCap, ctx.d_cnt, ctx.stream), "ring reset");
    else
        ck(ring_reset(ctx.d_slots, kRingCap, ctx.d_cnt, ctx.stream), "ring reset");
    if (!ex.seeded.empty()) {
        // published slots: sequence word = ticket + 1 (the consumer of ticket i reads it)
        std::vector<TaskSlot> staged(ex.seeded);
        for (size_t i = 0; i < staged.size(); ++i) staged[i].seq = i + 1;
        ck(cudaMemcpyAsync(ctx.d_slots, staged.data(), sizeof(TaskSlot) * staged.size(),
                           cudaMemcpyHostToDevice, ctx.stream),
           "h2d seeded tasks");
        ck(cudaStreamSynchronize(ctx.stream), "h2d seeded tasks");  // `staged` is pageable
    }
    if (!ex.wseeded.empty()) {
        std::vector<WideSlot> staged(ex.wseeded);
        for (size_t i = 0; i < staged.size(); ++i) staged[i].seq = i + 1;
        ck(cudaMemcpyAsync(ctx.d_wslots, staged.data(), sizeof(WideSlot) * staged.size(),
                           cudaMemcpyHostToDevice, ctx.stream),
           "h2d seeded tasks");
        ck(cudaStreamSynchronize(ctx.stream), "h2d seeded tasks");
    }
    f.seeded = n_seeded;
    *ctx.h_cancel = 0;
    *ctx.h_xbest = 0;
    *ctx.h_xfloor = o.shared_bound ? std::max(0, int(*o.shared_bound)) : 0;

    KernelParams p{};
    p.inst = ctx.d_inst;
    p.winst = ctx.d_winst;
    p.ist = ctx.d_ist;
    p.grp = ctx.d_grp;
    p.slots = ctx.d_slots;
    p.wslots = ctx.d_wslots;
    p.ctl = ctx.d_ctl;
    // Debug hooks (tests only): a smaller ring and a shorter producer
    // watchdog exercise the stall-abort path.
    uint32_t cap = ring_cap;
    if (const char* e = std::getenv("MCSG_DEBUG_RING_CAP")) {
        const uint32_t c = uint32_t(std::strtoul(e, nullptr, 10));
        if (c >= 1 && c <= ring_cap && (c & (c - 1)) == 0) cap = c;
    }
    p.cap_mask = cap - 1;
    p.ring_watchdog_ns = 2000000000ull;
    // compacted subtrees (64-bit kernel): slack 3 (C4 5.3 s at 2, 5.4 at 4;
    // C3 0.55 s at 2, 0.53 at 4; every nest costs ≈ 600 warp-instructions)
    // (round 2, after the nest pause: C4 4.33 / 4.24 / 4.31 s at slack 2 / 3 / 4;
    // the directed C3 launch 0.331 / 0.342 / 0.365 s)
    p.compact = f.directed ? 2 : 3;
    p.compact_room_cap = 0;
    if (const char* e = std::getenv("MCSG_DEBUG_COMPACT_ROOM")) p.compact_room_cap = int(std::strtol(e, nullptr, 10));
    if (const char* e = std::getenv("MCSG_DEBUG_COMPACT_SLACK")) p.compact = std::max(1, int(std::strtol(e, nullptr, 10)));
    if (const char* e = std::getenv("MCSG_DEBUG_NO_COMPACT")) p.compact = (e[0] == '0') ? p.compact : 0;
    if (const char* e = std::getenv("MCSG_DEBUG_RING_WATCHDOG_NS")) p.ring_watchdog_ns = std::strtoull(e, nullptr, 10);
    p.n_inst = n;
    p.n_roots = ex.roots ? n : 0;
    p.n_peers = int(ex.peers.size());
    if (p.n_peers > kMaxPeers) throw Error("too many peer devices");
    for (int q = 0; q < p.n_peers; ++q) p.peer_grp[q] = ex.peers[q];
    p.peer_done_on_complete = ex.peer_done_on_complete ? 1 : 0;
    if (ex.ladder_goal.size() > size_t(kMaxLadder)) throw Error("too many probe targets in one round");
    p.ladder_n = int(ex.ladder_goal.size());
    for (int k = 0; k < p.ladder_n; ++k) {
        p.ladder_goal[k] = ex.ladder_goal[k];
        p.ladder_grp[k] = ex.ladder_grp[k];
    }
    p.cancel = o.cancel ? ctx.d_cancel : nullptr;
    p.ext_floor = o.shared_bound ? ctx.d_xfloor : nullptr;
    p.ext_best = o.shared_bound ? ctx.d_xbest : nullptr;
    p.budget_ns = o.budget_s >= 1e8 ? 0ull : (unsigned long long)(o.budget_s * 1e9);
    p.spill = ctx.d_spill;
    p.spill_classes = f.spill_classes;
    p.smem_classes = f.smem_classes;
    p.donate = parity ? 0 : 1;
    // (<= 512: the kernel's packed split counters rely on it)
    // Throughput mode: a launch of a few small pairs is latency bound (its
    // tree fans out from one root: polls every 256 nodes, C1), a large or
    // many-pair launch throughput bound (every 512 nodes with the final
    // kernels: C4 -0.5%, C2 / C5 +0.3%, C3 unchanged against 384, which
    // had beaten 256 by 1-2% on C3-C5; C1 +12% at 384). tools/poll_sweep.sh,
    // tools/gpu_call_poll9.sh, tools/gpu_call_env64.sh.
    const bool latency_bound = n <= 8 && f.bits == 32;
    p.poll_interval = parity ? 512 : latency_bound ? 256 : 512;
    if (const char* e = std::getenv("MCSG_DEBUG_POLL_INTERVAL")) {  // tests / experiments only
        const int v = int(std::strtol(e, nullptr, 10));
        if (v >= 1 && v <= 512) p.poll_interval = v;
    }
    p.counters = ctx.d_cnt;
    if (!parity) p.restart_mult = o.restart_multiplier;
    // Dead-end monitor: per node in parity mode (stop when a jump follows,
    // else count suspect nodes); at polls in throughput mode, and only when a
    // jump follows (it then stops the launch).
    if (const int dk = deadend_kind(o); dk && (parity || o.deadend_jump != 0)) {
        p.deadend_kind = dk;
        p.deadend_stop = o.deadend_jump != 0 ? 1 : 0;
        p.deadend_abs = o.deadend_abs;
        p.deadend_rel = o.deadend_rel;
    }

    if (ex.rx) {
        if (!parity || n != 1) throw Error("the exact restart engine runs one instance in parity mode");
        ctx.ensure_rx();
        *ctx.h_rx = *ex.rx;
        ctx.h_rx->fired = ctx.h_rx->log_len = 0;
        ck(cudaMemcpyAsync(ctx.d_rx, ctx.h_rx, sizeof(RxState), cudaMemcpyHostToDevice, ctx.stream), "h2d");
        p.rx = ctx.d_rx;
        f.rx = true;
    }

    ck(cudaEventRecord(ctx.ev0, ctx.stream), "event");
    ck(kernel_launch(f.bits, f.directed, parity, p, f.ctas, ctx.stream), "search kernel launch");
    ck(cudaEventRecord(ctx.ev1, ctx.stream), "event");
    if (f.rx) ck(cudaMemcpyAsync(ctx.h_rx, ctx.d_rx, sizeof(RxState), cudaMemcpyDeviceToHost, ctx.stream), "d2h");
    ck(cudaMemcpyAsync(ctx.h_ist, ctx.d_ist, sizeof(InstanceState) * n, cudaMemcpyDeviceToHost, ctx.stream), "d2h");
    ck(cudaMemcpyAsync(ctx.h_grp, ctx.d_grp, sizeof(GroupState) * n_groups, cudaMemcpyDeviceToHost, ctx.stream), "d2h");
    ck(cudaMemcpyAsync(ctx.h_cnt, ctx.d_cnt, sizeof(Counters), cudaMemcpyDeviceToHost, ctx.stream), "d2h");
    ck(cudaMemcpyAsync(ctx.h_ctl, ctx.d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream), "d2h");
    f.h2d_s = secs_since(f.t_stage);
    return f;
}

// Waits for a launch and unpacks its results.
LaunchOut finish(InFlight& f) {
    Context& ctx = *f.ctx;
    ck(cudaSetDevice(ctx.device), "cudaSetDevice");
    LaunchOut out;
    const int n = f.n, n_groups = f.n_groups;
    out.jobs.resize(n);
    out.groups.resize(n_groups);
    if (f.o.cancel || f.o.shared_bound) {
        // mirror the caller's cancel flag and SharedBound into host-mapped
        // memory the kernel polls, and the kernel's stored improvements back
        volatile int32_t* xf = ctx.h_xfloor;
        volatile int32_t* xb = ctx.h_xbest;
        while (cudaStreamQuery(ctx.stream) == cudaErrorNotReady) {
            if (f.o.cancel && *f.o.cancel) *reinterpret_cast<volatile int32_t*>(ctx.h_cancel) = 1;
            if (f.o.shared_bound) {
                const int32_t ext = *f.o.shared_bound;
                if (ext > *xf) *xf = ext;
                bump_shared(f.o.shared_bound, *xb);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    ck(cudaStreamSynchronize(ctx.stream), "search kernel");
    if (f.o.shared_bound) bump_shared(f.o.shared_bound, *reinterpret_cast<volatile int32_t*>(ctx.h_xbest));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx.ev0, ctx.ev1);
    out.kernel_s = ms * 1e-3;
    out.h2d_s = f.h2d_s;
    out.counters = *ctx.h_cnt;
    out.warps = f.warps;
    out.ctas = f.ctas;
    out.clock_khz = ctx.clock_khz;
    out.smem_per_cta = kernel_smem_per_warp(f.bits, f.directed, f.smem_classes) * kWarpsPerCta;
    out.smem_classes = f.smem_classes;
    out.h2d_bytes = ((f.bits > 64 ? sizeof(WideDesc) : sizeof(InstanceDesc)) + sizeof(InstanceState)) * uint64_t(n) +
                    sizeof(GroupState) * uint64_t(n_groups) + sizeof(Ctl) +
                    (f.bits > 64 ? sizeof(WideSlot) : sizeof(TaskSlot)) * f.seeded;
    out.d2h_bytes = sizeof(InstanceState) * uint64_t(n) + sizeof(GroupState) * uint64_t(n_groups) +
                    sizeof(Counters) + sizeof(Ctl);
    out.launches = 2;  // ring reset + search kernel
    if (f.rx) {
        out.rx = *ctx.h_rx;
        out.h2d_bytes += sizeof(RxState);
        out.d2h_bytes += sizeof(RxState);
    }
    if (out.counters.overflow) throw Error("class stack overflow (internal error)");
    if (out.counters.bad_task)
        throw Error("malformed subtree in the task ring (internal error): ticket " +
                    std::to_string(out.counters.stall_pos) + " inst " + std::to_string(out.counters.stall_head) +
                    " depth<<8|nc " + std::to_string(out.counters.stall_tail) + " seq " +
                    std::to_string(out.counters.stall_seq));
    if (out.counters.ring_stall)
        throw Error("task ring stalled (internal error): ticket " + std::to_string(out.counters.stall_pos) +
                    " head " + std::to_string(out.counters.stall_head) + " tail " +
                    std::to_string(out.counters.stall_tail) + " slot seq " + std::to_string(out.counters.stall_seq));

    const int stop = ctx.h_ctl->stop.v;
    for (int gi = 0; gi < n_groups; ++gi) {
        out.groups[gi].done = ctx.h_grp[gi].done != 0;
        out.groups[gi].winner = ctx.h_grp[gi].winner;
        out.groups[gi].reached = ctx.h_grp[gi].reached != 0;
        out.groups[gi].suspect = ctx.h_grp[gi].suspect != 0;
        out.groups[gi].restarts = ctx.h_grp[gi].epoch;
    }
    for (int i = 0; i < n; ++i) {
        const InstanceState& s = ctx.h_ist[i];
        JobResult& r = out.jobs[i];
        const Job& j = (*f.jobs)[i];
        r.completed = s.open_tasks == 0;
        r.nodes = s.nodes;
        r.suspects = s.suspects;
        r.size = int(s.map_size);
        r.solve_s = s.t_done_ns > out.counters.t_start_ns ? (s.t_done_ns - out.counters.t_start_ns) * 1e-9 : 0.0;
        const bool group_done = out.groups[j.group].done;
        // a suspect verdict abandons the remaining tasks (they still finish, so
        // the open-task count says nothing about completion here)
        r.suspect = out.groups[j.group].suspect;
        if (stop != 0 && !(r.completed || group_done))
            r.status = stop == 2 ? MCSG_CANCELLED : MCSG_TIMEOUT;
        else if (r.suspect)
            r.status = MCSG_TIMEOUT;  // stopped by the dead-end policy; the caller resumes (jump)
        else
            r.status = MCSG_OPTIMAL;
        r.pairs.resize(2 * r.size);
        for (int k = 0; k < r.size; ++k) {
            int v = s.map_v[k], u = s.map_u[k];
            if (!j.inv_g.empty()) v = j.inv_g[v];
            if (!j.inv_h.empty()) u = j.inv_h[u];
            r.pairs[2 * k] = v;
            r.pairs[2 * k + 1] = u;
        }
    }
    return out;
}

// The single-device launch path shared by every entry point.
LaunchOut launch(std::vector<Job>& jobs, int n_groups, const mcsg_options& o, const LaunchExtras& ex = LaunchExtras{}) {
    if (jobs.empty()) {
        LaunchOut out;
        out.groups.resize(n_groups);
        return out;
    }
    // Calls from several host threads on one device (portfolio members racing
    // as separate engines) each take a free context slot — own stream, ring
    // and state — so their launches run concurrently (each sized by
    // warp_share); a thread only waits when every slot is busy.
    int dev = o.device;
    if (dev < 0) ck(cudaGetDevice(&dev), "cudaGetDevice");
    Context* ctx = nullptr;
    for (int slot = 0; slot < kMaxSlots && !ctx; ++slot) {
        Context& c = context(dev, slot);
        if (c.mu.try_lock()) ctx = &c;
    }
    if (!ctx) {
        ctx = &context(dev, 0);
        ctx->mu.lock();
    }
    std::lock_guard<std::mutex> lock(ctx->mu, std::adopt_lock);
    InFlight f = start(*ctx, jobs, n_groups, o, ex);
    return finish(f);
}

// ------------------------------------------------------------ multi-device --
// One launch per device; `members[i]` are the instances placed on device i
// (all in group 0). Contexts are locked in a fixed order, peer access is
// enabled between distinct physical devices, and every device gets the other
// devices' GroupState (group 0) as incumbent peers.
struct DevicePlan {
    int device = 0;
    std::vector<Job> jobs;
    std::vector<TaskSlot> seeded;
    std::vector<WideSlot> wseeded;
    bool roots = true;
    int n_groups = 1;
};

// Probe ladder of a parallel binary-search round: entry k (ascending goal)
// is group `group[k]` of plan `plan[k]`.
struct Ladder {
    std::vector<int> plan, group, goal;
};

std::vector<LaunchOut> launch_multi(std::vector<DevicePlan>& plans, const mcsg_options& o,
                                    bool peer_done_on_complete, int seed_best,
                                    const std::vector<uint8_t>& seed_v, const std::vector<uint8_t>& seed_u,
                                    const Ladder* ladder = nullptr) {
    const int D = int(plans.size());
    std::vector<Context*> ctxs(D);
    std::map<int, int> used;
    for (int i = 0; i < D; ++i) ctxs[i] = &context(plans[i].device, used[plans[i].device]++);
    std::vector<Context*> order(ctxs);
    std::sort(order.begin(), order.end());
    std::vector<std::unique_lock<std::mutex>> locks;
    for (Context* c : order) locks.emplace_back(c->mu);
    // peer access between distinct physical devices
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            const int a = ctxs[i]->device, b = ctxs[j]->device;
            if (a == b) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can)
                throw Error("devices " + std::to_string(a) + " and " + std::to_string(b) +
                            " cannot access each other (no P2P)");
            ck(cudaSetDevice(a), "cudaSetDevice");
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    // allocate every device's state first so that peer pointers exist
    for (int i = 0; i < D; ++i) {
        InFlight shape;
        mcsg_options oo = o;
        oo.mode = MCSG_MODE_THROUGHPUT;
        plan(*ctxs[i], plans[i].jobs, oo, &shape);
        ck(cudaSetDevice(ctxs[i]->device), "cudaSetDevice");
        ctxs[i]->reserve(plans[i].jobs.size(), size_t(plans[i].n_groups), shape.spill_bytes);
    }
    std::vector<InFlight> fl(D);
    for (int i = 0; i < D; ++i) {
        LaunchExtras ex;
        ex.seeded = plans[i].seeded;
        ex.wseeded = plans[i].wseeded;
        ex.roots = plans[i].roots;
        ex.relabeled = true;
        ex.peer_done_on_complete = peer_done_on_complete;
        if (ladder) {  // probes of different goals share no incumbent: only the ladder
            for (size_t k = 0; k < ladder->goal.size(); ++k) {
                ex.ladder_goal.push_back(ladder->goal[k]);
                ex.ladder_grp.push_back(ctxs[ladder->plan[k]]->d_grp + ladder->group[k]);
            }
        } else {
            for (int j = 0; j < D; ++j)
                if (j != i) ex.peers.push_back(ctxs[j]->d_grp);
        }
        ex.seed_best = seed_best;
        ex.seed_v = seed_v;
        ex.seed_u = seed_u;
        mcsg_options oo = o;
        oo.mode = MCSG_MODE_THROUGHPUT;
        oo.device = ctxs[i]->device;
        fl[i] = start(*ctxs[i], plans[i].jobs, plans[i].n_groups, oo, ex);
    }
    std::vector<LaunchOut> out(D);
    for (int i = 0; i < D; ++i) out[i] = finish(fl[i]);
    return out;
}

// One instance sharded over devices (SURVEY §8(e) "sharded" mode).
JobResult solve_sharded(const HostGraph& G, const HostGraph& H, const mcsg_options& o, LaunchOut* agg,
                        uint64_t* host_nodes) {
    const int D = o.n_devices;
    Job job = make_job(G, H, o.order);
    job.goal = o.goal;
    job.floor_size = o.floor_size;
    job.group = 0;
    relabel_for_throughput(job, o.seed);
    const int per_dev = o.frontier > 0 ? o.frontier : 256;
    Frontier fr;
    if (std::max(job.g.n, job.h.n) > kMaxN) {
        auto desc = std::make_unique<WideDesc>();
        pack_wide(job.g, job.h, job.goal, o.disable_pruning == 0, job.floor_size, 0, desc.get());
        fr = expand_frontier(*desc, job.g.directed, per_dev * D, 0);
    } else {
        InstanceDesc desc;
        pack_instance(job.g, job.h, job.goal, o.disable_pruning == 0, job.floor_size, 0, &desc);
        fr = expand_frontier(desc, job.g.directed, per_dev * D, 0);
    }
    *host_nodes = fr.nodes;
    auto host_result = [&](bool optimal_by_host) {
        JobResult r;
        r.status = MCSG_OPTIMAL;
        r.size = fr.best_size;
        r.completed = optimal_by_host;
        for (int k = 0; k < fr.best_size; ++k) {
            r.pairs.push_back(job.inv_g.empty() ? fr.best_v[k] : job.inv_g[fr.best_v[k]]);
            r.pairs.push_back(job.inv_h.empty() ? fr.best_u[k] : job.inv_h[fr.best_u[k]]);
        }
        r.nodes = fr.nodes;
        return r;
    };
    if (fr.max_reached || (fr.tasks.empty() && fr.wtasks.empty())) return host_result(true);  // the host already finished
    std::vector<DevicePlan> plans(D);
    for (int i = 0; i < D; ++i) {
        plans[i].device = o.devices[i];
        plans[i].jobs.push_back(job);
        plans[i].roots = false;
    }
    for (size_t k = 0; k < fr.tasks.size(); ++k) plans[k % D].seeded.push_back(fr.tasks[k]);
    for (size_t k = 0; k < fr.wtasks.size(); ++k) plans[k % D].wseeded.push_back(fr.wtasks[k]);
    std::vector<LaunchOut> outs = launch_multi(plans, o, false, fr.best_size, fr.best_v, fr.best_u);
    JobResult best = host_result(false);
    bool all_complete = true, any_done_max = false;
    int status = MCSG_OPTIMAL;
    uint64_t nodes = fr.nodes;
    for (const LaunchOut& lo : outs) {
        const JobResult& r = lo.jobs[0];
        nodes += r.nodes;
        all_complete &= r.completed;
        // stopped early because the max (or a probe goal) was reached; a
        // dead-end suspect verdict also raises done but proves nothing
        any_done_max |= lo.groups[0].done && !lo.groups[0].suspect && !r.completed;
        if (r.size > best.size) best = r;
        if (r.status != MCSG_OPTIMAL) status = r.status;
        best.solve_s = std::max(best.solve_s, r.solve_s);
    }
    best.nodes = nodes;
    best.status = (all_complete || any_done_max) ? MCSG_OPTIMAL : status;
    // aggregate counters for the stats record
    *agg = outs[0];
    agg->kernel_s = 0;
    for (const LaunchOut& lo : outs) agg->kernel_s = std::max(agg->kernel_s, lo.kernel_s);
    for (size_t i = 1; i < outs.size(); ++i) {
        agg->counters.nodes += outs[i].counters.nodes;
        agg->counters.splits += outs[i].counters.splits;
        agg->counters.donations += outs[i].counters.donations;
        agg->counters.tasks += outs[i].counters.tasks;
        agg->counters.busy_cycles += outs[i].counters.busy_cycles;
        agg->counters.idle_cycles += outs[i].counters.idle_cycles;
        agg->counters.peer_pushes += outs[i].counters.peer_pushes;
        agg->warps += outs[i].warps;
        agg->ctas += outs[i].ctas;
        agg->h2d_bytes += outs[i].h2d_bytes;
        agg->d2h_bytes += outs[i].d2h_bytes;
        agg->launches += outs[i].launches;
    }
    return best;
}

void fill_stats(mcsg_stats* st, const LaunchOut& lo, double wall, uint64_t probes) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->nodes = lo.counters.nodes;
    st->sum_classes = lo.counters.sum_classes;
    st->splits = lo.counters.splits;
    st->split_classes = lo.counters.split_classes;
    st->donations = lo.counters.donations;
    st->tasks = lo.counters.tasks;
    st->spills = lo.counters.spills;
    st->probes = probes;
    st->wall_s = wall;
    st->kernel_s = lo.kernel_s;
    st->h2d_s = lo.h2d_s;
    st->warps = lo.warps;
    st->ctas = lo.ctas;
    st->smem_per_cta = lo.smem_per_cta;
    st->smem_classes = lo.smem_classes;
    st->h2d_bytes = lo.h2d_bytes;
    st->d2h_bytes = lo.d2h_bytes;
    st->launches = lo.launches;
    st->busy_cycles = lo.counters.busy_cycles;
    st->idle_cycles = lo.counters.idle_cycles;
    st->restarts = lo.groups.empty() ? 0 : lo.groups[0].restarts;
    st->frozen = lo.counters.frozen;
    const double hz = lo.clock_khz > 0 ? lo.clock_khz * 1e3 : 1.0;
    st->idle_s = double(lo.counters.idle_cycles) / hz;
    st->busy_s = double(lo.counters.busy_cycles) / hz;
    st->peer_pushes = lo.counters.peer_pushes;
    if (std::getenv("MCSG_DEBUG_NESTS"))
        std::fprintf(stderr, "nests smem %llu hbm %llu\n", lo.counters.nests_smem, lo.counters.nests_hbm);
}

void accumulate(mcsg_stats* st, const LaunchOut& lo) {
    if (!st) return;
    st->nodes += lo.counters.nodes;
    st->sum_classes += lo.counters.sum_classes;
    st->splits += lo.counters.splits;
    st->split_classes += lo.counters.split_classes;
    st->donations += lo.counters.donations;
    st->tasks += lo.counters.tasks;
    st->spills += lo.counters.spills;
    st->kernel_s += lo.kernel_s;
    st->h2d_s += lo.h2d_s;
    st->warps = lo.warps;
    st->ctas = lo.ctas;
    st->smem_per_cta = lo.smem_per_cta;
    st->smem_classes = lo.smem_classes;
    st->h2d_bytes += lo.h2d_bytes;
    st->d2h_bytes += lo.d2h_bytes;
    st->launches += lo.launches;
    st->busy_cycles += lo.counters.busy_cycles;
    st->idle_cycles += lo.counters.idle_cycles;
    st->restarts += lo.groups.empty() ? 0 : lo.groups[0].restarts;
    st->frozen += lo.counters.frozen;
    const double hz = lo.clock_khz > 0 ? lo.clock_khz * 1e3 : 1.0;
    st->idle_s += double(lo.counters.idle_cycles) / hz;
    st->busy_s += double(lo.counters.busy_cycles) / hz;
    st->peer_pushes += lo.counters.peer_pushes;
}

mcsg_options defaults(const mcsg_options* o) {
    mcsg_options d{};
    d.budget_s = 1e9;
    d.device = -1;
    if (o) d = *o;
    return d;
}

void check_pair(const HostGraph& g, const HostGraph& h) {
    if (g.directed != h.directed) throw Error("solve: graphs must share a kind");
    if (g.labeled != h.labeled) throw Error("cannot mix a labeled graph with an unlabeled one");
    if (g.n > kMaxWideN || h.n > kMaxWideN)
        throw Error("graphs above " + std::to_string(kMaxWideN) + " vertices are not supported");
}

void write_result(const HostGraph& g, const HostGraph& h, const JobResult& r, mcsg_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = r.status;
    out->size = r.size;
    out->nodes = r.nodes;
    out->solve_s = r.solve_s;
    out->flags = r.suspect ? MCSG_RESULT_SUSPECT : 0;
    out->deadend_suspects = r.suspects ? r.suspects : (r.suspect ? 1 : 0);
    if (r.size > 0 && verify(g, h, r.pairs.data(), r.size) != 1)
        throw Error("internal error: kernel returned an invalid mapping");
    for (int k = 0; k < 2 * r.size; ++k) out->pairs[k] = r.pairs[k];
}

int fail(const std::exception& e) {
    t_err = e.what();
    t_err_kind = dynamic_cast<const ParseErr*>(&e) ? MCSG_ERR_PARSE
                 : dynamic_cast<const CudaErr*>(&e) ? MCSG_ERR_CUDA
                                                    : MCSG_ERR_GRAPH;
    return MCSG_ERROR;
}

void timed_out(mcsg_result* out, int status = MCSG_TIMEOUT) {
    std::memset(out, 0, sizeof(*out));
    out->status = status;
}

// One probe of the goal-directed / bound-jump schedules (solve.cpp:57-75).
struct Probe {
    bool reached = false;
    int status = MCSG_OPTIMAL;
    JobResult best;
};

Probe probe_goal(const HostGraph& g, const HostGraph& h, int goal, const mcsg_options& o,
                 mcsg_stats* st, std::chrono::steady_clock::time_point deadline, bool unlimited) {
    mcsg_options po = o;
    if (!unlimited) {
        po.budget_s = std::chrono::duration<double>(deadline - std::chrono::steady_clock::now()).count();
        if (po.budget_s <= 0) {
            Probe pr;
            pr.status = MCSG_TIMEOUT;
            return pr;
        }
    }
    std::vector<Job> jobs(1);
    jobs[0].g = g;
    jobs[0].h = h;
    jobs[0].goal = goal;
    LaunchOut lo = launch(jobs, 1, po);
    accumulate(st, lo);
    Probe pr;
    pr.reached = lo.groups[0].reached;
    pr.status = lo.jobs[0].status;
    pr.best = lo.jobs[0];
    return pr;
}

// ------------------------------------------------------ exact restarts --
// RestartDriver (restarts.cpp:35-246) with the reference's semantics, for
// parity mode: the host owns the segment pool as position keys (PositionKey,
// heuristics.hpp:77: the iteration taken at each depth; the depth is the
// index) and draws the next segment with the reference's seeded
// std::mt19937_64 (restarts.cpp:213-228). Each segment is one launch of the
// parity kernel (RxState): replay to the segment's node, resume at
// from_iter, per-node restart check. When a restart fires the kernel reports
// the path below the segment's node; the host then freezes it exactly as the
// unwinding in node() does — the node where it fired first (whole, :92-95),
// then every node on the path, deepest first, with its remaining iterations
// (:176-186) — and records the completed prefixes as visited ranges (:182).
// A segment that ends without a restart records its whole span (:113,119,189).
using PosKey = std::vector<int32_t>;

PosKey key_successor(const PosKey& pos) {  // restarts.cpp:13-18
    if (pos.empty()) return {std::numeric_limits<int32_t>::max()};
    PosKey s = pos;
    s.back() += 1;
    return s;
}

PosKey key_extend(const PosKey& pos, int it) {  // restarts.cpp:20-24
    PosKey s = pos;
    s.push_back(it);
    return s;
}

struct RestartOut {
    JobResult best;
    uint64_t nodes = 0, restarts = 0;
    std::vector<std::pair<PosKey, PosKey>> ranges;
};

RestartOut restarts_exact(const HostGraph& G, const HostGraph& H, const mcsg_options& o, mcsg_stats* st) {
    Job job = make_job(G, H, o.order);  // with_ordering (search_core.hpp:72-81)
    job.floor_size = o.floor_size;
    const int ng = job.g.n, nh = job.h.n;
    std::vector<int> fwd_g(ng), fwd_h(nh);  // original id -> searched id
    for (int x = 0; x < ng; ++x) fwd_g[job.inv_g.empty() ? x : job.inv_g[x]] = x;
    for (int x = 0; x < nh; ++x) fwd_h[job.inv_h.empty() ? x : job.inv_h[x]] = x;
    const int maxp = std::min(ng, nh);
    const bool unlimited = o.budget_s >= 1e8;
    const auto deadline = std::chrono::steady_clock::now() +
                          std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                              std::chrono::duration<double>(unlimited ? 0.0 : o.budget_s));
    mcsg_options lo = o;
    lo.mode = MCSG_MODE_PARITY;
    lo.goal = 0;
    lo.deadend_abs = 0;
    lo.deadend_rel = 0;
    lo.deadend_kind = 0;
    lo.deadend_jump = 0;
    lo.restart_multiplier = 0;
    lo.n_devices = 0;

    struct Segment {
        PosKey pos;
        int from_iter;
    };
    std::mt19937_64 rng(o.seed);
    std::vector<Segment> pool{{PosKey{}, 0}};
    RestartOut out;
    out.best.status = MCSG_OPTIMAL;
    uint64_t at = 0;
    LaunchExtras ex;
    RxState rx{};
    ex.rx = &rx;
    if (st) std::memset(st, 0, sizeof(*st));
    while (!pool.empty()) {
        const size_t idx = pool.size() == 1 ? 0 : size_t(rng() % pool.size());
        Segment seg = std::move(pool[idx]);
        pool.erase(pool.begin() + std::ptrdiff_t(idx));
        if (!unlimited) {
            lo.budget_s = std::chrono::duration<double>(deadline - std::chrono::steady_clock::now()).count();
            if (lo.budget_s <= 0) {
                out.best.status = MCSG_TIMEOUT;
                break;
            }
        }
        if (seg.pos.size() > sizeof(rx.script)) throw Error("restart segment deeper than the graph");
        rx.mult = o.restart_multiplier;
        rx.nodes0 = out.nodes;
        rx.at0 = at;
        rx.script_len = int32_t(seg.pos.size());
        rx.from_iter = seg.from_iter;
        for (size_t i = 0; i < seg.pos.size(); ++i) rx.script[i] = uint8_t(seg.pos[i]);
        std::vector<Job> jobs{job};
        LaunchOut r = launch(jobs, 1, lo, ex);
        accumulate(st, r);
        const JobResult& jr = r.jobs[0];
        out.nodes = r.rx.nodes;
        at = r.rx.at;
        if (jr.size > out.best.size) {  // the incumbent travels with the next segments
            const int status = out.best.status;
            out.best = jr;
            out.best.status = status;
            ex.seed_best = jr.size;
            ex.seed_v.assign(size_t(jr.size), 0);
            ex.seed_u.assign(size_t(jr.size), 0);
            for (int k = 0; k < jr.size; ++k) {
                ex.seed_v[k] = uint8_t(fwd_g[jr.pairs[2 * k]]);
                ex.seed_u[k] = uint8_t(fwd_h[jr.pairs[2 * k + 1]]);
            }
        }
        if (jr.status != MCSG_OPTIMAL) {  // timeout / cancel: the segment is abandoned
            out.best.status = jr.status;
            break;
        }
        if (!o.disable_pruning && out.best.size >= maxp) break;  // max_reached (restarts.cpp:108-111)
        const PosKey lo_key = seg.from_iter == 0 ? seg.pos : key_extend(seg.pos, seg.from_iter);
        if (!r.rx.fired) {
            out.ranges.emplace_back(lo_key, key_successor(seg.pos));
            continue;
        }
        ++out.restarts;
        at = out.nodes;  // rearm (restarts.cpp:90)
        const int len = r.rx.log_len;
        if (len == 0) {  // fired at the segment's own entry: frozen whole again
            pool.push_back(std::move(seg));
            continue;
        }
        std::vector<PosKey> path(size_t(len) + 1);
        path[0] = seg.pos;
        for (int k = 0; k < len; ++k) path[k + 1] = key_extend(path[k], r.rx.log[k]);
        pool.push_back({path[len], 0});
        for (int k = len - 1; k >= 0; --k) {
            pool.push_back({path[k], int(r.rx.log[k]) + 1});
            out.ranges.emplace_back(k == 0 ? lo_key : path[k], key_extend(path[k], r.rx.log[k]));
        }
    }
    out.best.nodes = out.nodes;
    return out;
}

}  // namespace
}  // namespace mcsg

using namespace mcsg;

extern "C" {

const char* mcsg_last_error(void) { return t_err.c_str(); }
int32_t mcsg_last_error_kind(void) { return t_err_kind; }
int32_t mcsg_abi_version(void) { return MCSG_ABI_VERSION; }

int32_t mcsg_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

void mcsg_shutdown(void) {
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    g_ctx.clear();  // device memory is reclaimed with the process / context
}

int32_t mcsg_solve_batch(int32_t count, const mcsg_graph* gs, const mcsg_graph* hs,
                         const mcsg_options* opt, mcsg_result* outs, mcsg_stats* stats) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const mcsg_options o = defaults(opt);
        if (count < 0) throw Error("negative batch size");
        std::vector<HostGraph> G(count), H(count);
        for (int i = 0; i < count; ++i) {
            G[i] = HostGraph::from_abi(&gs[i]);
            H[i] = HostGraph::from_abi(&hs[i]);
            check_pair(G[i], H[i]);
        }
        if (o.budget_s <= 0) {  // solve.cpp:95
            for (int i = 0; i < count; ++i) timed_out(&outs[i]);
            if (stats) std::memset(stats, 0, sizeof(*stats));
            return MCSG_TIMEOUT;
        }
        std::vector<Job> jobs;
        jobs.reserve(count);
        for (int i = 0; i < count; ++i) {
            jobs.push_back(make_job(G[i], H[i], o.order));
            jobs.back().group = i;
            jobs.back().goal = o.goal;
            jobs.back().floor_size = o.floor_size;
        }
        LaunchOut lo = launch(jobs, count, o);
        int worst = MCSG_OPTIMAL;
        for (int i = 0; i < count; ++i) {
            write_result(G[i], H[i], lo.jobs[i], &outs[i]);
            worst = std::max(worst, outs[i].status == MCSG_OPTIMAL ? 0 : outs[i].status);
        }
        fill_stats(stats, lo, secs_since(t0), 0);
        return worst;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// mcs::solve on one device (a batch of one) or sharded over o.n_devices.
static int32_t solve_plain(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options& o, mcsg_result* out,
                           mcsg_stats* stats) {
    if (o.n_devices <= 1) return mcsg_solve_batch(1, g, h, &o, out, stats);
    try {
        const auto t0 = std::chrono::steady_clock::now();
        if (o.n_devices > 16) throw Error("at most 16 devices");
        if (o.mode == MCSG_MODE_PARITY) throw Error("parity mode runs on one device");
        const HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (o.budget_s <= 0) {
            timed_out(out);
            return MCSG_TIMEOUT;
        }
        LaunchOut agg;
        uint64_t host_nodes = 0;
        const JobResult r = solve_sharded(G, H, o, &agg, &host_nodes);
        write_result(G, H, r, out);
        fill_stats(stats, agg, secs_since(t0), 0);
        if (stats) stats->nodes += host_nodes;
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_solve(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                   mcsg_result* out, mcsg_stats* stats) {
    const mcsg_options o = defaults(opt);
    if (o.deadend_jump != 0 && deadend_kind(o)) {
        // forecast-then-mitigate (portfolio.cpp:136-155): monitored solve; on a
        // suspect verdict the bound jump resumes from the incumbent size
        const auto t0 = std::chrono::steady_clock::now();
        const int32_t rc = solve_plain(g, h, o, out, stats);
        if (rc == MCSG_ERROR || !(out->flags & MCSG_RESULT_SUSPECT)) return rc;
        mcsg_options rest = o;
        rest.deadend_jump = 0;
        if (o.budget_s < 1e8) {
            rest.budget_s = o.budget_s - secs_since(t0);
            if (rest.budget_s <= 0) return out->status;
        }
        mcsg_result first = *out;
        mcsg_stats st2{};
        const int32_t rc2 = mcsg_bound_jump(g, h, first.size, o.deadend_jump == MCSG_JUMP_DOUBLING ? 1 : 0,
                                            &rest, out, &st2);
        if (rc2 == MCSG_ERROR) return rc2;
        if (out->size < first.size) {  // keep the better witness
            out->size = first.size;
            std::memcpy(out->pairs, first.pairs, sizeof(first.pairs));
        }
        out->nodes += first.nodes;
        out->flags = MCSG_RESULT_SUSPECT;
        out->deadend_suspects = first.deadend_suspects;
        if (stats) {
            stats->nodes += st2.nodes;
            stats->probes = st2.probes;
            stats->kernel_s += st2.kernel_s;
            stats->launches += st2.launches;
            stats->wall_s = secs_since(t0);
        }
        return out->status;
    }
    return solve_plain(g, h, o, out, stats);
}

int32_t mcsg_solve_with_restarts(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                                 mcsg_result* out, mcsg_stats* stats, int32_t* ranges_out, int64_t ranges_cap,
                                 int64_t* ranges_len) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const mcsg_options o = defaults(opt);
        const HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (ranges_len) *ranges_len = 0;
        if (o.budget_s <= 0) {  // restarts.cpp:197-202
            timed_out(out);
            if (stats) std::memset(stats, 0, sizeof(*stats));
            return MCSG_TIMEOUT;
        }
        if (o.mode != MCSG_MODE_PARITY) {  // the throughput engine's restart epochs
            const int32_t rc = solve_plain(g, h, o, out, stats);
            if (stats && rc == MCSG_OPTIMAL) stats->visited_ranges = 1;  // the whole tree, exactly once
            return rc;
        }
        if (o.n_devices > 1) throw Error("parity mode runs on one device");
        RestartOut r = restarts_exact(G, H, o, stats);
        write_result(G, H, r.best, out);
        if (stats) {
            stats->nodes = r.nodes;
            stats->restarts = r.restarts;
            stats->visited_ranges = r.ranges.size();
            stats->wall_s = secs_since(t0);
        }
        // ranges: per run [len(lo), lo..., len(hi), hi...]
        int64_t w = 0;
        for (const auto& run : r.ranges)
            for (const PosKey* k : {&run.first, &run.second}) {
                if (ranges_out && w < ranges_cap) ranges_out[w] = int32_t(k->size());
                ++w;
                for (int32_t x : *k) {
                    if (ranges_out && w < ranges_cap) ranges_out[w] = x;
                    ++w;
                }
            }
        if (ranges_len) *ranges_len = w;
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_solve_parallel(const mcsg_graph* g, const mcsg_graph* h, const mcsg_options* opt,
                            mcsg_result* out, mcsg_stats* stats) {
    mcsg_options o = defaults(opt);
    o.mode = MCSG_MODE_THROUGHPUT;
    return mcsg_solve_batch(1, g, h, &o, out, stats);
}

int32_t mcsg_portfolio(const mcsg_graph* g, const mcsg_graph* h, int32_t count,
                       const int32_t* orders, const uint64_t* seeds, const mcsg_options* opt,
                       mcsg_result* out, int32_t* winner_out, mcsg_stats* stats) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const mcsg_options o = defaults(opt);
        if (count <= 0) throw Error("portfolio needs at least one engine spec");
        const HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (o.budget_s <= 0) {
            timed_out(out);
            return MCSG_TIMEOUT;
        }
        std::vector<Job> jobs;
        for (int i = 0; i < count; ++i) {
            jobs.push_back(make_job(G, H, orders ? orders[i] : MCSG_ORDER_NONE));
            jobs.back().seed = seeds ? seeds[i] : 0;
            jobs.back().group = 0;
            jobs.back().goal = o.goal;
            jobs.back().floor_size = o.floor_size;
        }
        mcsg_options lo_opt = o;
        lo_opt.mode = MCSG_MODE_THROUGHPUT;  // members share the incumbent size
        // dead-end handling belongs to a member's engine spec (run_engine,
        // portfolio.cpp:136-155), never to the race: a suspect verdict would
        // stop every member without proving anything
        lo_opt.deadend_abs = 0;
        lo_opt.deadend_rel = 0;
        lo_opt.deadend_jump = 0;
        lo_opt.deadend_kind = 0;
        std::vector<JobResult> members(count);
        bool done = false;
        int w = -1;
        LaunchOut lo;
        if (o.n_devices <= 1) {
            lo = launch(jobs, 1, lo_opt);
            members = lo.jobs;
            done = lo.groups[0].done && !lo.groups[0].suspect;
            w = lo.groups[0].winner;
        } else {
            // members spread over the devices; the first to finish stops all (P2P done flag)
            const int D = std::min<int>(o.n_devices, 16);
            std::vector<DevicePlan> plans(D);
            std::vector<std::vector<int>> index(D);
            for (int d = 0; d < D; ++d) plans[d].device = o.devices[d];
            for (int i = 0; i < count; ++i) {
                plans[i % D].jobs.push_back(jobs[i]);
                index[i % D].push_back(i);
            }
            for (int d = 0; d < D; ++d)
                for (Job& j : plans[d].jobs) relabel_for_throughput(j, j.seed ? j.seed : o.seed);
            std::vector<DevicePlan> used;
            std::vector<std::vector<int>> used_index;
            for (int d = 0; d < D; ++d)
                if (!plans[d].jobs.empty()) used.push_back(std::move(plans[d])), used_index.push_back(index[d]);
            std::vector<LaunchOut> outs = launch_multi(used, lo_opt, true, 0, {}, {});
            double first = 1e300;
            for (size_t d = 0; d < outs.size(); ++d) {
                for (size_t k = 0; k < used_index[d].size(); ++k) members[used_index[d][k]] = outs[d].jobs[k];
                if (outs[d].groups[0].done && !outs[d].groups[0].suspect) {
                    done = true;
                    const int lw = outs[d].groups[0].winner;
                    if (lw >= 0 && outs[d].jobs[lw].completed && outs[d].jobs[lw].solve_s < first) {
                        first = outs[d].jobs[lw].solve_s;
                        w = used_index[d][lw];
                    }
                }
            }
            lo = outs[0];
            for (size_t d = 1; d < outs.size(); ++d) {
                lo.counters.nodes += outs[d].counters.nodes;
                lo.counters.peer_pushes += outs[d].counters.peer_pushes;
                lo.kernel_s = std::max(lo.kernel_s, outs[d].kernel_s);
                lo.warps += outs[d].warps;
                lo.launches += outs[d].launches;
            }
        }
        // best mapping among members (sizes are shared, mappings are per member)
        int bi = 0;
        for (int i = 1; i < count; ++i)
            if (members[i].size > members[bi].size) bi = i;
        JobResult r = members[bi];
        r.nodes = 0;
        for (const auto& jr : members) r.nodes += jr.nodes;
        r.status = done ? MCSG_OPTIMAL : members[bi].status;
        if (w >= 0) r.solve_s = members[w].solve_s;
        write_result(G, H, r, out);
        if (winner_out) *winner_out = w;
        fill_stats(stats, lo, secs_since(t0), 0);
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// solve.cpp:131-168: goals n_G, n_G-1, ... over the smaller graph.
int32_t mcsg_solve_goal_directed(const mcsg_graph* g, const mcsg_graph* h,
                                 const mcsg_options* opt, mcsg_result* out, mcsg_stats* stats) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const mcsg_options o = defaults(opt);
        HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (o.budget_s <= 0) {
            timed_out(out);
            return MCSG_TIMEOUT;
        }
        const bool swapped = G.n > H.n;
        if (swapped) std::swap(G, H);
        Job base = make_job(G, H, o.order);
        const bool unlimited = o.budget_s >= 1e8;
        const auto deadline = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                                       std::chrono::duration<double>(unlimited ? 0.0 : o.budget_s));
        if (stats) std::memset(stats, 0, sizeof(*stats));
        JobResult best;
        int status = MCSG_OPTIMAL;
        uint64_t probes = 0, nodes = 0;
        for (int goal = base.g.n; goal >= 1; --goal) {
            Probe pr = probe_goal(base.g, base.h, goal, o, stats, deadline, unlimited);
            ++probes;
            nodes += pr.best.nodes;
            if (pr.best.size > best.size) best = pr.best;
            if (pr.status != MCSG_OPTIMAL) {
                status = pr.status;
                break;
            }
            if (pr.reached) break;
        }
        // map back through the ordering, then undo the swap
        JobResult r = best;
        r.status = status;
        r.nodes = nodes;
        for (int k = 0; k < r.size; ++k) {
            int v = r.pairs[2 * k], u = r.pairs[2 * k + 1];
            if (!base.inv_g.empty()) v = base.inv_g[v];
            if (!base.inv_h.empty()) u = base.inv_h[u];
            r.pairs[2 * k] = swapped ? u : v;
            r.pairs[2 * k + 1] = swapped ? v : u;
        }
        if (swapped) std::swap(G, H);
        write_result(G, H, r, out);
        out->probes = int32_t(probes);
        if (stats) {
            stats->probes = probes;
            stats->wall_s = secs_since(t0);
        }
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// heuristics.cpp:114-185: jump the target (+1 or x2) until a probe fails,
// then binary-search the bracket; recover a witness for a supplied size.
int32_t mcsg_bound_jump(const mcsg_graph* g, const mcsg_graph* h, int32_t current_best,
                        int32_t doubling, const mcsg_options* opt, mcsg_result* out,
                        mcsg_stats* stats) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const mcsg_options o = defaults(opt);
        const HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (o.budget_s <= 0) {
            timed_out(out);
            return MCSG_TIMEOUT;
        }
        Job base = make_job(G, H, o.order);
        const bool unlimited = o.budget_s >= 1e8;
        const auto deadline = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                                       std::chrono::duration<double>(unlimited ? 0.0 : o.budget_s));
        if (stats) std::memset(stats, 0, sizeof(*stats));
        long long lower = current_best, upper = std::min(G.n, H.n);
        JobResult wit;
        int status = MCSG_OPTIMAL;
        uint64_t probes = 0, nodes = 0;
        bool stopped = false;
        auto run = [&](long long goal) -> bool {
            Probe pr = probe_goal(base.g, base.h, int(goal), o, stats, deadline, unlimited);
            ++probes;
            nodes += pr.best.nodes;
            if (pr.best.size > wit.size) wit = pr.best;
            if (pr.status != MCSG_OPTIMAL) {
                status = pr.status;
                stopped = true;
            }
            return pr.reached;
        };
        auto settle = [&](long long target, bool reached) {
            const long long lo = lower, up = upper;
            if (reached) lower = target;
            else upper = target - 1;
            if (lower < lo || upper > up || lower > upper) throw Error("bound jump bracket violated");
        };
        while (lower < upper) {
            long long target = doubling ? std::max<long long>(1, lower * 2) : lower + 1;
            target = std::min(target, upper);
            const bool reached = run(target);
            if (stopped) break;
            settle(target, reached);
        }
        while (!stopped && lower < upper) {
            const long long mid = lower + (upper - lower + 1) / 2;
            const bool reached = run(mid);
            if (stopped) break;
            settle(mid, reached);
        }
        if (!stopped && wit.size < lower && lower > 0) run(lower);
        JobResult r = wit;
        r.status = status;
        r.nodes = nodes;
        for (int k = 0; k < r.size; ++k) {
            if (!base.inv_g.empty()) r.pairs[2 * k] = base.inv_g[r.pairs[2 * k]];
            if (!base.inv_h.empty()) r.pairs[2 * k + 1] = base.inv_h[r.pairs[2 * k + 1]];
        }
        write_result(G, H, r, out);
        out->probes = int32_t(probes);
        if (stats) {
            stats->probes = probes;
            stats->wall_s = secs_since(t0);
        }
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Parallel binary search over goal probes (the GPU form of
// bound_jump_search's bracket, heuristics.cpp:114-185): every round probes up
// to `width` targets of the open bracket (lower, upper] at once, dealt over
// the devices, each target a group of its device's launch. Inside a round a
// reached target marks every lower one reached and an exhausted one marks
// every higher one failed, across devices over NVLink P2P (probe ladder), so
// each probe stops as soon as its answer is implied.
int32_t mcsg_probe_parallel(const mcsg_graph* g, const mcsg_graph* h, int32_t current_best, int32_t width,
                            const mcsg_options* opt, mcsg_result* out, mcsg_stats* stats) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        mcsg_options o = defaults(opt);
        const HostGraph G = HostGraph::from_abi(g), H = HostGraph::from_abi(h);
        check_pair(G, H);
        if (stats) std::memset(stats, 0, sizeof(*stats));
        if (o.budget_s <= 0) {
            timed_out(out);
            return MCSG_TIMEOUT;
        }
        if (o.mode == MCSG_MODE_PARITY) throw Error("probe ladders run in throughput mode");
        if (o.n_devices > 16) throw Error("at most 16 devices");
        std::vector<int> devs;
        if (o.n_devices > 0)
            for (int i = 0; i < o.n_devices; ++i) devs.push_back(o.devices[i]);
        else
            devs.push_back(o.device);
        if (width <= 0) width = std::max<int>(8, int(devs.size()));
        width = std::min(width, kMaxLadder);
        Job base = make_job(G, H, o.order);
        relabel_for_throughput(base, o.seed);
        long long lower = std::max(0, current_best), upper = std::min(G.n, H.n);
        if (lower > upper) throw Error("current best exceeds the smaller graph");
        const bool unlimited = o.budget_s >= 1e8;
        JobResult wit;
        int status = MCSG_OPTIMAL;
        uint64_t probes = 0, nodes = 0;
        LaunchOut agg;
        bool first = true;
        double ktot = 0;
        // one round over the given ascending targets; false when stopped
        auto round = [&](const std::vector<int>& targets) -> bool {
            const int K = int(targets.size());
            const int D = std::min<int>(int(devs.size()), K);
            std::vector<DevicePlan> plans(D);
            Ladder lad;
            for (int d = 0; d < D; ++d) {
                plans[d].device = devs[d] < 0 ? 0 : devs[d];
                plans[d].n_groups = 0;
            }
            if (devs[0] < 0) ck(cudaGetDevice(&plans[0].device), "cudaGetDevice");
            for (int k = 0; k < K; ++k) {
                DevicePlan& pl = plans[k % D];
                Job j = base;
                j.goal = targets[k];
                j.group = pl.n_groups;
                lad.plan.push_back(k % D);
                lad.group.push_back(pl.n_groups);
                lad.goal.push_back(targets[k]);
                pl.jobs.push_back(std::move(j));
                pl.n_groups += 1;
            }
            mcsg_options oo = o;
            oo.goal = 0;
            oo.deadend_abs = 0;
            oo.deadend_rel = 0;
            oo.deadend_jump = 0;
            oo.deadend_kind = 0;
            oo.restart_multiplier = 0;
            if (!unlimited) {
                oo.budget_s = o.budget_s - secs_since(t0);
                if (oo.budget_s <= 0) {
                    status = MCSG_TIMEOUT;
                    return false;
                }
            }
            std::vector<LaunchOut> outs = launch_multi(plans, oo, false, 0, {}, {}, &lad);
            probes += uint64_t(K);
            long long lo2 = lower, up2 = upper;
            bool stopped = false;
            for (int k = 0; k < K; ++k) {
                const JobResult& r = outs[lad.plan[k]].jobs[lad.group[k]];
                const GroupResult& gr = outs[lad.plan[k]].groups[lad.group[k]];
                nodes += r.nodes;
                if (r.size > wit.size) wit = r;
                if (gr.reached) lo2 = std::max<long long>(lo2, targets[k]);
                else if (r.status == MCSG_OPTIMAL && gr.done) up2 = std::min<long long>(up2, targets[k] - 1);
                else if (r.status != MCSG_OPTIMAL) {
                    stopped = true;
                    status = r.status;
                }
            }
            for (LaunchOut& lo : outs) {
                if (first) {
                    agg = lo;
                    first = false;
                } else {
                    agg.counters.nodes += lo.counters.nodes;
                    agg.counters.donations += lo.counters.donations;
                    agg.counters.tasks += lo.counters.tasks;
                    agg.counters.busy_cycles += lo.counters.busy_cycles;
                    agg.counters.idle_cycles += lo.counters.idle_cycles;
                    agg.launches += lo.launches;
                    agg.h2d_bytes += lo.h2d_bytes;
                    agg.d2h_bytes += lo.d2h_bytes;
                }
            }
            double kmax = 0;
            for (LaunchOut& lo : outs) kmax = std::max(kmax, lo.kernel_s);
            ktot += kmax;  // rounds run one after another; devices of a round concurrently
            if (stopped) return false;
            lo2 = std::max<long long>(lo2, wit.size);  // a stored mapping proves its size
            if (lo2 < lower || up2 > upper || lo2 > up2) throw Error("bound jump bracket violated");
            lower = lo2;
            upper = up2;
            return true;
        };
        bool ok = true;
        // Targets of a round: the first half just above the bracket's floor
        // (the incumbent is usually close to the optimum: plus_one's jumps, in
        // parallel), the rest spaced geometrically up to its ceiling (doubling's
        // reach: high goals fail fast, so they cost little).
        while (ok && lower < upper) {
            const long long span = upper - lower;
            const int K = int(std::min<long long>(width, span));
            const int hcons = (K + 1) / 2, geo = K - hcons;
            std::vector<int> targets;
            for (int k = 1; k <= hcons; ++k) targets.push_back(int(lower + k));
            for (int i = 1; i <= geo; ++i) {
                const long long rest = span - hcons;
                const long long num = rest * ((1ll << i) - 1), den = (1ll << geo) - 1;
                const int t = int(lower + hcons + (num + den - 1) / den);
                if (t > targets.back()) targets.push_back(t);
            }
            ok = round(targets);
        }
        if (ok && wit.size < lower && lower > 0) round({int(lower)});  // a witness for a supplied size
        JobResult r = wit;  // (finish() already mapped it back to original ids)
        r.status = status;
        r.nodes = nodes;
        write_result(G, H, r, out);
        out->probes = int32_t(probes);
        if (stats && !first) {
            agg.kernel_s = ktot;
            fill_stats(stats, agg, secs_since(t0), probes);
            stats->nodes = nodes;
        }
        return out->status;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_verify(const mcsg_graph* g, const mcsg_graph* h, const int32_t* pairs, int32_t k) {
    try {
        return verify(HostGraph::from_abi(g), HostGraph::from_abi(h), pairs, k);
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

int32_t mcsg_random_graph(int32_t n, double density, uint64_t seed, uint32_t flags,
                          int32_t label_count, uint8_t* codes_out, int32_t* labels_out) {
    try {
        random_graph(n, density, seed, (flags & MCSG_DIRECTED) != 0, label_count, codes_out, labels_out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_random_permutation(int32_t n, uint64_t seed, int32_t* fwd_out) {
    const auto f = random_permutation(n, seed);
    for (int i = 0; i < n; ++i) fwd_out[i] = f[i];
    return 0;
}

int32_t mcsg_ordering(const mcsg_graph* g, int32_t strategy, int32_t* fwd_out) {
    try {
        const auto f = make_ordering(HostGraph::from_abi(g), strategy);
        for (size_t i = 0; i < f.size(); ++i) fwd_out[i] = f[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_load_graph_file(const char* path, int32_t format, int32_t* n_out, uint32_t* flags_out,
                             uint8_t* codes_out, int32_t* labels_out) {
    try {
        const HostGraph g = load_graph_file(path, format);
        *n_out = g.n;
        *flags_out = (g.directed ? MCSG_DIRECTED : 0u) | (g.labeled ? MCSG_LABELED : 0u);
        if (codes_out) std::memcpy(codes_out, g.codes.data(), g.codes.size());
        if (labels_out && g.labeled) std::memcpy(labels_out, g.labels.data(), sizeof(int32_t) * g.n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_save_graph_file(const mcsg_graph* g, const char* path, int32_t format) {
    try {
        save_graph_file(HostGraph::from_abi(g), path, format);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_pack_graph(const mcsg_graph* g, uint64_t* out_rows, uint64_t* in_rows) {
    try {
        const HostGraph x = HostGraph::from_abi(g);
        if (x.n > kMaxN) throw Error("graph above 64 vertices");
        InstanceDesc d;
        HostGraph empty = x;
        pack_instance(x, empty, 0, true, 0, 0, &d);
        for (int v = 0; v < x.n; ++v) {
            out_rows[v] = d.out_g[v];
            if (in_rows) in_rows[v] = d.in_g[v];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int32_t mcsg_pack_graph_words(const mcsg_graph* g, int32_t words, uint64_t* out_rows, uint64_t* in_rows) {
    try {
        const HostGraph x = HostGraph::from_abi(g);
        if (x.n > kMaxWideN) throw Error("graph above " + std::to_string(kMaxWideN) + " vertices");
        if (words < (x.n + 63) / 64 || words > kWideWords) throw Error("row width does not fit the graph");
        auto d = std::make_unique<WideDesc>();
        pack_wide(x, x, 0, true, 0, 0, d.get());
        for (int v = 0; v < x.n; ++v)
            for (int w = 0; w < words; ++w) {
                out_rows[size_t(v) * words + w] = d->out_g[v][w];
                if (in_rows) in_rows[size_t(v) * words + w] = d->in_g[v][w];
            }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
