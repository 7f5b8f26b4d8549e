// The persistent McSplit search kernel (sm_100a) and its launch glue.
//
// Each warp loops: take a task (an instance root from an atomic counter, or a
// donated subtree from the HBM ring), run its DFS, finish it. The DFS itself:
//
//   select  choose the label class (min max(|L|,|R|), label_classes.cpp:47-67)
//           and the vertex v (max degree, label_classes.cpp:69-78); offer
//           the first child's mapping when it improves
//           (search_core.hpp:145-155); count the level's |R*| children and
//           its continuation in bulk (each is a counted node,
//           search_core.hpp:130) and poll
//   next    for each u of the class's right side (search_core.hpp:183-200):
//           compute the child's bound from the register-resident level
//           (label_classes.cpp:41-45) and only when it survives the prune
//           test (search_core.hpp:166) materialise it with filter_classes
//           (label_classes.cpp:80-108) and descend
//   cont    then the "v unmatched" continuation at the same level
//           (search_core.hpp:201-212)
//   pop     back to the parent level
//
// Specialisations:
//   PAR = true   parity mode: one warp per instance, no donation, u in
//                ascending id; the host keeps the reference's vertex ids so
//                the DFS visits the reference's nodes in the reference's
//                order (tests compare node counts and mappings exactly).
//   PAR = false  throughput mode: every resident warp, subtree donation to
//                idle warps, group incumbent shared through HBM, u walked
//                from the top. The host relabels G in REVERSE (degree desc,
//                id asc) order so select_vertex is a single FLO.
//   RST = true   throughput mode with restarts (restart_mult > 0).
//   X = Search<u64>, throughput, no restarts: a level whose live vertex sets
//                fit 32 bits runs its subtree in place with the 32-bit
//                policy on renumbered vertices (CompactSearch, run_nested).
// The task body (select/next/cont/pop and the task's bookkeeping) is
// mcsg_task_body.inc, included once per policy.
#include "mcsg_search.cuh"

namespace mcsg {

// Fairness between the instances of one launch: an instance running on fewer
// than half its share of the warps (warps / live instances) keeps donating
// while fewer than kStarvedQueue subtrees are queued, even when no warp is
// waiting; warps that finish a task take queued subtrees in ticket order.
constexpr int kStarvedQueue = 256;
// Poll interval (nodes) while warps are waiting for work.
constexpr int kFastPoll = 16;


// RST: restarts compiled in (throughput mode with restart_mult > 0 only), so
// that the common launch carries none of their code.
template <class X, bool PAR, bool RST = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32, X::kMinBlocks)
    mcs_search_kernel(KernelParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using Sm = typename X::Sm;
    using W = typename X::Set;  // vertex bitset (one word, or WSet for wide graphs)
    using Cl = Cls<W>;
    using Slot = typename X::Slot;
    constexpr int NB = X::NB;
    constexpr int P = X::P;
    const int lane = threadIdx.x & 31;
    // warp index via a warp reduction: the result lives in a uniform register,
    // so the per-warp shared-memory addresses below stay in the uniform
    // datapath instead of being rematerialised from SR_TID in the hot loop
    const int wib = int(__reduce_min_sync(kFull, threadIdx.x >> 5));
    const int gw = blockIdx.x * kWarpsPerCta + wib;
    const int per_warp = warp_smem_bytes<X>(p.smem_classes);
    Sm& s = *reinterpret_cast<Sm*>(smem_raw + size_t(wib) * per_warp);
    X x(s, reinterpret_cast<Cl*>(smem_raw + size_t(wib) * per_warp + warp_smem_fixed<X>()),
        reinterpret_cast<Cl*>(p.spill) + size_t(gw) * p.spill_classes, p.smem_classes, lane, lanemask_lt());
    Slot* const ring = X::slots(p);
    Ctl* const ctl = p.ctl;
    const int interval = p.poll_interval;

    {
        const unsigned long long t_warp0 = globaltimer();
        if (lane == 0) {
            atomicMin(&p.counters->t_start_ns, t_warp0);
            s.deadline = p.budget_ns ? t_warp0 + p.budget_ns : 0ull;  // (read by lane 0 at polls)
        }
    }

    if (lane == 0)
        s.st_nodes = s.st_splits = s.st_split_cls = s.st_donations = s.st_tasks = s.st_spills = s.st_idle = s.st_busy = 0;
    if constexpr (X::kNest) {
        if (lane == 0) s.ca.nests_smem = s.ca.nests_hbm = 0;
    }
    if (lane == 0) s.t_mark = clock64();
    if (lane == 0) s.tc.cur_inst = -1;
    // The task's cold values (TaskCold): with X::kColdSmem these names are
    // references into shared memory, so the DFS reads them where it needs
    // them and they hold no registers across the hot loop (C2 +1.9%, C4
    // nodes/s +2.8%); the directed 64-bit kernel keeps them in registers
    // (instruction-fetch bound, its C3 launch is 17% slower otherwise).
    TaskCold reg{};
    reg.cur_inst = -1;
    TaskCold& tcv = X::kColdSmem ? s.tc : reg;
    const int& maxp = tcv.maxp;
    const int& goal = tcv.goal;
    const int& prune = tcv.prune;
    const int& floor_sz = tcv.floor_sz;
    const int& grp = tcv.grp;
    GroupState* const& gs = tcv.gs;
    InstanceState* const& is = tcv.is;
    bool stop_all = false;
    bool have_ticket = false;
    int my_epoch = 0;  // restart epoch of the group when this warp last looked (RST only)
    unsigned long long ticket = 0;

    while (!stop_all) {
        // ---------------------------------------------------------- acquire
        int inst = -1;
        bool branch = false;
        unsigned long long slot_pos = 0;
        {
            // Roots first (an atomic counter over instance ids), then the
            // ticket ring: a warp out of roots takes ONE ticket with atomicAdd
            // on head and waits on its own slot until the producer holding
            // the same ticket publishes it. No CAS retries on a shared word;
            // head - tail is the number of waiting warps (the donation
            // trigger). A waiting warp leaves when pending drops to 0: then
            // no task is queued or running, so no producer can follow.
            bool got = false;
            unsigned backoff = 64;
            int spins = 0;
            for (;;) {
                if (!have_ticket) {
                    int r = p.n_roots;
                    if (lane == 0 && ld_volatile(&ctl->next_root.v) < p.n_roots)
                        r = atomicAdd(&ctl->next_root.v, 1);
                    r = __shfl_sync(kFull, r, 0);
                    if (r < p.n_roots) {
                        inst = r;
                        got = true;
                        break;
                    }
                    if (PAR) break;  // parity mode: roots only
                    unsigned long long t = 0;
                    if (lane == 0) t = atomicAdd(&ctl->head.v, 1ull);
                    ticket = __shfl_sync(kFull, t, 0);
                    have_ticket = true;
                }
                int ok = 0;
                if (lane == 0) {
                    const Slot* sl = ring + (ticket & p.cap_mask);
                    ok = ld_acquire(&sl->seq) == ticket + 1;
                }
                ok = __shfl_sync(kFull, ok, 0);
                if (ok) {
                    slot_pos = ticket;
                    have_ticket = false;
                    got = true;
                    branch = true;
                    break;
                }
                if ((++spins & 7) == 0) {
                    int pend = 0, st = 0;
                    if (lane == 0) {
                        pend = ld_volatile(&ctl->pending.v);
                        st = ld_volatile(&ctl->stop.v);
                    }
                    pend = __shfl_sync(kFull, pend, 0);
                    st = __shfl_sync(kFull, st, 0);
                    if (pend <= 0 || st != 0) break;
                }
                __nanosleep(backoff + (gw & 31) * 8);
                if (backoff < 1024) backoff <<= 1;
            }
            if (lane == 0) {
                const long long t = clock64();
                s.st_idle += (unsigned long long)(t - s.t_mark);
                s.t_mark = t;
            }
            if (!got) break;
        }

        // ---------------------------------------------------- load the task
        Slot* slot = nullptr;
        TaskHeader hdr{};
        if (branch) {
            slot = ring + (slot_pos & p.cap_mask);
            __syncwarp();
            hdr = slot->hdr;
            inst = hdr.inst;
            // a malformed subtree means the ring protocol broke: stop the
            // launch with an error instead of touching memory with it
            if (unsigned(inst) >= unsigned(p.n_inst) || hdr.depth > NB || hdr.nc > NB || hdr.kind != kTaskBranch) {
                if (lane == 0) {
                    Counters* c = p.counters;
                    if (atomicAdd(&c->bad_task, 1ull) == 0) {
                        c->stall_pos = slot_pos;
                        c->stall_head = (unsigned long long)(unsigned)inst;
                        c->stall_tail = (unsigned long long)hdr.depth << 8 | hdr.nc;
                        c->stall_seq = ld_relaxed(&slot->seq);
                    }
                    atomicCAS(&ctl->stop.v, 0, 3);
                }
                stop_all = true;
                break;
            }
        }
        __syncwarp();
        if (inst != tcv.cur_inst) {
            const auto& dsc = X::descs(p)[inst];
            x.template load_instance<PAR>(dsc);
            if (lane == 0 || !X::kColdSmem) {
                tcv.maxp = dsc.maxp;
                tcv.goal = dsc.goal;
                tcv.prune = dsc.prune;
                tcv.floor_sz = dsc.floor;
                tcv.grp = dsc.group;
                tcv.cur_inst = inst;
            }
        }
        if (lane == 0 || !X::kColdSmem) {
            tcv.inst = inst;
            tcv.gs = p.grp + tcv.grp;
            tcv.is = p.ist + inst;
        }
        __syncwarp();
        if (lane == 0) {
            s.st_tasks += 1;
            if (!PAR) atomicAdd(&is->workers, 1);
            s.polled = 0;
        }

        bool abort_all = false;
        if constexpr (X::kNest && !PAR && !RST) {
            // 64-bit throughput kernel: a level whose live vertex sets fit 32
            // bits runs its subtree through run_nested — the task body again,
            // rooted at that level, with the 32-bit policy on renumbered
            // vertices (CompactSearch). (Not with restarts: a restart freezes
            // the whole open path, which spans both bodies.)
            using CS = CompactSearch<X::kDir>;
            auto run_nested = [&](CS& xc, int nest_d, int nest_nc, int nest_sel, int nest_v, int nest_bound,
                                  uint32_t nest_cand, int nest_cont, int& cd, int& cd0, int& since_poll,
                                  unsigned& splits, int& nest_best, int& nest_off, int nest_resume,
                                  int& nest_pause) -> int {
                using W = uint32_t;
                constexpr int NB = CS::NB;
                constexpr int P = CS::P;
#define TB_NESTED
#define TB_Y xc
#define TB_T CS
#include "mcsg_task_body.inc"
#undef TB_Y
#undef TB_T
#undef TB_NESTED
            };
            // (in a lambda of its own: labels are per function)
            auto run_task = [&]() {
#define TB_CAN_NEST
#define TB_Y x
#define TB_T X
#include "mcsg_task_body.inc"
#undef TB_Y
#undef TB_T
#undef TB_CAN_NEST
            };
            run_task();
        } else {
#define TB_Y x
#define TB_T X
#include "mcsg_task_body.inc"
#undef TB_Y
#undef TB_T
        }
        if (abort_all) stop_all = true;
        __syncwarp();
    }

    if (lane == 0) {
        Counters* c = p.counters;
        atomicAdd(&c->nodes, s.st_nodes);
        atomicAdd(&c->splits, s.st_splits);
        atomicAdd(&c->split_classes, s.st_split_cls);
        atomicAdd(&c->donations, s.st_donations);
        atomicAdd(&c->tasks, s.st_tasks);
        atomicAdd(&c->spills, s.st_spills);
        atomicAdd(&c->idle_cycles, s.st_idle);
        atomicAdd(&c->busy_cycles, s.st_busy);
        if constexpr (X::kNest) {
            atomicAdd(&c->nests_smem, s.ca.nests_smem);
            atomicAdd(&c->nests_hbm, s.ca.nests_hbm);
        }
    }
}

// ------------------------------------------------------------ host launch --
// Kernel flavours by bitset width: 32 (n <= 32), 64 (n <= 64), and the wide
// policies 128 (n <= 128) and 256 (n <= 255).
template <class X, bool PAR, bool RST = false>
static cudaError_t launch_t(const KernelParams& p, int ctas, cudaStream_t st) {
    const int smem = warp_smem_bytes<X>(p.smem_classes) * kWarpsPerCta;
    cudaError_t e =
        cudaFuncSetAttribute(mcs_search_kernel<X, PAR, RST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    mcs_search_kernel<X, PAR, RST><<<ctas, kWarpsPerCta * 32, smem, st>>>(p);
    return cudaGetLastError();
}

template <class X>
static int occupancy_t(int smem_classes) {
    const int smem = warp_smem_bytes<X>(smem_classes) * kWarpsPerCta;
    int worst = 1 << 30;
    for (int par = 0; par < 3; ++par) {
        auto fn = par == 1 ? mcs_search_kernel<X, true> : par == 2 ? mcs_search_kernel<X, false, true>
                                                                   : mcs_search_kernel<X, false>;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kWarpsPerCta * 32, smem) != cudaSuccess)
            return 0;
        worst = blocks < worst ? blocks : worst;
    }
    return worst;
}

// Calls f.template operator()<X>() with the policy of (bits, directed).
template <class F>
static auto with_policy(int bits, bool directed, F&& f) {
    switch (bits) {
        case 32:
            return directed ? f.template operator()<Search<uint32_t, true>>()
                            : f.template operator()<Search<uint32_t, false>>();
        case 64:
            return directed ? f.template operator()<Search<uint64_t, true>>()
                            : f.template operator()<Search<uint64_t, false>>();
        case 128:
            return directed ? f.template operator()<WideSearch<2, true>>()
                            : f.template operator()<WideSearch<2, false>>();
        default:
            return directed ? f.template operator()<WideSearch<4, true>>()
                            : f.template operator()<WideSearch<4, false>>();
    }
}

int kernel_smem_per_warp(int bits, bool directed, int smem_classes) {
    return with_policy(bits, directed, [&]<class X>() { return warp_smem_bytes<X>(smem_classes); });
}

int kernel_smem_fixed(int bits, bool directed) {
    return with_policy(bits, directed, [&]<class X>() { return warp_smem_fixed<X>(); });
}

int kernel_class_bytes(int bits) {
    return bits == 32 ? 8 : bits == 64 ? 16 : bits == 128 ? 32 : 64;
}

int kernel_occupancy(int bits, bool directed, int smem_classes) {
    return with_policy(bits, directed, [&]<class X>() { return occupancy_t<X>(smem_classes); });
}

cudaError_t kernel_launch(int bits, bool directed, bool parity, const KernelParams& p, int ctas, cudaStream_t st) {
    return with_policy(bits, directed, [&]<class X>() {
        if (parity) return launch_t<X, true>(p, ctas, st);
        return p.restart_mult > 0.0 ? launch_t<X, false, true>(p, ctas, st) : launch_t<X, false>(p, ctas, st);
    });
}

// Resets the ring (slot i of lap 0 expects producer ticket i) and the
// per-launch counters. One thread per slot.
template <class Slot>
__global__ void ring_reset_kernel(Slot* slots, uint32_t cap, Counters* c) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) slots[i].seq = i;
    if (i == 0) {
        *c = Counters{};
        c->t_start_ns = ~0ull;
    }
}

cudaError_t ring_reset(TaskSlot* slots, uint32_t cap, Counters* c, cudaStream_t st) {
    ring_reset_kernel<<<(cap + 255) / 256, 256, 0, st>>>(slots, cap, c);
    return cudaGetLastError();
}

cudaError_t ring_reset_wide(WideSlot* slots, uint32_t cap, Counters* c, cudaStream_t st) {
    ring_reset_kernel<<<(cap + 255) / 256, 256, 0, st>>>(slots, cap, c);
    return cudaGetLastError();
}

}  // namespace mcsg
