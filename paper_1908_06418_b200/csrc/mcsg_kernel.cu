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
    const int stack_limit = p.smem_classes + p.spill_classes;
    Ctl* const ctl = p.ctl;
    const int interval = p.poll_interval;

    const unsigned long long t_warp0 = globaltimer();
    const unsigned long long deadline = p.budget_ns ? t_warp0 + p.budget_ns : 0ull;
    if (lane == 0) atomicMin(&p.counters->t_start_ns, t_warp0);

    if (lane == 0) s.st_nodes = s.st_splits = s.st_donations = s.st_tasks = s.st_spills = s.st_idle = s.st_busy = 0;
    long long t_mark = clock64();
    int cur_inst = -1;
    int maxp = 0, goal = 0, prune = 1, floor_sz = 0, grp = 0;
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
            {
                const long long t = clock64();
                if (lane == 0) s.st_idle += (unsigned long long)(t - t_mark);
                t_mark = t;
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
        if (inst != cur_inst) {
            const auto& dsc = X::descs(p)[inst];
            x.template load_instance<PAR>(dsc);
            maxp = dsc.maxp;
            goal = dsc.goal;
            prune = dsc.prune;
            floor_sz = dsc.floor;
            grp = dsc.group;
            cur_inst = inst;
        }
        GroupState* const gs = p.grp + grp;
        InstanceState* const is = p.ist + inst;
        if (lane == 0) {
            s.st_tasks += 1;
            if (!PAR) atomicAdd(&is->workers, 1);
            s.polled = 0;
        }

        // Incumbent sizes. Parity: offers compare with the warp's own mapping
        // (LocalIncumbent::offer, search_core.hpp:29-31) and pruning adds the
        // external floor (size(), :25-28). Throughput: both use the group size.
        int best_local = 0, best_eff = floor_sz;
        bool skip = false;
        {
            int gb = 0, gd = 0, ge = 0;
            if (lane == 0) {
                gb = int(ld_volatile_u(&gs->best));
                gd = int(ld_volatile_u(&gs->done));
                ge = int(ld_volatile_u(&gs->epoch));
            }
            gb = __shfl_sync(kFull, gb, 0);
            gd = __shfl_sync(kFull, gd, 0);
            my_epoch = __shfl_sync(kFull, ge, 0);
            if (!PAR) best_eff = max(best_eff, gb);
            skip = gd != 0;
        }
        // prefetch the control words the first poll will read
        auto prefetch_ctl = [&]() {
            if (lane == 0) cp_async16(&s.pf[0], &ctl->stop);
            if (!PAR && lane == 1) cp_async16(&s.pf[4], &ctl->head);
            if (!PAR && lane == 2) cp_async16(&s.pf[8], &ctl->tail);
            if (!PAR && lane == 3) cp_async16(&s.pf[12], gs);
            if (!PAR && lane == 4) cp_async16(&s.pf[16], is);
            if (!PAR && lane == 5) cp_async16(&s.pf[20], &ctl->live);
            cp_async_commit();
        };
        cp_async_wait_all();  // the previous task's copies must not land after these
        __syncwarp();
        prefetch_ctl();
        int off_thr = PAR ? best_local : best_eff;                  // offer when |M| > off_thr
        int prn_thr = prune ? max(best_eff, goal - 1) : -1;         // prune when bound <= prn_thr
        auto raise_best = [&](int b) {
            best_local = max(best_local, b);
            best_eff = max(best_eff, b);
            off_thr = PAR ? best_local : best_eff;
            prn_thr = prune ? max(best_eff, goal - 1) : -1;
        };

        int d, root, base = 0, nc, bound, sel = 0, v = 0;
        W cand{};
        int cont = 0;
        unsigned key = kNoKey;
        bool have_key = false;
        bool at_next = false;  // true: resume the u loop of the task's level
        if (!branch) {
            const auto& dsc = X::descs(p)[inst];
            nc = dsc.n_init;
            x.load_root(dsc, nc);
            __syncwarp();
            d = root = 0;
            x.load_level(0, nc);
            unsigned sm;
            key = x.template scan_key<!PAR>(nc, &sm);
            have_key = true;
            bound = int(sm);
        } else {
            d = root = hdr.depth;
            nc = hdr.nc;
            x.load_task(*slot, nc, d);
            sel = hdr.sel;
            v = hdr.v;
            bound = hdr.bound;
            cand = X::slot_cand(*slot);
            cont = hdr.cont;
            __syncwarp();
            if (lane == 0) st_release(&slot->seq, slot_pos + p.cap_mask + 1);  // free the slot
            x.load_level(0, nc);
            x.prep_v(v, sel);
            at_next = true;
            // task-level prune (engine_parallel.cpp:148-155): every child would prune
            if (bound <= prn_thr) skip = true;
        }
        if (skip) {  // nothing of this task is entered (or counted)
            cand = W{};
            cont = 0;
        }

        // nodes until the next poll (cd), counted from cd0; a throughput task
        // polls early once, and every kFastPoll nodes while warps wait for work
        // a root task, and a subtree donated while many warps waited, polls
        // early: a launch with few roots fans out in tens of microseconds
        int cd0 = (!PAR && (!branch || hdr.fanout)) ? kFastPoll : interval;
        int cd = cd0;
        int since_poll = 0;  // nodes counted between the last two polls (dead-end monitor)
        int lim = 0;           // u loop: prune threshold minus |M|+1
        unsigned splits = 0;   // flushed to s.st_splits at polls and at the task's end
        bool abort_all = false;

        // Stores M ∪ {(v,u)} (|M| = dd) as the instance's mapping if it still
        // improves there, then raises the group size (an incumbent size never
        // exceeds a mapping actually written).
        auto offer = [&](int dd, int uu) {
            int stored = 0;
            if (lane == 0)
                while (atomicCAS(&is->lock, 0, 1) != 0) __nanosleep(64);
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                stored = ld_volatile_u(&is->map_size) < unsigned(dd + 1);
            }
            stored = __shfl_sync(kFull, stored, 0);
            if (stored) {
                for (int k = lane; k <= dd; k += 32) {
                    int mv, mu;
                    if (k < root) {
                        mv = s.map_v[k];
                        mu = s.map_u[k];
                    } else if (k < dd) {
                        const unsigned long long f = s.f_word[k];
                        mv = fr_v(f);
                        mu = fr_u(f);
                    } else {
                        mv = v;
                        mu = uu;
                    }
                    is->map_v[k] = uint8_t(mv);
                    is->map_u[k] = uint8_t(mu);
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    is->map_size = unsigned(dd + 1);
                    __threadfence();
                    atomicMax(&gs->best, unsigned(dd + 1));
                    // DeadEndMonitor::note_improvement (heuristics.hpp:45)
                    // (restarts.cpp:91: at_improvement = nodes on improvement)
                    if (p.deadend_abs || p.deadend_rel > 0.0 || (RST && p.restart_mult > 0.0))
                        atomicMax(&gs->at_improve, *reinterpret_cast<volatile unsigned long long*>(&gs->nodes));
                }
                // push the size to the other devices' incumbents (NVLink P2P)
                if (grp == 0 && lane < p.n_peers) atomicMax_system(&p.peer_grp[lane]->best, unsigned(dd + 1));
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                atomicExch(&is->lock, 0);
            }
        };

        // Hands level f's remaining u candidates (all of them, or the half
        // the donor would reach last) and its continuation to the ring as a
        // frozen subtree. False when the producer watchdog fired (abort).
        auto donate_level = [&](int f, bool all, bool fanout) -> bool {
            const W fc = s.f_cand[f];
            const unsigned long long fw = s.f_word[f];
            const int cnt = set_popc(fc);
            // hand over the half the donor would reach last (throughput mode
            // walks u from the top: the lower half)
            W keep = fc;
            if (all || cnt < 2)
                keep = W{};
            else
                for (int i = 0; i < cnt / 2; ++i) keep = set_drop_lowest(keep);
            const W give = set_andnot(fc, keep);
            // the donor counted these children (and the continuation) when it
            // selected level f; the receiver counts them when it resumes
            cd += set_popc(give) + (fr_cont(fw) != 0);
            // producer ticket; a warp is (probably) already waiting on it.
            // The slot is free once the consumer of ticket pos - cap released
            // it; the ring is far larger than the warp count, so this wait is
            // normally zero.
            unsigned long long pos = 0;
            int stalled = 0;
            if (lane == 0) {
                atomicAdd(&ctl->pending.v, 1);
                atomicAdd(&is->open_tasks, 1);
                pos = atomicAdd(&ctl->tail.v, 1ull);
                const Slot* sl = ring + (pos & p.cap_mask);
                // watchdog: a slot that stays taken for 2 s means the ring
                // invariant broke — stop the launch with an error, never hang
                unsigned long long t_wait = 0, seq;
                unsigned spins = 0;
                while ((seq = ld_acquire(&sl->seq)) != pos) {
                    __nanosleep(32);
                    if ((++spins & 1023u) == 0) {
                        const unsigned long long now = globaltimer();
                        if (!t_wait) t_wait = now;
                        else if (now - t_wait > p.ring_watchdog_ns) {
                            Counters* c = p.counters;
                            if (atomicAdd(&c->ring_stall, 1ull) == 0) {
                                c->stall_pos = pos;
                                c->stall_head = ld_relaxed(&ctl->head.v);
                                c->stall_tail = ld_relaxed(&ctl->tail.v);
                                c->stall_seq = seq;
                            }
                            atomicCAS(&ctl->stop.v, 0, 3);
                            stalled = 1;
                            break;
                        }
                    }
                }
            }
            if (__shfl_sync(kFull, stalled, 0)) {
                abort_all = true;
                return false;
            }
            pos = __shfl_sync(kFull, pos, 0);
            Slot* sl = ring + (pos & p.cap_mask);
            const int fnc = fr_nc(fw);
            x.store_task(*sl, fr_base(fw), fnc);
            for (int k = lane; k < f; k += 32) {
                int mv, mu;
                if (k < root) {
                    mv = s.map_v[k];
                    mu = s.map_u[k];
                } else {
                    const unsigned long long g2 = s.f_word[k];
                    mv = fr_v(g2);
                    mu = fr_u(g2);
                }
                sl->map_v[k] = uint8_t(mv);
                sl->map_u[k] = uint8_t(mu);
            }
            if (lane == 0) {
                TaskHeader h;
                h.inst = inst;
                h.kind = kTaskBranch;
                h.depth = uint8_t(f);
                h.nc = uint8_t(fnc);
                h.sel = uint8_t(fr_sel(fw));
                h.v = uint8_t(fr_v(fw));
                h.bound = uint8_t(fr_bound(fw));
                h.cont = uint8_t(fr_cont(fw));
                h.fanout = fanout ? 1 : 0;
                h.pad1 = 0;
                X::put_cand(*sl, h, give);
                sl->hdr = h;
                s.f_cand[f] = keep;
                s.f_word[f] = fw & ~kFrameContByte;  // the continuation left with the task
            }
            fence_acq_rel_gpu();  // payload before the release of the slot
            __syncwarp();
            if (lane == 0) {
                st_release(&sl->seq, pos + 1);
                s.st_donations += 1;
            }
            return true;
        };

        // Periodic poll: stop/deadline/cancel, group done, shared incumbent,
        // and subtree donation to idle warps. Returns false to end the task.
        auto poll = [&]() -> bool {
            // values prefetched at the previous poll (one interval stale: stale
            // reads only delay a stop or weaken pruning)
            cp_async_wait_all();
            __syncwarp();
            int st = int(s.pf[0]);
            long long waiting = 0;  // warps holding a ticket no producer has served yet
            if (!PAR) {
                const unsigned long long hd = (unsigned long long)s.pf[4] | ((unsigned long long)s.pf[5] << 32);
                const unsigned long long tl = (unsigned long long)s.pf[8] | ((unsigned long long)s.pf[9] << 32);
                waiting = (long long)(hd - tl);
            }
            const int gb = PAR ? 0 : int(s.pf[12]);  // GroupState::best
            const int gd = PAR ? 0 : int(s.pf[13]);  // GroupState::done
            const int workers = int(s.pf[19]);      // InstanceState::workers
            const int live = max(int(s.pf[20]), 1); // instances still open
            // Every prefetched word is read above this barrier: the next
            // prefetch rewrites the buffer asynchronously, and a word read
            // after it could differ between lanes (a diverged warp).
            __syncwarp();
            prefetch_ctl();
            if (lane == 0 && st == 0) {
                if (deadline && globaltimer() >= deadline) {
                    atomicCAS(&ctl->stop.v, 0, 1);
                    st = 1;
                }
                if (st == 0 && gw == 0 && p.cancel && *p.cancel) {
                    atomicCAS(&ctl->stop.v, 0, 2);
                    st = 2;
                }
            }
            st = __shfl_sync(kFull, st, 0);
            if (st != 0) {
                abort_all = true;
                return false;
            }
            if (PAR) return true;
            if (gd != 0) return false;
            if (gb > best_eff) raise_best(gb);
            if (p.deadend_abs || p.deadend_rel > 0.0 || (RST && p.restart_mult > 0.0)) {
                // the group's node count since its last improvement drives
                // deadend_check (heuristics.cpp:103-112) and restart_due
                // (restarts.cpp:66-70)
                int sus = 0, ep = my_epoch;
                if (lane == 0) {
                    const unsigned long long add = (unsigned long long)max(since_poll, 0);
                    const unsigned long long total = atomicAdd(&gs->nodes, add) + add;
                    const unsigned long long at = *reinterpret_cast<volatile unsigned long long*>(&gs->at_improve);
                    const unsigned long long since = total - at;
                    sus = (p.deadend_abs && since >= p.deadend_abs) ||
                          (p.deadend_rel > 0.0 && double(since) >= p.deadend_rel * double(at > 0 ? at : 1ull));
                    if (sus) {
                        gs->suspect = 1u;
                        atomicExch(&gs->done, 1u);
                    }
                    // a restart is due: the first warp to see it rearms the
                    // monitor (at_improvement = nodes) and opens a new epoch
                    if (RST && p.restart_mult > 0.0 && double(since) >= p.restart_mult * double(at > 0 ? at : 1ull) &&
                        atomicCAS(&gs->at_improve, at, total) == at)
                        atomicAdd(&gs->epoch, 1u);
                    ep = int(ld_volatile_u(&gs->epoch));
                }
                if (__shfl_sync(kFull, sus, 0)) return false;
                ep = __shfl_sync(kFull, ep, 0);
                if (RST && ep != my_epoch) {
                    my_epoch = ep;
                    // Restart: freeze the open path — every level with work,
                    // the current one included — into the ring as frozen
                    // subtrees (the pool of segments, restarts.cpp:80-97),
                    // end this task, and take the oldest queued subtree next.
                    // Skipped when the ring lacks room (the search stays
                    // complete either way).
                    long long queued = 0;
                    if (lane == 0) queued = (long long)(ld_relaxed(&ctl->tail.v) - ld_relaxed(&ctl->head.v));
                    queued = __shfl_sync(kFull, queued, 0);
                    // (only once the current node is selected: the root
                    // count's poll comes before its select)
                    if ((set_any(cand) || cont) && queued + (d - root + 1) < (long long)(p.cap_mask + 1) / 2) {
                        s.f_cand[d] = cand;  // the current level becomes a frame like the others
                        s.f_word[d] = pack_frame(base, nc, sel, v, bound, cont, 0);
                        __syncwarp();
                        int frozen = 0;
                        for (int lv = root; lv <= d; ++lv) {
                            if (!set_any(s.f_cand[lv]) && !fr_cont(s.f_word[lv])) continue;
                            if (!donate_level(lv, true, false)) return false;
                            ++frozen;
                        }
                        cand = W{};
                        cont = 0;
                        if (lane == 0) atomicAdd(&p.counters->frozen, (unsigned long long)frozen);
                        return false;
                    }
                }
            }
            // Donate when warps wait for work, or — fairness between the
            // instances of a batch — when this instance runs on few warps and
            // the queue is short: a busy batch would otherwise never hand a
            // small instance's subtrees to anyone (FIFO tickets serve them next).
            const int total_warps = int(gridDim.x) * kWarpsPerCta;
            const bool starved = 2 * workers * live < total_warps && waiting > -kStarvedQueue;
            // while many warps wait (a fresh launch with few roots), poll
            // again soon: the launch fans out in tens of microseconds
            const bool fanout = waiting > total_warps / 4;  // 2..32 measure alike (tools/fanout_sweep.sh)
            if (fanout) cd = cd0 = kFastPoll;
            if ((waiting <= 0 && !starved) || d <= root) return true;
            // The prefetched counters are one poll old: confirm with a fresh
            // read before taking a producer ticket, so that the queue stays
            // short (bounded by the warps racing here plus kStarvedQueue, far
            // below the ring capacity: producers never wait on a full ring).
            {
                long long fresh = 0;
                if (lane == 0) fresh = (long long)(ld_relaxed(&ctl->head.v) - ld_relaxed(&ctl->tail.v));
                fresh = __shfl_sync(kFull, fresh, 0);
                const bool starved_now = 2 * workers * live < total_warps && fresh > -kStarvedQueue;
                if (fresh <= 0 && !starved_now) return true;
            }
            // donate the shallowest level that still owns work
            int f = -1;
            for (int b0 = root; b0 < d && f < 0; b0 += 32) {
                const int lv = b0 + lane;
                bool has = false;
                if (lv < d) has = set_any(s.f_cand[lv]) || fr_cont(s.f_word[lv]);
                const unsigned m = __ballot_sync(kFull, has);
                if (m) f = b0 + __ffs(m) - 1;
            }
            if (f < 0) return true;
            return donate_level(f, false, fanout);
        };

// Node counting (search_core.hpp:130). Nodes are counted in bulk when a level
// is selected: its |R*| children and its continuation are all counted nodes
// (each is entered, even when its bound prunes it at once), so the u loop
// carries no per-child counter. What a stop leaves unentered is subtracted at
// the task's end; a donation hands its share of the count to the receiver.
// The periodic poll runs when the countdown crosses zero.
#define MCSG_COUNT_NODES(k)                                                     \
    cd -= (k);                                                                 \
    if (cd <= 0) {                                                             \
        since_poll = cd0 - cd;                                                 \
        if (lane == 0) {                                                       \
            s.polled += (unsigned long long)(long long)since_poll;             \
            s.st_splits += splits;                                             \
        }                                                                      \
        splits = 0;                                                            \
        cd = cd0 = interval;                                                   \
        if (!poll()) goto finish;                                              \
    }

        if (!skip) {
            if (!at_next) {
                // the root node (search_core.hpp:129-166)
                MCSG_COUNT_NODES(1);
                if (bound <= prn_thr) goto pop;
                goto select;
            }
            // a donated subtree: its remaining children and continuation (the
            // level's first-child offer happened in the donor)
            cd -= set_popc(cand) + (cont != 0);
            goto next;

        select:
            // ---- the node survived its prune test: choose class and vertex
            if (!have_key) key = x.template scan_key<!PAR>(nc, nullptr);
            if (key == kNoKey) goto pop;
            sel = X::key_slot(key);
            {
                const W lsel = x.class_l(sel);
                if constexpr (PAR) v = x.select_vertex(lsel);
                else v = set_top(lsel);  // G is relabelled in reverse select_vertex order
                cand = x.class_r(sel);
                cont = kContOwned | (set_popc(lsel) <= set_popc(cand) ? kContDec : 0);
            }
            x.prep_v(v, sel);
            // Incumbent offer at the entry of the level's first child
            // (search_core.hpp:145-155). Only a first child can improve: once
            // it is entered the threshold is >= d+1 for its siblings, for
            // later selects at this depth and after every pop back here. It
            // runs before the level's nodes are counted (so a restart that
            // freezes the level at the count's poll finds the offer done); a
            // stop here counts the one child it entered.
            if (d + 1 > off_thr) {
                const int u = PAR ? set_ctz(cand) : set_top(cand);
                offer(d, u);
                raise_best(d + 1);
                const bool goal_hit = goal > 0 && d + 1 >= goal;                 // search_core.hpp:147-150
                const bool max_hit = prune && goal == 0 && d + 1 >= maxp;        // search_core.hpp:151-154
                if (goal_hit || max_hit) {
                    if (lane == 0) {
                        if (goal_hit) gs->reached = 1;
                        if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                    }
                    if (grp == 0 && lane < p.n_peers) {  // stop every device
                        if (goal_hit) atomicExch_system(&p.peer_grp[lane]->reached, 1);
                        atomicExch_system(&p.peer_grp[lane]->done, 1u);
                    }
                    cd -= 1;  // u was entered; nothing else of this level is
                    cand = W{};
                    cont = 0;
                    goto finish;
                }
            }
            MCSG_COUNT_NODES(set_popc(cand) + 1);  // the children and the continuation

        next:
            // ---- u loop (search_core.hpp:183-200): children in ascending u
            // Parity mode walks u in ascending id (the reference's order);
            // throughput mode from the top (one FLO instead of BREV + FLO).
            lim = prn_thr - (d + 1);  // a child survives when its class sum exceeds lim
            while (set_any(cand)) {
                const int u = PAR ? set_ctz(cand) : set_top(cand);  // the child's entry (counted at select)
                cand = set_without(cand, u);
                typename X::HParts h;
                x.h_parts(u, h);
                const int csum = int(x.child_sum(u, h));
                if (csum <= lim) continue;  // pruned at entry
                const int cbound = d + 1 + csum;
                // ---- materialise the child (filter_classes) one level up
                int cb = base + nc;
                const int need = min(nc * P, NB);
                if constexpr (X::kSpill) {
                    // a level never straddles shared memory and the HBM spill area
                    if (cb < x.cap && cb + need > x.cap) {
                        cb = x.cap;
                        if (lane == 0) s.st_spills += 1;
                    }
                }
                if (cb + need > stack_limit) {  // cannot happen with the host's sizing
                    if (lane == 0) {
                        atomicAdd(&p.counters->overflow, 1ull);
                        atomicCAS(&ctl->stop.v, 0, 3);
                    }
                    abort_all = true;
                    goto finish;
                }
                // every lane stores the same (uniform) frame: no branch
                s.f_cand[d] = cand;
                s.f_word[d] = pack_frame(base, nc, sel, v, bound, cont, u);
                unsigned ckey;
                const int cnc = x.template split<!PAR>(u, v, h, cb, &ckey);
                __syncwarp();
                ++splits;
                ++d;
                base = cb;
                nc = cnc;
                bound = cbound;
                x.load_level(base, nc);
                key = ckey;
                have_key = true;
                goto select;
            }
            // ---- v left unmatched (search_core.hpp:201-212): a counted node
            if (cont) {  // (counted at select)
                x.cont_step(sel, cont, base, bound);
                __syncwarp();
                cont = 0;
                have_key = false;
                if (bound <= prn_thr) goto pop;
                goto select;
            }

        pop:
            // ---- return to the parent level
            if (d == root) goto finish;
            --d;
            {
                const unsigned long long f = s.f_word[d];
                cand = s.f_cand[d];
                base = fr_base(f);
                nc = fr_nc(f);
                sel = fr_sel(f);
                v = fr_v(f);
                bound = fr_bound(f);
                cont = fr_cont(f);
            }
            x.load_level(base, nc);
            x.prep_v(v, sel);
            goto next;
        }
#undef MCSG_COUNT_NODES
    finish : {
        {
            const long long t = clock64();
            if (lane == 0) s.st_busy += (unsigned long long)(t - t_mark);
            t_mark = t;
        }
        {
            // nodes counted at select but never entered (a stop, or levels
            // abandoned by an abort): the open levels' remaining children
            // and continuations, plus the current level's
            int left = 0;
            for (int lv = root + lane; lv < d; lv += 32) left += set_popc(s.f_cand[lv]) + (fr_cont(s.f_word[lv]) != 0);
            cd += int(__reduce_add_sync(kFull, unsigned(left))) + set_popc(cand) + (cont != 0);
        }
        if (lane == 0) {
            const unsigned long long task_nodes = s.polled + (unsigned long long)(long long)(cd0 - cd);
            s.st_nodes += task_nodes;
            s.st_splits += splits;
            if (task_nodes) atomicAdd(&is->nodes, task_nodes);
            if (!abort_all) {
                if (!PAR) atomicSub(&is->workers, 1);
                const int left = atomicSub(&is->open_tasks, 1) - 1;
                if (left == 0) {
                    is->t_done_ns = globaltimer();
                    atomicSub(&ctl->live.v, 1);
                    if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                    // portfolio across devices: a complete member search proves
                    // the optimum for every member (portfolio.cpp:271-279)
                    if (grp == 0 && p.peer_done_on_complete)
                        for (int q = 0; q < p.n_peers; ++q) atomicExch_system(&p.peer_grp[q]->done, 1u);
                }
                atomicSub(&ctl->pending.v, 1);
            }
        }
    }
        if (abort_all) stop_all = true;
        __syncwarp();
    }

    if (lane == 0) {
        Counters* c = p.counters;
        atomicAdd(&c->nodes, s.st_nodes);
        atomicAdd(&c->splits, s.st_splits);
        atomicAdd(&c->donations, s.st_donations);
        atomicAdd(&c->tasks, s.st_tasks);
        atomicAdd(&c->spills, s.st_spills);
        atomicAdd(&c->idle_cycles, s.st_idle);
        atomicAdd(&c->busy_cycles, s.st_busy);
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
