// McSplit branch-and-bound on sm_100a: one warp owns one DFS, lanes own label
// classes, the DFS stack lives in shared memory and spills to HBM, subtrees
// move between warps through a lock-free ring in HBM.
//
// Reference semantics restated (file:line under /root/reference/proj):
//   node entry / counting         src/search_core.hpp:129-131
//   incumbent offer + stops       src/search_core.hpp:145-155, src/solve.cpp:19-28
//   bound (Eq. 1)                 src/label_classes.cpp:41-45
//   prune test                    src/search_core.hpp:166
//   select_label_class            src/label_classes.cpp:47-67
//   select_vertex                 src/label_classes.cpp:69-78
//   u loop, ascending ids         src/search_core.hpp:183-200
//   filter_classes (2/4-way)      src/label_classes.cpp:80-108
//   v-unmatched continuation      src/search_core.hpp:201-212
//   task queue / delegation       src/task_queue.cpp, src/engine_parallel.cpp:86-117
//
// Bitset form (n <= 64): bit i of a class side <-> vertex id i, so "lowest id"
// is ctz and every selection rule is a total order on ids; the DFS visits the
// reference's nodes in the reference's order when donation is off ("parity
// mode"), which the tests check node-for-node.
#include <cuda_runtime.h>

#include <cstdint>

#include "mcsg_device.h"

namespace mcsg {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kNoKey = 0xffffffffu;

template <typename W>
struct Cls {
    W l, r;
};

template <typename W>
struct Bits;
template <>
struct Bits<uint32_t> {
    static constexpr int n = 32;
    __device__ static __forceinline__ int popc(uint32_t x) { return __popc(x); }
    __device__ static __forceinline__ int ctz(uint32_t x) { return __ffs(x) - 1; }
};
template <>
struct Bits<uint64_t> {
    static constexpr int n = 64;
    __device__ static __forceinline__ int popc(uint64_t x) { return __popcll(x); }
    __device__ static __forceinline__ int ctz(uint64_t x) { return __ffsll(x) - 1; }
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int ld_volatile(const int32_t* p) {
    return *reinterpret_cast<const volatile int32_t*>(p);
}
__device__ __forceinline__ unsigned ld_volatile_u(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// select_label_class key (label_classes.cpp:47-67): min over classes of
// (max(|L|,|R|), min(|L|,|R|), lowest left id); low 7 bits carry the slot.
template <typename W>
__device__ __forceinline__ unsigned class_key(int pl, int pr, W l, int slot) {
    unsigned mx = pl > pr ? pl : pr;
    unsigned mn = pl < pr ? pl : pr;
    return (mx << 20) | (mn << 13) | (unsigned(Bits<W>::ctz(l)) << 7) | unsigned(slot);
}

// Per-warp shared-memory image. The class stack follows it (dynamic size).
template <typename W, bool DIR>
struct WarpSmem {
    static constexpr int NB = Bits<W>::n;
    W out_g[NB];
    W out_h[NB];
    W in_g[DIR ? NB : 1];
    W in_h[DIR ? NB : 1];
    W f_cand[kMaxDepth + 1];
    uint16_t vkey[NB];
    uint16_t f_base[kMaxDepth + 1];
    uint8_t f_nc[kMaxDepth + 1];
    uint8_t f_sel[kMaxDepth + 1];
    uint8_t f_v[kMaxDepth + 1];
    uint8_t f_bound[kMaxDepth + 1];
    uint8_t f_cont[kMaxDepth + 1];
    uint8_t map_v[kMaxDepth + 1];
    uint8_t map_u[kMaxDepth + 1];
};

template <typename W, bool DIR>
__host__ __device__ constexpr int warp_smem_fixed() {
    return (int)((sizeof(WarpSmem<W, DIR>) + 15) & ~size_t(15));
}

template <typename W, bool DIR>
__host__ __device__ constexpr int warp_smem_bytes(int classes) {
    return (warp_smem_fixed<W, DIR>() + classes * int(sizeof(Cls<W>)) + 15) & ~15;
}

struct SplitOut {
    int nc;
    unsigned sum;
    unsigned key;
};

// filter_classes (label_classes.cpp:80-108) fused with compute_bound and
// select_label_class of the child: lane j splits parent classes j, j+32 by the
// adjacency of (v,u), ballots compact the non-empty parts into the child level,
// and two warp reductions return Σ min(|L|,|R|) and the child's best class key.
template <typename W, bool DIR>
__device__ __forceinline__ SplitOut split_level(const Cls<W>* P, int nc, W keep_l, W keep_r,
                                                W ao, W ai, W bo, W bi, Cls<W>* Q, int lane,
                                                unsigned lt) {
    int total = 0;
    unsigned sum = 0, key = kNoKey;
    for (int j0 = 0; j0 < nc; j0 += 32) {
        const int j = j0 + lane;
        W l = 0, r = 0;
        if (j < nc) {
            Cls<W> c = P[j];
            l = c.l & keep_l;
            r = c.r & keep_r;
        }
        if constexpr (!DIR) {
            const W l1 = l & ao, r1 = r & bo;
            const W l0 = l ^ l1, r0 = r ^ r1;
            const bool k0 = (l0 != 0) & (r0 != 0);
            const bool k1 = (l1 != 0) & (r1 != 0);
            const unsigned m0 = __ballot_sync(kFull, k0);
            const unsigned m1 = __ballot_sync(kFull, k1);
            const int c0 = __popc(m0);
            const int p0 = total + __popc(m0 & lt);
            const int p1 = total + c0 + __popc(m1 & lt);
            const int pl1 = Bits<W>::popc(l1), pr1 = Bits<W>::popc(r1);
            const int pl0 = Bits<W>::popc(l) - pl1, pr0 = Bits<W>::popc(r) - pr1;
            sum += unsigned(min(pl0, pr0) + min(pl1, pr1));
            if (k0) {
                Q[p0] = Cls<W>{l0, r0};
                key = min(key, class_key<W>(pl0, pr0, l0, p0));
            }
            if (k1) {
                Q[p1] = Cls<W>{l1, r1};
                key = min(key, class_key<W>(pl1, pr1, l1, p1));
            }
            total += c0 + __popc(m1);
        } else {
            // code(v,x) = out bit | in bit << 1: none, forward, backward, both.
            const W lo = l & ao, li = l & ai, ro = r & bo, ri = r & bi;
            const W lp[4] = {l & ~(ao | ai), lo & ~ai, li & ~ao, lo & ai};
            const W rp[4] = {r & ~(bo | bi), ro & ~bi, ri & ~bo, ro & bi};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool kk = (lp[k] != 0) & (rp[k] != 0);
                const unsigned m = __ballot_sync(kFull, kk);
                const int p = total + __popc(m & lt);
                const int pl = Bits<W>::popc(lp[k]), pr = Bits<W>::popc(rp[k]);
                sum += unsigned(min(pl, pr));
                if (kk) {
                    Q[p] = Cls<W>{lp[k], rp[k]};
                    key = min(key, class_key<W>(pl, pr, lp[k], p));
                }
                total += __popc(m);
            }
        }
    }
    sum = __reduce_add_sync(kFull, sum);
    key = __reduce_min_sync(kFull, key);
    return {total, sum, key};
}

// compute_bound + select_label_class over a stored level (root and
// continuation nodes, whose classes were not produced by a split).
template <typename W>
__device__ __forceinline__ void scan_level(const Cls<W>* P, int nc, int lane, unsigned& sum,
                                           unsigned& key) {
    unsigned s = 0, k = kNoKey;
    for (int j = lane; j < nc; j += 32) {
        Cls<W> c = P[j];
        const int pl = Bits<W>::popc(c.l), pr = Bits<W>::popc(c.r);
        s += unsigned(min(pl, pr));
        k = min(k, class_key<W>(pl, pr, c.l, j));
    }
    sum = __reduce_add_sync(kFull, s);
    key = __reduce_min_sync(kFull, k);
}

// select_vertex (label_classes.cpp:69-78): max degree, then lowest id.
template <typename W>
__device__ __forceinline__ int select_vertex(W l, const uint16_t* vkey, int lane) {
    unsigned k = kNoKey;
#pragma unroll
    for (int b = lane; b < Bits<W>::n; b += 32)
        if ((l >> b) & 1) k = min(k, unsigned(vkey[b]));
    k = __reduce_min_sync(kFull, k);
    return int(k & 63u);
}

template <typename W, bool DIR>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    mcs_search_kernel(KernelParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using S = WarpSmem<W, DIR>;
    constexpr int NB = Bits<W>::n;
    constexpr int kParts = DIR ? 4 : 2;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerCta + wib;
    const unsigned lt = lanemask_lt();
    const int cap = p.smem_classes;
    const int per_warp = warp_smem_bytes<W, DIR>(cap);
    S& s = *reinterpret_cast<S*>(smem_raw + size_t(wib) * per_warp);
    Cls<W>* const scls = reinterpret_cast<Cls<W>*>(smem_raw + size_t(wib) * per_warp +
                                                   warp_smem_fixed<W, DIR>());
    Cls<W>* const gcls = reinterpret_cast<Cls<W>*>(p.spill) + size_t(gw) * p.spill_classes;
    const int stack_limit = cap + p.spill_classes;
    auto level = [&](int base) -> Cls<W>* { return base < cap ? scls + base : gcls + (base - cap); };

    const unsigned long long t_warp0 = globaltimer();
    const unsigned long long deadline = p.budget_ns ? t_warp0 + p.budget_ns : 0ull;
    if (lane == 0) atomicMin(&p.counters->t_start_ns, t_warp0);

    unsigned long long nodes = 0, sum_cls = 0, splits = 0, split_cls = 0, donations = 0;
    unsigned long long tasks = 0, spills = 0;
    int cur_inst = -1;
    int n_g = 0, maxp = 0, goal = 0, prune = 1, floor_sz = 0, grp = 0;
    bool stop_all = false;

    while (!stop_all) {
        // ------------------------------------------------------------ acquire
        int inst = -1;
        int kind = kTaskRoot;
        unsigned long long slot_pos = 0;
        {
            int got = -1;  // 0 root, 1 queue, -1 none
            bool registered_idle = false;
            unsigned backoff = 32;
            for (;;) {
                int r = p.n_inst;
                if (lane == 0 && ld_volatile(p.next_root) < p.n_inst) r = atomicAdd(p.next_root, 1);
                r = __shfl_sync(kFull, r, 0);
                if (r < p.n_inst) {
                    inst = r;
                    got = 0;
                    break;
                }
                // queue (Vyukov bounded MPMC ring)
                int ok = 0;
                unsigned long long pos = 0;
                if (lane == 0) {
                    for (;;) {
                        pos = *reinterpret_cast<volatile unsigned long long*>(p.head);
                        TaskSlot* sl = p.slots + (pos & p.cap_mask);
                        const unsigned long long seq = ld_acquire(&sl->seq);
                        const long long dif = (long long)(seq - (pos + 1));
                        if (dif == 0) {
                            if (atomicCAS(p.head, pos, pos + 1) == pos) {
                                ok = 1;
                                break;
                            }
                        } else if (dif < 0) {
                            break;  // empty
                        }
                    }
                }
                ok = __shfl_sync(kFull, ok, 0);
                if (ok) {
                    slot_pos = __shfl_sync(kFull, pos, 0);
                    got = 1;
                    break;
                }
                int pend = 0, st = 0;
                if (lane == 0) {
                    if (!registered_idle) atomicAdd(p.idle, 1);
                    pend = ld_volatile(p.pending);
                    st = ld_volatile(p.stop);
                }
                registered_idle = true;
                pend = __shfl_sync(kFull, pend, 0);
                st = __shfl_sync(kFull, st, 0);
                if (pend <= 0 || st != 0) break;
                __nanosleep(backoff);
                if (backoff < 2048) backoff <<= 1;
            }
            if (registered_idle && lane == 0) atomicSub(p.idle, 1);
            if (got < 0) break;
            kind = got == 0 ? kTaskRoot : kTaskBranch;
        }

        // ---------------------------------------------------- load the task
        TaskSlot* slot = nullptr;
        TaskHeader hdr{};
        if (kind == kTaskBranch) {
            slot = p.slots + (slot_pos & p.cap_mask);
            if (lane == 0) __threadfence();
            __syncwarp();
            hdr = slot->hdr;
            inst = hdr.inst;
        }
        if (inst != cur_inst) {
            const InstanceDesc& d = p.inst[inst];
            for (int i = lane; i < NB; i += 32) {
                s.out_g[i] = W(d.out_g[i]);
                s.out_h[i] = W(d.out_h[i]);
                if constexpr (DIR) {
                    s.in_g[i] = W(d.in_g[i]);
                    s.in_h[i] = W(d.in_h[i]);
                }
                s.vkey[i] = d.vkey[i];
            }
            n_g = d.n_g;
            maxp = d.maxp;
            goal = d.goal;
            prune = d.prune;
            floor_sz = d.floor;
            grp = d.group;
            cur_inst = inst;
        }
        GroupState* const gs = p.grp + grp;
        InstanceState* const is = p.ist + inst;
        ++tasks;

        int d, root, base, nc, bound;
        unsigned key = kNoKey;
        bool keyvalid = false;
        int sel = 0, v = 0;
        W cand = 0;
        bool cont = false;
        int phase;  // 0 ENTER, 1 NEXT
        // Best sizes: best_local backs offers (LocalIncumbent::offer compares
        // with its own mapping only, search_core.hpp:29-31); best_eff adds the
        // external floor and, when sharing, the group incumbent (size()).
        int best_local = 0, best_eff = floor_sz;
        bool skip = false;
        {
            int gb = 0, gd = 0;
            if (lane == 0) {
                gb = (int)ld_volatile_u(&gs->best);
                gd = (int)ld_volatile_u(&gs->done);
            }
            gb = __shfl_sync(kFull, gb, 0);
            gd = __shfl_sync(kFull, gd, 0);
            if (p.donate) best_eff = max(best_eff, gb);
            skip = gd != 0;
        }

        if (kind == kTaskRoot) {
            const InstanceDesc& dd = p.inst[inst];
            nc = dd.n_init;
            for (int i = lane; i < nc; i += 32) scls[i] = Cls<W>{W(dd.init_l[i]), W(dd.init_r[i])};
            __syncwarp();
            d = root = 0;
            base = 0;
            unsigned sum;
            scan_level<W>(scls, nc, lane, sum, key);
            bound = int(sum);
            keyvalid = true;
            phase = 0;
        } else {
            d = root = hdr.depth;
            base = 0;
            nc = hdr.nc;
            for (int i = lane; i < nc; i += 32) scls[i] = Cls<W>{W(slot->cls_l[i]), W(slot->cls_r[i])};
            for (int i = lane; i < d; i += 32) {
                s.map_v[i] = slot->map_v[i];
                s.map_u[i] = slot->map_u[i];
            }
            sel = hdr.sel;
            v = hdr.v;
            bound = hdr.bound;
            cand = W(hdr.cand);
            cont = hdr.cont != 0;
            __syncwarp();
            // release the slot for the next lap of the ring
            if (lane == 0) st_release(&slot->seq, slot_pos + p.cap_mask + 1);
            phase = 1;
            // task-level prune (engine_parallel.cpp:148-155): every child would prune
            if (p.donate && prune && bound <= max(best_eff, goal - 1)) skip = true;
        }

        unsigned long long task_nodes = 0;
        bool abort_all = false;
        if (!skip) {
            for (;;) {
                if (phase == 0) {
                    // ------------------------------------------------ ENTER
                    ++task_nodes;
                    sum_cls += unsigned(nc);
                    if ((task_nodes & unsigned(p.poll_mask)) == 0) {
                        int st = 0, gb = 0, gd = 0, idl = 0;
                        if (lane == 0) {
                            st = ld_volatile(p.stop);
                            if (st == 0 && deadline && globaltimer() >= deadline) {
                                atomicCAS(p.stop, 0, 1);
                                st = 1;
                            }
                            if (st == 0 && gw == 0 && p.cancel && *p.cancel) {
                                atomicCAS(p.stop, 0, 2);
                                st = 2;
                            }
                            gb = (int)ld_volatile_u(&gs->best);
                            gd = (int)ld_volatile_u(&gs->done);
                            if (p.donate) idl = ld_volatile(p.idle);
                        }
                        st = __shfl_sync(kFull, st, 0);
                        gd = __shfl_sync(kFull, gd, 0);
                        if (st != 0) {
                            abort_all = true;
                            break;
                        }
                        if (gd != 0) break;
                        if (p.donate) {
                            gb = __shfl_sync(kFull, gb, 0);
                            idl = __shfl_sync(kFull, idl, 0);
                            best_eff = max(best_eff, gb);
                            if (idl > 0 && d > root) {
                                // donate the shallowest level with work left
                                int f = -1;
                                for (int b0 = root; b0 < d && f < 0; b0 += 32) {
                                    const int lv = b0 + lane;
                                    const bool has = lv < d && (s.f_cand[lv] != 0 || s.f_cont[lv] != 0);
                                    const unsigned m = __ballot_sync(kFull, has);
                                    if (m) f = b0 + __ffs(m) - 1;
                                }
                                if (f >= 0) {
                                    const W fc = s.f_cand[f];
                                    const int cnt = Bits<W>::popc(fc);
                                    W give = fc;
                                    for (int i = 0; i < (cnt + 1) / 2 && cnt >= 2; ++i) give &= give - 1;
                                    const W keep = fc & ~give;
                                    // reserve a slot
                                    int ok = 0;
                                    unsigned long long pos = 0;
                                    if (lane == 0) {
                                        for (;;) {
                                            pos = *reinterpret_cast<volatile unsigned long long*>(p.tail);
                                            TaskSlot* sl = p.slots + (pos & p.cap_mask);
                                            const unsigned long long seq = ld_acquire(&sl->seq);
                                            const long long dif = (long long)(seq - pos);
                                            if (dif == 0) {
                                                if (atomicCAS(p.tail, pos, pos + 1) == pos) {
                                                    ok = 1;
                                                    break;
                                                }
                                            } else if (dif < 0) {
                                                break;  // full
                                            }
                                        }
                                        if (ok) {
                                            atomicAdd(p.pending, 1);
                                            atomicAdd(&is->open_tasks, 1);
                                        }
                                    }
                                    ok = __shfl_sync(kFull, ok, 0);
                                    if (ok) {
                                        pos = __shfl_sync(kFull, pos, 0);
                                        TaskSlot* sl = p.slots + (pos & p.cap_mask);
                                        const int fnc = s.f_nc[f];
                                        const Cls<W>* FP = level(s.f_base[f]);
                                        for (int i = lane; i < fnc; i += 32) {
                                            Cls<W> c = FP[i];
                                            sl->cls_l[i] = uint64_t(c.l);
                                            sl->cls_r[i] = uint64_t(c.r);
                                        }
                                        for (int i = lane; i < f; i += 32) {
                                            sl->map_v[i] = s.map_v[i];
                                            sl->map_u[i] = s.map_u[i];
                                        }
                                        if (lane == 0) {
                                            TaskHeader h;
                                            h.inst = inst;
                                            h.kind = kTaskBranch;
                                            h.depth = uint8_t(f);
                                            h.nc = uint8_t(fnc);
                                            h.sel = s.f_sel[f];
                                            h.v = s.f_v[f];
                                            h.bound = s.f_bound[f];
                                            h.cont = s.f_cont[f];
                                            h.pad0 = 0;
                                            h.cand = uint64_t(give);
                                            h.pad1 = 0;
                                            sl->hdr = h;
                                            s.f_cand[f] = keep;
                                            s.f_cont[f] = 0;
                                        }
                                        __threadfence();
                                        __syncwarp();
                                        if (lane == 0) st_release(&sl->seq, pos + 1);
                                        ++donations;
                                    }
                                }
                            }
                        }
                    }
                    // inc.offer (search_core.hpp:145): strict improvement
                    if (d > (p.donate ? best_eff : best_local)) {
                        // store the mapping under the instance lock, then raise the size
                        int stored = 0;
                        if (lane == 0)
                            while (atomicCAS(&is->lock, 0, 1) != 0) __nanosleep(64);
                        __syncwarp();
                        if (lane == 0) {
                            __threadfence();
                            stored = ld_volatile_u(&is->map_size) < unsigned(d);
                        }
                        stored = __shfl_sync(kFull, stored, 0);
                        if (stored) {
                            for (int i = lane; i < d; i += 32) {
                                is->map_v[i] = s.map_v[i];
                                is->map_u[i] = s.map_u[i];
                            }
                            __threadfence();
                            __syncwarp();
                            if (lane == 0) {
                                is->map_size = unsigned(d);
                                __threadfence();
                                atomicMax(&gs->best, unsigned(d));
                            }
                        }
                        __syncwarp();
                        if (lane == 0) {
                            __threadfence();
                            atomicExch(&is->lock, 0);
                        }
                        best_local = d;
                        best_eff = max(best_eff, d);
                        if (goal > 0 && d >= goal) {  // search_core.hpp:147-150
                            if (lane == 0) {
                                gs->reached = 1;
                                if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                            }
                            break;
                        }
                        if (prune && goal == 0 && d >= maxp) {  // search_core.hpp:151-154
                            if (lane == 0 && atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                            break;
                        }
                    }
                    // prune (search_core.hpp:166)
                    if (prune && bound <= max(best_eff, goal - 1)) {
                        phase = 2;
                        continue;
                    }
                    Cls<W>* P = level(base);
                    if (!keyvalid) {
                        unsigned sum;
                        scan_level<W>(P, nc, lane, sum, key);
                    }
                    if (key == kNoKey) {
                        phase = 2;
                        continue;
                    }
                    sel = int(key & 127u);
                    const Cls<W> c = P[sel];
                    v = select_vertex<W>(c.l, s.vkey, lane);
                    cand = c.r;
                    cont = true;
                    phase = 1;
                } else if (phase == 1) {
                    // ------------------------------------------------- NEXT
                    if (cand != 0) {
                        const int u = Bits<W>::ctz(cand);
                        cand &= cand - 1;
                        if (lane == 0) {
                            s.f_cand[d] = cand;
                            s.f_base[d] = uint16_t(base);
                            s.f_nc[d] = uint8_t(nc);
                            s.f_sel[d] = uint8_t(sel);
                            s.f_v[d] = uint8_t(v);
                            s.f_bound[d] = uint8_t(bound);
                            s.f_cont[d] = uint8_t(cont);
                            s.map_v[d] = uint8_t(v);
                            s.map_u[d] = uint8_t(u);
                        }
                        int cb = base + nc;
                        const int need = min(nc * kParts, NB);
                        if (cb < cap && cb + need > cap) {
                            cb = cap;
                            ++spills;
                        }
                        if (cb + need > stack_limit) {  // cannot happen with the host's sizing
                            if (lane == 0) {
                                atomicAdd(&p.counters->overflow, 1ull);
                                atomicCAS(p.stop, 0, 3);
                            }
                            abort_all = true;
                            break;
                        }
                        const W vb = W(1) << v, ub = W(1) << u;
                        W ao, ai = 0, bo, bi = 0;
                        ao = s.out_g[v];
                        bo = s.out_h[u];
                        if constexpr (DIR) {
                            ai = s.in_g[v];
                            bi = s.in_h[u];
                        }
                        const SplitOut so = split_level<W, DIR>(level(base), nc, ~vb, ~ub, ao, ai, bo,
                                                                bi, level(cb), lane, lt);
                        __syncwarp();
                        ++splits;
                        split_cls += unsigned(nc);
                        ++d;
                        base = cb;
                        nc = so.nc;
                        bound = d + int(so.sum);
                        key = so.key;
                        keyvalid = true;
                        phase = 0;
                    } else if (cont) {
                        // v left unmatched (search_core.hpp:201-212): same level,
                        // v removed from the selected class, which drops if empty.
                        Cls<W>* P = level(base);
                        const Cls<W> c = P[sel];
                        const int pl = Bits<W>::popc(c.l), pr = Bits<W>::popc(c.r);
                        bound -= (pl <= pr) ? 1 : 0;
                        const W nl = c.l & ~(W(1) << v);
                        Cls<W> last = P[nc - 1];
                        __syncwarp();
                        if (lane == 0) {
                            if (nl != 0) P[sel].l = nl;
                            else P[sel] = last;
                        }
                        if (nl == 0) --nc;
                        __syncwarp();
                        keyvalid = false;
                        cont = false;
                        phase = 0;
                    } else {
                        phase = 2;
                    }
                } else {
                    // ----------------------------------------------- RETURN
                    if (d == root) break;
                    --d;
                    cand = s.f_cand[d];
                    base = s.f_base[d];
                    nc = s.f_nc[d];
                    sel = s.f_sel[d];
                    v = s.f_v[d];
                    bound = s.f_bound[d];
                    cont = s.f_cont[d] != 0;
                    phase = 1;
                }
            }
        }
        (void)n_g;
        nodes += task_nodes;
        // --------------------------------------------------- finish the task
        if (lane == 0) {
            if (task_nodes) atomicAdd(&is->nodes, task_nodes);
            if (!abort_all) {
                const int left = atomicSub(&is->open_tasks, 1) - 1;
                if (left == 0) {
                    is->t_done_ns = globaltimer();
                    if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                }
                __threadfence();
                atomicSub(p.pending, 1);
            }
        }
        if (abort_all) stop_all = true;
        __syncwarp();
    }

    if (lane == 0) {
        Counters* c = p.counters;
        atomicAdd(&c->nodes, nodes);
        atomicAdd(&c->sum_classes, sum_cls);
        atomicAdd(&c->splits, splits);
        atomicAdd(&c->split_classes, split_cls);
        atomicAdd(&c->donations, donations);
        atomicAdd(&c->tasks, tasks);
        atomicAdd(&c->spills, spills);
    }
}

// ------------------------------------------------------------ host launch --
template <typename W, bool DIR>
static cudaError_t launch_t(const KernelParams& p, int ctas, cudaStream_t st) {
    const int smem = warp_smem_bytes<W, DIR>(p.smem_classes) * kWarpsPerCta;
    cudaError_t e = cudaFuncSetAttribute(mcs_search_kernel<W, DIR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    mcs_search_kernel<W, DIR><<<ctas, kWarpsPerCta * 32, smem, st>>>(p);
    return cudaGetLastError();
}

template <typename W, bool DIR>
static int occupancy_t(int smem_classes) {
    const int smem = warp_smem_bytes<W, DIR>(smem_classes) * kWarpsPerCta;
    if (cudaFuncSetAttribute(mcs_search_kernel<W, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
        return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, mcs_search_kernel<W, DIR>,
                                                      kWarpsPerCta * 32, smem) != cudaSuccess)
        return 0;
    return blocks;
}

int kernel_smem_per_warp(bool wide, bool directed, int smem_classes) {
    if (wide) return directed ? warp_smem_bytes<uint64_t, true>(smem_classes)
                              : warp_smem_bytes<uint64_t, false>(smem_classes);
    return directed ? warp_smem_bytes<uint32_t, true>(smem_classes)
                    : warp_smem_bytes<uint32_t, false>(smem_classes);
}

int kernel_occupancy(bool wide, bool directed, int smem_classes) {
    if (wide) return directed ? occupancy_t<uint64_t, true>(smem_classes)
                              : occupancy_t<uint64_t, false>(smem_classes);
    return directed ? occupancy_t<uint32_t, true>(smem_classes)
                    : occupancy_t<uint32_t, false>(smem_classes);
}

cudaError_t kernel_launch(bool wide, bool directed, const KernelParams& p, int ctas,
                          cudaStream_t st) {
    if (wide) return directed ? launch_t<uint64_t, true>(p, ctas, st)
                              : launch_t<uint64_t, false>(p, ctas, st);
    return directed ? launch_t<uint32_t, true>(p, ctas, st) : launch_t<uint32_t, false>(p, ctas, st);
}

}  // namespace mcsg

namespace mcsg {

// Resets the ring (slot i of lap 0 expects producer ticket i) and the
// per-launch control words. One thread per slot.
__global__ void ring_reset_kernel(TaskSlot* slots, uint32_t cap, Counters* c) {
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

}  // namespace mcsg
