// McSplit branch-and-bound on sm_100a.
//
// One warp owns one DFS; lane c holds label class c of the current search
// level in registers (class = pair of vertex bitsets L ⊆ V_G, R ⊆ V_H); the
// levels of the current path live in a per-warp shared-memory stack (64-bit
// kernel: spills to HBM past the shared-memory capacity); subtrees move
// between warps through a lock-free ring in HBM.
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
// Per u candidate the child's bound is computed first from the parent's
// register-resident classes (one popcount pass + one warp reduction); the
// child is only materialised (split + compaction into the next stack level)
// when it survives the prune test. The child is still a counted node either
// way, in the reference's order, so with donation off ("parity mode") the
// kernel reproduces solve()'s node count and mapping exactly.
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
    static constexpr int slots = 1;
    __device__ static __forceinline__ int popc(uint32_t x) { return __popc(x); }
    __device__ static __forceinline__ int ctz(uint32_t x) { return __ffs(x) - 1; }
};
template <>
struct Bits<uint64_t> {
    static constexpr int n = 64;
    static constexpr int slots = 2;
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

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
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
    const unsigned mx = max(pl, pr), mn = min(pl, pr);
    return (mx << 20) | (mn << 13) | (unsigned(Bits<W>::ctz(l)) << 7) | unsigned(slot);
}

// Packed DFS frame (one per search level): where the level's classes are,
// which class/vertex it branches on, its bound, whether the v-unmatched
// continuation is still owned, and the u of the child being explored.
__device__ __forceinline__ unsigned long long pack_frame(int base, int nc, int sel, int v, int bound,
                                                         int cont, int u) {
    return (unsigned long long)base | ((unsigned long long)nc << 14) |
           ((unsigned long long)sel << 21) | ((unsigned long long)v << 28) |
           ((unsigned long long)bound << 34) | ((unsigned long long)cont << 41) |
           ((unsigned long long)u << 42);
}
__device__ __forceinline__ int fr_base(unsigned long long f) { return int(f & 0x3fff); }
__device__ __forceinline__ int fr_nc(unsigned long long f) { return int((f >> 14) & 0x7f); }
__device__ __forceinline__ int fr_sel(unsigned long long f) { return int((f >> 21) & 0x7f); }
__device__ __forceinline__ int fr_v(unsigned long long f) { return int((f >> 28) & 0x3f); }
__device__ __forceinline__ int fr_bound(unsigned long long f) { return int((f >> 34) & 0x7f); }
__device__ __forceinline__ int fr_cont(unsigned long long f) { return int((f >> 41) & 1); }
__device__ __forceinline__ int fr_u(unsigned long long f) { return int((f >> 42) & 0x3f); }

// Per-warp shared-memory image; the class stack follows it.
template <typename W, bool DIR>
struct WarpSmem {
    static constexpr int NB = Bits<W>::n;
    W out_g[NB];
    W out_h[NB];
    W in_g[DIR ? NB : 1];
    W in_h[DIR ? NB : 1];
    unsigned long long f_word[kMaxDepth + 1];
    W f_cand[kMaxDepth + 1];
    uint16_t vkey[NB];
    uint8_t map_v[kMaxDepth + 1];  // mapping prefix below the task's root level
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

// The per-warp search state held in registers plus its views of memory.
template <typename W, bool DIR>
struct Search {
    static constexpr int S = Bits<W>::slots;
    static constexpr int NB = Bits<W>::n;
    static constexpr int P = DIR ? 4 : 2;  // split parts (codes 0..3 / 0..1)

    WarpSmem<W, DIR>& s;
    Cls<W>* scls;   // shared-memory class stack
    Cls<W>* gcls;   // HBM spill area (64-bit kernel)
    int cap;
    int lane;
    unsigned lt;

    // class (lane + 32*k) of the current level
    W L[S], R[S];
    W LX[S];        // L with the branching vertex v removed
    int lc[S][P];   // |LX ∩ part_q(v)|

    __device__ __forceinline__ Cls<W>* at(int base) const {
        return base < cap ? scls + base : gcls + (base - cap);
    }

    __device__ __forceinline__ void load_level(int base, int nc) {
        const Cls<W>* p = at(base);
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int c = lane + 32 * k;
            Cls<W> x{0, 0};
            if (c < nc) x = p[c];
            L[k] = x.l;
            R[k] = x.r;
        }
    }

    // compute_bound + select_label_class over the register-resident level
    __device__ __forceinline__ unsigned scan_key(int nc, unsigned* sum) const {
        unsigned key = kNoKey, sm = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int c = lane + 32 * k;
            if (c < nc) {
                const int pl = Bits<W>::popc(L[k]), pr = Bits<W>::popc(R[k]);
                sm += unsigned(min(pl, pr));
                key = min(key, class_key<W>(pl, pr, L[k], c));
            }
        }
        if (sum) *sum = __reduce_add_sync(kFull, sm);
        return __reduce_min_sync(kFull, key);
    }

    // select_vertex (label_classes.cpp:69-78): max degree, lowest id on ties
    __device__ __forceinline__ int select_vertex(W lsel) const {
        unsigned k = kNoKey;
#pragma unroll
        for (int b = 0; b < S; ++b) {
            const int xb = lane + 32 * b;
            if ((lsel >> xb) & 1) k = min(k, unsigned(s.vkey[xb]));
        }
        return int(__reduce_min_sync(kFull, k) & 63u);
    }

    __device__ __forceinline__ W class_l(int c) const {
        if constexpr (S == 1) {
            return __shfl_sync(kFull, L[0], c);
        } else {
            const W a = __shfl_sync(kFull, L[0], c & 31), b = __shfl_sync(kFull, L[1], c & 31);
            return c < 32 ? a : b;
        }
    }
    __device__ __forceinline__ W class_r(int c) const {
        if constexpr (S == 1) {
            return __shfl_sync(kFull, R[0], c);
        } else {
            const W a = __shfl_sync(kFull, R[0], c & 31), b = __shfl_sync(kFull, R[1], c & 31);
            return c < 32 ? a : b;
        }
    }

    __device__ __forceinline__ void g_parts(int v, W g[P]) const {
        const W ao = s.out_g[v];
        if constexpr (!DIR) {
            g[0] = ~ao;
            g[1] = ao;
        } else {
            const W ai = s.in_g[v];
            g[0] = ~(ao | ai);
            g[1] = ao & ~ai;
            g[2] = ai & ~ao;
            g[3] = ao & ai;
        }
    }
    __device__ __forceinline__ void h_parts(int u, W h[P]) const {
        const W bo = s.out_h[u];
        if constexpr (!DIR) {
            h[0] = ~bo;
            h[1] = bo;
        } else {
            const W bi = s.in_h[u];
            h[0] = ~(bo | bi);
            h[1] = bo & ~bi;
            h[2] = bi & ~bo;
            h[3] = bo & bi;
        }
    }

    // After choosing v: LX = L \ {v}, and the per-part left counts.
    __device__ __forceinline__ void prep_v(int v) {
        W g[P];
        g_parts(v, g);
        const W vb = W(1) << v;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            LX[k] = L[k] & ~vb;
            if constexpr (!DIR) {
                const int a = Bits<W>::popc(LX[k] & g[1]);
                lc[k][1] = a;
                lc[k][0] = Bits<W>::popc(LX[k]) - a;
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q) lc[k][q] = Bits<W>::popc(LX[k] & g[q]);
            }
        }
    }

    // Bound of the child (v,u) minus |M|+1: Σ_c Σ_parts min(|L_part|, |R_part|).
    __device__ __forceinline__ unsigned child_sum(int u, const W h[P]) const {
        const W ub = W(1) << u;
        unsigned sm = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const W rx = R[k] & ~ub;
            if constexpr (!DIR) {
                const int b = Bits<W>::popc(rx & h[1]);
                const int r0 = Bits<W>::popc(rx) - b;
                sm += unsigned(min(lc[k][0], r0) + min(lc[k][1], b));
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q) sm += unsigned(min(lc[k][q], Bits<W>::popc(rx & h[q])));
            }
        }
        return __reduce_add_sync(kFull, sm);
    }

    // filter_classes (label_classes.cpp:80-108): split every class by the
    // codes toward (v,u), drop one-sided parts, compact into the next level
    // with ballots; returns the child's class count and its best class key.
    __device__ __forceinline__ int split(int u, int v, const W h[P], int cbase, unsigned* key_out) {
        W g[P];
        g_parts(v, g);
        const W ub = W(1) << u;
        Cls<W>* q = at(cbase);
        int total = 0;
        unsigned key = kNoKey;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const W rx = R[k] & ~ub;
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                const W lp = LX[k] & g[pp], rp = rx & h[pp];
                const bool keep = (lp != 0) & (rp != 0);
                const unsigned m = __ballot_sync(kFull, keep);
                if (keep) {
                    const int pos = total + __popc(m & lt);
                    q[pos] = Cls<W>{lp, rp};
                    key = min(key, class_key<W>(lc[k][pp], Bits<W>::popc(rp), lp, pos));
                }
                total += __popc(m);
            }
        }
        *key_out = __reduce_min_sync(kFull, key);
        return total;
    }
};

template <typename W, bool DIR>
__global__ void __launch_bounds__(kWarpsPerCta * 32, (sizeof(W) == 4 ? 8 : 5))
    mcs_search_kernel(KernelParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using Sm = WarpSmem<W, DIR>;
    using X = Search<W, DIR>;
    constexpr int NB = Bits<W>::n;
    constexpr int S = Bits<W>::slots;
    constexpr int P = X::P;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerCta + wib;
    const int per_warp = warp_smem_bytes<W, DIR>(p.smem_classes);
    Sm& s = *reinterpret_cast<Sm*>(smem_raw + size_t(wib) * per_warp);
    X x{s,
        reinterpret_cast<Cls<W>*>(smem_raw + size_t(wib) * per_warp + warp_smem_fixed<W, DIR>()),
        reinterpret_cast<Cls<W>*>(p.spill) + size_t(gw) * p.spill_classes,
        p.smem_classes,
        lane,
        lanemask_lt(),
        {},
        {},
        {},
        {}};
    const int stack_limit = p.smem_classes + p.spill_classes;
    Ctl* const ctl = p.ctl;

    const unsigned long long t_warp0 = globaltimer();
    const unsigned long long deadline = p.budget_ns ? t_warp0 + p.budget_ns : 0ull;
    if (lane == 0) atomicMin(&p.counters->t_start_ns, t_warp0);

    unsigned long long nodes = 0, sum_cls = 0, splits = 0, split_cls = 0, donations = 0;
    unsigned long long tasks = 0, spills = 0;
    int cur_inst = -1;
    int maxp = 0, goal = 0, prune = 1, floor_sz = 0, grp = 0;
    bool stop_all = false;

    while (!stop_all) {
        // ---------------------------------------------------------- acquire
        int inst = -1;
        bool branch = false;
        unsigned long long slot_pos = 0;
        {
            bool got = false;
            bool registered_idle = false;
            unsigned backoff = 64;
            for (;;) {
                int r = p.n_inst;
                if (lane == 0 && ld_volatile(&ctl->next_root.v) < p.n_inst)
                    r = atomicAdd(&ctl->next_root.v, 1);
                r = __shfl_sync(kFull, r, 0);
                if (r < p.n_inst) {
                    inst = r;
                    got = true;
                    break;
                }
                int ok = 0;
                unsigned long long pos = 0;
                if (lane == 0) {
                    // cheap emptiness test before touching the ring
                    pos = ld_relaxed(&ctl->head.v);
                    if (ld_relaxed(&ctl->tail.v) != pos) {
                        for (int tries = 0; tries < 8; ++tries) {
                            TaskSlot* sl = p.slots + (pos & p.cap_mask);
                            const unsigned long long seq = ld_acquire(&sl->seq);
                            const long long dif = (long long)(seq - (pos + 1));
                            if (dif == 0) {
                                const unsigned long long prev = atomicCAS(&ctl->head.v, pos, pos + 1);
                                if (prev == pos) {
                                    ok = 1;
                                    break;
                                }
                                pos = prev;
                            } else if (dif < 0) {
                                break;  // not yet published / empty
                            } else {
                                pos = ld_relaxed(&ctl->head.v);
                            }
                        }
                    }
                }
                ok = __shfl_sync(kFull, ok, 0);
                if (ok) {
                    slot_pos = __shfl_sync(kFull, pos, 0);
                    got = true;
                    branch = true;
                    break;
                }
                int pend = 0, st = 0;
                if (lane == 0) {
                    if (!registered_idle) atomicAdd(&ctl->idle.v, 1);
                    pend = ld_volatile(&ctl->pending.v);
                    st = ld_volatile(&ctl->stop.v);
                }
                registered_idle = true;
                pend = __shfl_sync(kFull, pend, 0);
                st = __shfl_sync(kFull, st, 0);
                if (pend <= 0 || st != 0) break;
                __nanosleep(backoff + (gw & 63) * 8);
                if (backoff < 4096) backoff <<= 1;
            }
            if (registered_idle && lane == 0) atomicSub(&ctl->idle.v, 1);
            if (!got) break;
        }

        // ---------------------------------------------------- load the task
        TaskSlot* slot = nullptr;
        TaskHeader hdr{};
        if (branch) {
            slot = p.slots + (slot_pos & p.cap_mask);
            __syncwarp();
            hdr = slot->hdr;
            inst = hdr.inst;
        }
        if (inst != cur_inst) {
            const InstanceDesc& dsc = p.inst[inst];
            for (int i = lane; i < NB; i += 32) {
                s.out_g[i] = W(dsc.out_g[i]);
                s.out_h[i] = W(dsc.out_h[i]);
                if constexpr (DIR) {
                    s.in_g[i] = W(dsc.in_g[i]);
                    s.in_h[i] = W(dsc.in_h[i]);
                }
                s.vkey[i] = dsc.vkey[i];
            }
            maxp = dsc.maxp;
            goal = dsc.goal;
            prune = dsc.prune;
            floor_sz = dsc.floor;
            grp = dsc.group;
            cur_inst = inst;
        }
        GroupState* const gs = p.grp + grp;
        InstanceState* const is = p.ist + inst;
        ++tasks;

        // Best sizes: best_local backs offers (LocalIncumbent::offer compares
        // with its own mapping only, search_core.hpp:29-31); best_eff adds the
        // external floor and, when sharing, the group incumbent (size()).
        int best_local = 0, best_eff = floor_sz;
        bool skip = false;
        {
            int gb = 0, gd = 0;
            if (lane == 0) {
                gb = int(ld_volatile_u(&gs->best));
                gd = int(ld_volatile_u(&gs->done));
            }
            gb = __shfl_sync(kFull, gb, 0);
            gd = __shfl_sync(kFull, gd, 0);
            if (p.donate) best_eff = max(best_eff, gb);
            skip = gd != 0;
        }

        int d, root, base = 0, nc, bound, sel = 0, v = 0;
        W cand = 0;
        int cont = 0;
        unsigned key = kNoKey;
        bool have_key = false;
        bool at_next = false;  // true: resume the u loop of the current level
        if (!branch) {
            const InstanceDesc& dsc = p.inst[inst];
            nc = dsc.n_init;
            for (int i = lane; i < nc; i += 32) x.scls[i] = Cls<W>{W(dsc.init_l[i]), W(dsc.init_r[i])};
            __syncwarp();
            d = root = 0;
            x.load_level(0, nc);
            unsigned sm;
            key = x.scan_key(nc, &sm);
            have_key = true;
            bound = int(sm);
        } else {
            d = root = hdr.depth;
            nc = hdr.nc;
            for (int i = lane; i < nc; i += 32) x.scls[i] = Cls<W>{W(slot->cls_l[i]), W(slot->cls_r[i])};
            for (int i = lane; i < d; i += 32) {
                s.map_v[i] = slot->map_v[i];
                s.map_u[i] = slot->map_u[i];
            }
            sel = hdr.sel;
            v = hdr.v;
            bound = hdr.bound;
            cand = W(hdr.cand);
            cont = hdr.cont;
            __syncwarp();
            if (lane == 0) st_release(&slot->seq, slot_pos + p.cap_mask + 1);  // free the slot
            x.load_level(0, nc);
            x.prep_v(v);
            at_next = true;
            // task-level prune (engine_parallel.cpp:148-155): every child would prune
            if (p.donate && prune && bound <= max(best_eff, goal - 1)) skip = true;
        }

        unsigned long long task_nodes = 0, next_poll = p.poll_interval;
        bool abort_all = false;

        // Writes M ∪ {(v,u)} (|M| = dd) as the instance's mapping if it is
        // still an improvement there; raises the group size afterwards.
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
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                atomicExch(&is->lock, 0);
            }
        };

        // Periodic poll: stop/deadline/cancel, group done, shared incumbent,
        // and subtree donation to idle warps. Returns false to end the task.
        auto poll = [&]() -> bool {
            int st = 0, gb = 0, gd = 0, idl = 0;
            if (lane == 0) {
                st = ld_volatile(&ctl->stop.v);
                if (st == 0 && deadline && globaltimer() >= deadline) {
                    atomicCAS(&ctl->stop.v, 0, 1);
                    st = 1;
                }
                if (st == 0 && gw == 0 && p.cancel && *p.cancel) {
                    atomicCAS(&ctl->stop.v, 0, 2);
                    st = 2;
                }
                gb = int(ld_volatile_u(&gs->best));
                gd = int(ld_volatile_u(&gs->done));
                if (p.donate) idl = ld_volatile(&ctl->idle.v);
            }
            st = __shfl_sync(kFull, st, 0);
            gd = __shfl_sync(kFull, gd, 0);
            if (st != 0) {
                abort_all = true;
                return false;
            }
            if (gd != 0) return false;
            if (!p.donate) return true;
            gb = __shfl_sync(kFull, gb, 0);
            idl = __shfl_sync(kFull, idl, 0);
            best_eff = max(best_eff, gb);
            if (idl <= 0 || d <= root) return true;
            // donate the shallowest level that still owns work
            int f = -1;
            for (int b0 = root; b0 < d && f < 0; b0 += 32) {
                const int lv = b0 + lane;
                bool has = false;
                if (lv < d) has = s.f_cand[lv] != 0 || fr_cont(s.f_word[lv]);
                const unsigned m = __ballot_sync(kFull, has);
                if (m) f = b0 + __ffs(m) - 1;
            }
            if (f < 0) return true;
            const W fc = s.f_cand[f];
            const unsigned long long fw = s.f_word[f];
            const int cnt = Bits<W>::popc(fc);
            W give = fc;
            if (cnt >= 2)
                for (int i = 0; i < (cnt + 1) / 2; ++i) give &= give - 1;  // upper half
            const W keep = fc & ~give;
            int ok = 0;
            unsigned long long pos = 0;
            if (lane == 0) {
                for (int tries = 0; tries < 16; ++tries) {
                    pos = ld_relaxed(&ctl->tail.v);
                    TaskSlot* sl = p.slots + (pos & p.cap_mask);
                    const unsigned long long seq = ld_acquire(&sl->seq);
                    const long long dif = (long long)(seq - pos);
                    if (dif == 0) {
                        if (atomicCAS(&ctl->tail.v, pos, pos + 1) == pos) {
                            ok = 1;
                            break;
                        }
                    } else if (dif < 0) {
                        break;  // full
                    }
                }
                if (ok) {
                    atomicAdd(&ctl->pending.v, 1);
                    atomicAdd(&is->open_tasks, 1);
                }
            }
            ok = __shfl_sync(kFull, ok, 0);
            if (!ok) return true;
            pos = __shfl_sync(kFull, pos, 0);
            TaskSlot* sl = p.slots + (pos & p.cap_mask);
            const int fnc = fr_nc(fw);
            const Cls<W>* fp = x.at(fr_base(fw));
            for (int i = lane; i < fnc; i += 32) {
                const Cls<W> c = fp[i];
                sl->cls_l[i] = uint64_t(c.l);
                sl->cls_r[i] = uint64_t(c.r);
            }
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
                h.pad0 = 0;
                h.cand = uint64_t(give);
                h.pad1 = 0;
                sl->hdr = h;
                s.f_cand[f] = keep;
                s.f_word[f] = fw & ~(1ull << 41);  // the continuation left with the task
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release(&sl->seq, pos + 1);
            ++donations;
            return true;
        };

        if (!skip) {
            if (!at_next) {
                // the root node (search_core.hpp:129-166)
                ++task_nodes;
                sum_cls += unsigned(nc);
                if (prune && bound <= max(best_eff, goal - 1)) goto pop;
                goto select;
            }
            goto next;

        select:
            // ---- the node survived its prune test: choose class and vertex
            if (!have_key) key = x.scan_key(nc, nullptr);
            if (key == kNoKey) goto pop;
            sel = int(key & 127u);
            {
                const W lsel = x.class_l(sel);
                v = x.select_vertex(lsel);
                cand = x.class_r(sel);
            }
            x.prep_v(v);
            cont = 1;

        next:
            // ---- u loop (search_core.hpp:183-200): children in ascending u
            while (cand != 0) {
                const int u = Bits<W>::ctz(cand);
                cand &= cand - 1;
                ++task_nodes;  // the child's entry (search_core.hpp:130)
                if (d + 1 > (p.donate ? best_eff : best_local)) {
                    offer(d, u);
                    best_local = d + 1;
                    best_eff = max(best_eff, d + 1);
                    if (goal > 0 && d + 1 >= goal) {  // search_core.hpp:147-150
                        if (lane == 0) {
                            gs->reached = 1;
                            if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                        }
                        goto finish;
                    }
                    if (prune && goal == 0 && d + 1 >= maxp) {  // search_core.hpp:151-154
                        if (lane == 0 && atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                        goto finish;
                    }
                }
                if (task_nodes >= next_poll) {
                    next_poll = task_nodes + p.poll_interval;
                    if (!poll()) goto finish;
                }
                W h[P];
                x.h_parts(u, h);
                const int cbound = d + 1 + int(x.child_sum(u, h));
                if (prune && cbound <= max(best_eff, goal - 1)) continue;  // pruned child
                // ---- materialise the child (filter_classes) one level up
                int cb = base + nc;
                const int need = min(nc * P, NB);
                if (cb < x.cap && cb + need > x.cap) {
                    cb = x.cap;
                    ++spills;
                }
                if (cb + need > stack_limit) {  // cannot happen with the host's sizing
                    if (lane == 0) {
                        atomicAdd(&p.counters->overflow, 1ull);
                        atomicCAS(&ctl->stop.v, 0, 3);
                    }
                    abort_all = true;
                    goto finish;
                }
                if (lane == 0) {
                    s.f_cand[d] = cand;
                    s.f_word[d] = pack_frame(base, nc, sel, v, bound, cont, u);
                }
                unsigned ckey;
                const int cnc = x.split(u, v, h, cb, &ckey);
                __syncwarp();
                ++splits;
                split_cls += unsigned(nc);
                ++d;
                base = cb;
                nc = cnc;
                bound = cbound;
                sum_cls += unsigned(nc);
                x.load_level(base, nc);
                key = ckey;
                have_key = true;
                goto select;
            }
            // ---- v left unmatched (search_core.hpp:201-212): a counted node
            if (cont) {
                ++task_nodes;
                if (task_nodes >= next_poll) {
                    next_poll = task_nodes + p.poll_interval;
                    if (!poll()) goto finish;
                }
                const W lsel = x.class_l(sel), rsel = x.class_r(sel);
                bound -= (Bits<W>::popc(lsel) <= Bits<W>::popc(rsel)) ? 1 : 0;
                const W nl = lsel & ~(W(1) << v);
                Cls<W>* lvl = x.at(base);
                if (nl != 0) {
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        if (lane + 32 * k == sel) x.L[k] = nl;
                    if (lane == 0) lvl[sel].l = nl;
                } else {
                    // drop the emptied class: the last class takes its slot
                    const W ll = x.class_l(nc - 1), lr = x.class_r(nc - 1);
#pragma unroll
                    for (int k = 0; k < S; ++k) {
                        const int c = lane + 32 * k;
                        if (c == nc - 1) {  // lanes past the level must hold empty classes
                            x.L[k] = 0;
                            x.R[k] = 0;
                        }
                        if (c == sel && sel != nc - 1) {
                            x.L[k] = ll;
                            x.R[k] = lr;
                        }
                    }
                    if (lane == 0 && sel != nc - 1) lvl[sel] = Cls<W>{ll, lr};
                    --nc;
                }
                __syncwarp();
                cont = 0;
                sum_cls += unsigned(nc);
                have_key = false;
                if (prune && bound <= max(best_eff, goal - 1)) goto pop;
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
            x.prep_v(v);
            goto next;
        }
    finish:
        nodes += task_nodes;
        if (lane == 0) {
            if (task_nodes) atomicAdd(&is->nodes, task_nodes);
            if (!abort_all) {
                const int left = atomicSub(&is->open_tasks, 1) - 1;
                if (left == 0) {
                    is->t_done_ns = globaltimer();
                    if (atomicCAS(&gs->done, 0u, 1u) == 0u) gs->winner = inst;
                }
                __threadfence();
                atomicSub(&ctl->pending.v, 1);
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
    (void)S;
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

// Resets the ring (slot i of lap 0 expects producer ticket i) and the
// per-launch counters. One thread per slot.
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
