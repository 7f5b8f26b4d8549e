#pragma once
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

// 16-byte global -> shared copy that bypasses L1 (device-coherent values),
// completing in the background; used to prefetch control words.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned dst = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

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
// Byte-aligned fields: packing is a chain of IMADs, unpacking byte extracts.
//   low word : base (16 bits) | nc << 16 | sel << 24
//   high word: v | bound << 8 | cont << 16 | u << 24
constexpr unsigned long long kFrameCont = 1ull << 48;
__device__ __forceinline__ unsigned long long pack_frame(int base, int nc, int sel, int v, int bound,
                                                         int cont, int u) {
    const unsigned lo = unsigned(base) + (unsigned(nc) << 16) + (unsigned(sel) << 24);
    const unsigned hi = unsigned(v) + (unsigned(bound) << 8) + (unsigned(cont) << 16) + (unsigned(u) << 24);
    return (unsigned long long)lo | ((unsigned long long)hi << 32);
}
__device__ __forceinline__ int fr_base(unsigned long long f) { return int(unsigned(f) & 0xffffu); }
__device__ __forceinline__ int fr_nc(unsigned long long f) { return int(__byte_perm(unsigned(f), 0, 0x4442)); }
__device__ __forceinline__ int fr_sel(unsigned long long f) { return int(unsigned(f) >> 24); }
__device__ __forceinline__ int fr_v(unsigned long long f) { return int(unsigned(f >> 32) & 0xffu); }
__device__ __forceinline__ int fr_bound(unsigned long long f) { return int(__byte_perm(unsigned(f >> 32), 0, 0x4441)); }
__device__ __forceinline__ int fr_cont(unsigned long long f) { return int(__byte_perm(unsigned(f >> 32), 0, 0x4442)); }
__device__ __forceinline__ int fr_u(unsigned long long f) { return int(unsigned(f >> 32) >> 24); }

// Per-warp shared-memory image; the class stack follows it.
template <typename W, bool DIR>
struct WarpSmem {
    static constexpr int NB = Bits<W>::n;
    W out_g[NB];
    W out_h[NB];
    W in_g[DIR ? NB : 1];
    W in_h[DIR ? NB : 1];
    unsigned long long f_word[kMaxDepth + 1];
    // Control words prefetched one poll ahead with cp.async (16 B each):
    // [0..3] the stop line, [4..7] ring head, [8..11] ring tail, [12..15] GroupState,
    // [16..19] the first 16 B of the task's InstanceState (workers at [19]),
    // [20..23] the live-instance line.
    alignas(16) uint32_t pf[24];
    // per-warp counters kept out of registers (written by lane 0)
    unsigned long long polled;     // nodes of the current task counted at earlier polls
    unsigned long long st_nodes, st_splits, st_donations, st_tasks, st_spills;
    unsigned long long st_idle, st_busy;  // clock64 cycles waiting for / running tasks
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
    int rs[S];      // |R| minus 1 on the selected class (u leaves exactly that class)
    bool two = false;  // 64-bit kernel: the level has classes in the second slot (nc > 32)

    // slot k holds live classes (slot 0 always; slot 1 only when nc > 32)
    __device__ __forceinline__ bool live(int k) const { return k == 0 || two; }

    // The 32-bit kernel never spills: the host sizes its shared stack to the
    // path bound m(m+1)/2. The 64-bit kernel keeps levels past `cap` in HBM;
    // a level lies entirely on one side, and the hot accessors branch on it
    // so that the shared-memory case compiles to LDS/STS (not generic LD/ST).
    static constexpr bool kSpill = sizeof(W) == 8;

    __device__ __forceinline__ bool in_smem(int base) const { return !kSpill || base < cap; }

    // generic pointer, for the rare paths (donation, continuation write-back)
    __device__ __forceinline__ Cls<W>* at(int base) const {
        return in_smem(base) ? scls + base : gcls + (base - cap);
    }

    template <typename Ptr>
    __device__ __forceinline__ void load_from(const Ptr* p, int nc) {
        two = S > 1 && nc > 32;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int c = lane + 32 * k;
            Cls<W> x{0, 0};
            if (c < nc) x = p[c];
            L[k] = x.l;
            R[k] = x.r;
        }
    }

    __device__ __forceinline__ void load_level(int base, int nc) {
        if (in_smem(base)) load_from(scls + base, nc);
        else load_from(gcls + (base - cap), nc);
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
    __device__ __forceinline__ void prep_v(int v, int sel) {
        W g[P];
        g_parts(v, g);
        const W vb = W(1) << v;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            LX[k] = L[k] & ~vb;
            if (!live(k)) {
#pragma unroll
                for (int q = 0; q < P; ++q) lc[k][q] = 0;
                rs[k] = 0;
                continue;
            }
            rs[k] = Bits<W>::popc(R[k]) - (lane + 32 * k == sel ? 1 : 0);
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
    // u is in no adjacency row of its own, so it only ever sits in part 0 of
    // the selected class: |R\{u} ∩ part_q| = |R ∩ part_q| for q > 0, and part
    // 0 follows from rs = |R| - [selected] by subtraction (no per-u masking).
    __device__ __forceinline__ unsigned child_sum(int u, const W h[P]) const {
        (void)u;
        unsigned sm = 0;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            if (!live(k)) continue;
            if constexpr (!DIR) {
                const int b = Bits<W>::popc(R[k] & h[1]);
                sm += unsigned(min(lc[k][0], rs[k] - b) + min(lc[k][1], b));
            } else {
                int rest = rs[k];
#pragma unroll
                for (int q = 1; q < P; ++q) {
                    const int b = Bits<W>::popc(R[k] & h[q]);
                    rest -= b;
                    sm += unsigned(min(lc[k][q], b));
                }
                sm += unsigned(min(lc[k][0], rest));
            }
        }
        return __reduce_add_sync(kFull, sm);
    }

    // filter_classes (label_classes.cpp:80-108): split every class by the
    // codes toward (v,u), drop one-sided parts, compact into the next level
    // with ballots; returns the child's class count and its best class key.
    __device__ __forceinline__ int split(int u, int v, const W h[P], int cbase, unsigned* key_out) {
        if (in_smem(cbase)) return split_into(u, v, h, scls + cbase, key_out);
        return split_into(u, v, h, gcls + (cbase - cap), key_out);
    }

    __device__ __forceinline__ int split_into(int u, int v, const W h[P], Cls<W>* q, unsigned* key_out) {
        W g[P];
        g_parts(v, g);
        const W ub = W(1) << u;
        int total = 0;
        unsigned key = kNoKey;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            if (!live(k)) continue;
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

}  // namespace mcsg
