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
#include <type_traits>

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

// Bitset operations shared by the 32/64-bit kernels (one machine word) and
// the wide kernels (WSet: NW 64-bit words, vertex v = bit v%64 of word v/64).
template <int NW>
struct alignas(16) WSet {
    uint64_t w[NW];
};

template <typename W>
__device__ __forceinline__ bool set_any(W x) { return x != 0; }
template <typename W>
__device__ __forceinline__ int set_ctz(W x) { return Bits<W>::ctz(x); }
template <typename W>
__device__ __forceinline__ int set_popc(W x) { return Bits<W>::popc(x); }
template <typename W>
__device__ __forceinline__ W set_drop_lowest(W x) { return x & (x - 1); }
template <typename W>
__device__ __forceinline__ W set_andnot(W a, W b) { return a & ~b; }
// highest set bit (-1 when empty): one FLO, where the lowest costs BREV + FLO
// highest set bit (-1 when empty): one FLO, where the lowest costs BREV + FLO
__device__ __forceinline__ int set_top(uint32_t x) { return 31 - __clz(x); }
__device__ __forceinline__ int set_top(uint64_t x) { return 63 - __clzll(x); }
// the same through PTX bfind, which yields the position directly: the 31 - clz
// form costs a subtract ptxas does not fold into the address and shift that
// use it (C2 +2.7%). Used by the 32-bit kernel only: the same change in the
// 64-bit kernel's compacted subtrees slows the directed C3 launch by 6%
// (instruction-fetch bound).
__device__ __forceinline__ int set_top_bf(uint32_t x) {
    unsigned r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return int(r);
}
template <typename W>
__device__ __forceinline__ W set_without(W x, int b) { return x & ~(W(1) << b); }

template <int NW>
__device__ __forceinline__ bool set_any(const WSet<NW>& x) {
    uint64_t o = x.w[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) o |= x.w[i];
    return o != 0;
}
template <int NW>
__device__ __forceinline__ int set_popc(const WSet<NW>& x) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) c += __popcll(x.w[i]);
    return c;
}
// lowest set bit (-1 when empty)
template <int NW>
__device__ __forceinline__ int set_ctz(const WSet<NW>& x) {
    int r = -1;
#pragma unroll
    for (int i = NW - 1; i >= 0; --i)
        if (x.w[i]) r = 64 * i + __ffsll(x.w[i]) - 1;
    return r;
}
template <int NW>
__device__ __forceinline__ int set_top(const WSet<NW>& x) {
    int r = -1;
#pragma unroll
    for (int i = 0; i < NW; ++i)
        if (x.w[i]) r = 64 * i + 63 - __clzll(x.w[i]);
    return r;
}
template <int NW>
__device__ __forceinline__ WSet<NW> set_drop_lowest(WSet<NW> x) {
    bool done = false;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        if (!done && x.w[i]) {
            x.w[i] &= x.w[i] - 1;
            done = true;
        }
    }
    return x;
}
template <int NW>
__device__ __forceinline__ WSet<NW> set_andnot(const WSet<NW>& a, const WSet<NW>& b) {
    WSet<NW> r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.w[i] = a.w[i] & ~b.w[i];
    return r;
}
template <int NW>
__device__ __forceinline__ WSet<NW> set_and(const WSet<NW>& a, const WSet<NW>& b) {
    WSet<NW> r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.w[i] = a.w[i] & b.w[i];
    return r;
}
template <int NW>
__device__ __forceinline__ WSet<NW> set_bit(int v) {
    WSet<NW> r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.w[i] = (v >> 6) == i ? (1ull << (v & 63)) : 0ull;
    return r;
}
template <int NW>
__device__ __forceinline__ WSet<NW> set_without(const WSet<NW>& x, int b) {
    return set_andnot(x, set_bit<NW>(b));
}

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
__device__ __forceinline__ int ld_volatile_i(const int32_t* p) {
    return *reinterpret_cast<const volatile int32_t*>(p);
}
__device__ __forceinline__ unsigned ld_volatile_u(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// select_label_class key (label_classes.cpp:47-67): min over classes of
// (max(|L|,|R|), min(|L|,|R|), lowest left id); low 7 bits carry the slot.
// TOP (throughput mode): the host relabels G in REVERSE select_vertex order,
// so "lowest left id" there is "highest left id" here: the tie field is the
// highest id flipped within its 6-bit field, and the min still picks that
// class. The fields are packed with multiply-adds (mx < 128, mn < 128,
// tie < 64, slot < 128).
template <typename W, bool TOP = false, bool BF = false>
__device__ __forceinline__ unsigned class_key(int pl, int pr, W l, int slot) {
    const unsigned mx = max(pl, pr), mn = min(pl, pr);
    int t;
    if constexpr (BF) t = set_top_bf(uint32_t(l));
    else t = set_top(l);
    const unsigned tie = TOP ? unsigned(t) ^ 63u : unsigned(Bits<W>::ctz(l));
    return ((mx * 128u + mn) * 64u + tie) * 128u + unsigned(slot);
}

// Packed DFS frame (one per search level): where the level's classes are,
// which class/vertex it branches on, its bound, whether the v-unmatched
// continuation is still owned, and the u of the child being explored.
// Byte-aligned fields: packing is a chain of IMADs, unpacking byte extracts.
//   low word : base (16 bits) | nc << 16 | sel << 24
//   high word: v | bound << 8 | cont << 16 | u << 24
// The continuation byte: 0 when the "v unmatched" continuation no longer
// belongs to the level, else kContOwned | (kContDec when |L*| <= |R*|, i.e.
// when the continuation lowers the bound by one).
constexpr int kContOwned = 1, kContDec = 2;
constexpr unsigned long long kFrameContByte = 0xffull << 48;
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

template <typename W, bool DIR>
struct WarpSmem;

// Per-task values the DFS only needs on cold paths (offers, polls,
// donations, the task's end), kept in shared memory (written by lane 0 at
// task start) so that they hold no registers across the hot loop.
struct TaskCold {
    GroupState* gs;
    InstanceState* is;
    int inst, cur_inst;
    int maxp, goal, prune, floor_sz, grp;
};

// The 64-bit kernel's area for a subtree compacted to 32 bits: a 32-bit
// search image (rows of the live vertices, renumbered 0..31) and the maps
// between compact and original ids.
struct NoCompactArea {};
template <bool DIR>
struct CompactRows {  // what the 32-bit policy reads through its `s`
    uint32_t out_g[32];
    uint32_t out_h[32];
    uint32_t in_g[DIR ? 32 : 1];
    uint32_t in_h[DIR ? 32 : 1];
    uint16_t vkey[32];  // (parity mode only; compaction runs in throughput mode)
};
template <bool DIR>
struct CompactArea {
    CompactRows<DIR> img;            // rows of the live vertices, renumbered
    uint8_t gid[32], hid[32];        // compact id -> original id
    // original -> compact ids: a parallel bit extract (PEXT) through the live
    // sets, by the shift-and-mask compress of Hacker's Delight §7-4 with its
    // five move masks per 32-bit half precomputed once per nest:
    // mv[0..1] = G low / high half, mv[2..3] = H low / high half
    alignas(16) uint32_t mv[4][8];
    uint64_t lg, lh;                 // the live sets
    unsigned long long nests_smem, nests_hbm;  // subtrees run compacted, by stack placement (nests_hbm: 0 since nests are shared-memory only)
};

// 64-bit kernel: a level of more than 32 classes keeps classes 32..63 (its
// second slot) in its stack copy, not in registers; the policy reads them
// through this (rare: classes are disjoint and non-empty on both sides, so
// more than 32 of them need more than 32 live vertices in G and in H — on
// C3/C4 (n = 40/45) only levels near the top), so the hot loop holds one
// class per lane.
template <typename W>
struct HiSlot {
    Cls<W>* lvl;  // the current level's classes (shared memory or the HBM spill area)
    int nc, v, sel;
};
struct NoHiSlot {};

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
    unsigned long long st_nodes, st_splits, st_split_cls, st_donations, st_tasks, st_spills;
    unsigned long long st_idle, st_busy;  // clock64 cycles waiting for / running tasks
    // cold per-warp values kept out of the hot loop's registers (lane 0)
    unsigned long long deadline;          // %globaltimer deadline (0 = none)
    long long t_mark;                     // clock64 at the last idle/busy switch
    TaskCold tc;
    W f_cand[kMaxDepth + 1];
    uint16_t vkey[NB];
    uint8_t map_v[kMaxDepth + 1];  // mapping prefix below the task's root level
    uint8_t map_u[kMaxDepth + 1];
    // 64-bit kernel only: a subtree compacted to 32 bits (CompactSearch)
    [[no_unique_address]] std::conditional_t<sizeof(W) == 8, CompactArea<DIR>, NoCompactArea> ca;
    [[no_unique_address]] std::conditional_t<sizeof(W) == 8, HiSlot<W>, NoHiSlot> hi;
};

// Per-warp shared memory of a search policy X: its fixed image, then the
// class stack.
template <class X>
__host__ __device__ constexpr int warp_smem_fixed() {
    return (int)((sizeof(typename X::Sm) + 15) & ~size_t(15));
}

template <class X>
__host__ __device__ constexpr int warp_smem_bytes(int classes) {
    return (warp_smem_fixed<X>() + classes * int(sizeof(Cls<typename X::Set>)) + 15) & ~15;
}

// The per-warp search state held in registers plus its views of memory.
//
// The kernel body (mcsg_kernel.cu) is written against this policy interface;
// WideSearch below implements the same interface for 64 < n <= 255.
template <typename W, bool DIR, class SmT = WarpSmem<W, DIR>>
struct Search {
    static constexpr int S = Bits<W>::slots;
    static constexpr int NB = Bits<W>::n;
    static constexpr int P = DIR ? 4 : 2;  // split parts (codes 0..3 / 0..1)
    // __launch_bounds__ CTAs/SM. The 32-bit kernel: 9 (56 registers, no
    // spill in the undirected kernels; 36 warps/SM: C2 +3.2%, C5 +3% against
    // 8 at 64 registers; 10 at 48 registers spills: +0.7%). The 64-bit
    // kernels hold one class per lane in registers (a second slot lives in
    // the level's stack copy, HiSlot): the undirected one then fits 64
    // registers at 8 CTAs/SM with an 8-byte spill (C4 3.97 -> 3.62 s against
    // 7 CTAs at 72 registers); the directed one runs 7 (72 registers, 16 B
    // stack, more shared memory per warp for its compacted subtrees: C3
    // -0.9% time, +2% nodes/s against 8 at 64 registers with 48 B of spills)
    static constexpr int kMinBlocks = sizeof(W) == 4 ? 9 : (DIR ? 7 : 8);
    // 64-bit kernel: a level whose live vertex sets fit 32 bits runs its
    // subtree compacted (CompactSearch, nested in the task) — 97% of C4's nodes
    static constexpr bool kNest = sizeof(W) == 8;
    static constexpr bool kDir = DIR;
    using Set = W;
    using Sm = SmT;
    using Desc = InstanceDesc;
    using Slot = TaskSlot;
    struct HParts {
        W h[P];
    };

    Sm& s;
    Cls<W>* scls;   // shared-memory class stack
    Cls<W>* gcls;   // HBM spill area (64-bit kernel)
    int cap;
    int lane;
    unsigned lt;

    // class `lane` of the current level (classes 32..63 of a 64-bit level:
    // HiSlot, read from the level's stack copy)
    W L[1], R[1];
    W LX[1];        // L with the branching vertex v removed
    int lc[1][P];   // |LX ∩ part_q(v)|
    int rs[1];      // |R| minus 1 on the selected class (u leaves exactly that class)
    bool two = false;  // 64-bit kernel: the level has classes in the second slot (nc > 32)

    // the second slot's class of this lane (lane + 32), from the stack copy,
    // with its prep_v values (LX, per-part left counts, rs) recomputed
    struct HiCls {
        W lx, r;
        int lc[P];
        int rs;
    };
    __device__ __forceinline__ HiCls hi_cls(const W g[P]) const {
        HiCls o;
        const int c = lane + 32;
        Cls<W> x{0, 0};
        if (c < s.hi.nc) x = s.hi.lvl[c];
        o.lx = x.l & ~(W(1) << s.hi.v);
        o.r = x.r;
        o.rs = Bits<W>::popc(x.r) - (c == s.hi.sel ? 1 : 0);
        if constexpr (!DIR) {
            const int a = Bits<W>::popc(o.lx & g[1]);
            o.lc[1] = a;
            o.lc[0] = Bits<W>::popc(o.lx) - a;
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) o.lc[q] = Bits<W>::popc(o.lx & g[q]);
        }
        return o;
    }

    __device__ __forceinline__ Search(Sm& s_, Cls<W>* scls_, Cls<W>* gcls_, int cap_, int lane_, unsigned lt_)
        : s(s_), scls(scls_), gcls(gcls_), cap(cap_), lane(lane_), lt(lt_) {}

    __device__ static __forceinline__ const Desc* descs(const KernelParams& p) { return p.inst; }
    __device__ static __forceinline__ Slot* slots(const KernelParams& p) { return p.slots; }
    __device__ static __forceinline__ int key_slot(unsigned key) { return int(key & 127u); }
    // vertex-id hooks (identity: the 32-bit compacted policy maps ids) and
    // the class-stack limit of the level placement
    __device__ __forceinline__ int g_orig(int v) const { return v; }
    __device__ __forceinline__ int h_orig(int u) const { return u; }
    __device__ __forceinline__ int g_local(int v) const { return v; }
    __device__ __forceinline__ int stack_limit(const KernelParams& p) const { return p.smem_classes + p.spill_classes; }
    // the current level's live vertex sets (∪L, ∪R) fit 32 bits
    __device__ __forceinline__ bool level_live(int nc, uint64_t& lg, uint64_t& lh) const {
        if (nc > 32 || two) return false;
        const uint64_t l = uint64_t(L[0]), r = uint64_t(R[0]);
        lg = uint64_t(__reduce_or_sync(kFull, unsigned(l))) | (uint64_t(__reduce_or_sync(kFull, unsigned(l >> 32))) << 32);
        lh = uint64_t(__reduce_or_sync(kFull, unsigned(r))) | (uint64_t(__reduce_or_sync(kFull, unsigned(r >> 32))) << 32);
        return __popcll(lg) <= 32 && __popcll(lh) <= 32;
    }

    // adjacency rows (and the parity-mode vertex keys) of a new instance
    template <bool PAR>
    __device__ __forceinline__ void load_instance(const Desc& d) {
        for (int i = lane; i < NB; i += 32) {
            s.out_g[i] = W(d.out_g[i]);
            s.out_h[i] = W(d.out_h[i]);
            if constexpr (DIR) {
                s.in_g[i] = W(d.in_g[i]);
                s.in_h[i] = W(d.in_h[i]);
            }
            if constexpr (PAR) s.vkey[i] = d.vkey[i];
        }
    }
    // initial classes (label_classes.cpp:8-39) at stack position 0
    __device__ __forceinline__ void load_root(const Desc& d, int nc) {
        for (int i = lane; i < nc; i += 32) scls[i] = Cls<W>{W(d.init_l[i]), W(d.init_r[i])};
    }
    // a donated subtree: its classes at stack position 0, its mapping prefix
    __device__ __forceinline__ void load_task(const Slot& sl, int nc, int d) {
        for (int i = lane; i < nc; i += 32) scls[i] = Cls<W>{W(sl.cls_l[i]), W(sl.cls_r[i])};
        for (int i = lane; i < d; i += 32) {
            s.map_v[i] = sl.map_v[i];
            s.map_u[i] = sl.map_u[i];
        }
    }
    __device__ static __forceinline__ W slot_cand(const Slot& sl) { return W(sl.hdr.cand); }
    __device__ __forceinline__ void store_task(Slot& sl, int fbase, int fnc) const {
        const Cls<W>* fp = at(fbase);
        for (int i = lane; i < fnc; i += 32) {
            const Cls<W> c = fp[i];
            sl.cls_l[i] = uint64_t(c.l);
            sl.cls_r[i] = uint64_t(c.r);
        }
    }
    __device__ static __forceinline__ void put_cand(Slot&, TaskHeader& h, W give) { h.cand = uint64_t(give); }

    // The 32-bit kernel never spills: the host sizes its shared stack to the
    // path bound m(m+1)/2. The 64-bit kernel keeps levels past `cap` in HBM;
    // a level lies entirely on one side, and the hot accessors branch on it
    // so that the shared-memory case compiles to LDS/STS (not generic LD/ST).
    static constexpr bool kSpill = sizeof(W) == 8;
    // A 32-bit class stack provably cannot overflow: a level at depth k
    // holds at most m - k classes (disjoint non-empty L sides), so the host's
    // m(m+1)/2 + 64 entries (plan(), mcsg_host.cpp) bound every path of the
    // 32-bit kernel, and a compacted subtree only starts when its room holds
    // nc + s0(s0-1)/2 + 32 entries, s0 = min(m, the level's Σ min) (the nest
    // entry in mcsg_task_body.inc): the
    // split's overflow check is compiled out, and a level load may read up to
    // 31 entries past the level's start. The spilling kernels keep both checks.
    static constexpr bool kBoundedStack = sizeof(W) == 4;
    // cont_step updates the owner lane's registers; its shared-memory copy is
    // next read by another lane only after a warp barrier (the split's
    // __syncwarp before a child's level load, or the poll's before a
    // donation), so no barrier follows the step
    static constexpr bool kContSync = false;
    static constexpr bool kColdSmem = true;  // TaskCold in shared memory (mcsg_kernel.cu)
    // highest set bit of a vertex set (throughput mode's v and u walk)
    __device__ static __forceinline__ int top(W x) {
        if constexpr (sizeof(W) == 4) return set_top_bf(uint32_t(x));
        else {
            unsigned r;
            asm("bfind.u64 %0, %1;" : "=r"(r) : "l"(uint64_t(x)));
            return int(r);
        }
    }

    __device__ __forceinline__ bool in_smem(int base) const { return !kSpill || base < cap; }

    // generic pointer, for the rare paths (donation, continuation write-back)
    __device__ __forceinline__ Cls<W>* at(int base) const {
        return in_smem(base) ? scls + base : gcls + (base - cap);
    }

    template <typename Ptr>
    __device__ __forceinline__ void load_from(const Ptr* p, int nc) {
        two = S > 1 && nc > 32;
        if constexpr (kBoundedStack) {
            // 32-bit kernel: every lane loads (a level starts at most
            // m(m+1)/2 entries into a stack of m(m+1)/2 + 64, so slot 31 is
            // inside it) and lanes past nc zero their class: no branch
            const Cls<W> x = p[lane];
            L[0] = lane < nc ? x.l : W(0);
            R[0] = lane < nc ? x.r : W(0);
        } else {
            Cls<W> x{0, 0};
            if (lane < nc) x = p[lane];
            L[0] = x.l;
            R[0] = x.r;
            if constexpr (S > 1) {
                if (two) {  // (uniform stores)
                    s.hi.lvl = const_cast<Cls<W>*>(reinterpret_cast<const Cls<W>*>(p));
                    s.hi.nc = nc;
                }
            }
        }
    }

    __device__ __forceinline__ void load_level(int base, int nc) {
        if (in_smem(base)) load_from(scls + base, nc);
        else load_from(gcls + (base - cap), nc);
    }

    // compute_bound + select_label_class over the register-resident level
    template <bool TOP>
    __device__ __forceinline__ unsigned scan_key(int nc, unsigned* sum) const {
        unsigned key = kNoKey, sm = 0;
        if (lane < nc) {
            const int pl = Bits<W>::popc(L[0]), pr = Bits<W>::popc(R[0]);
            sm += unsigned(min(pl, pr));
            if (pl) key = min(key, class_key<W, TOP, sizeof(W) == 4>(pl, pr, L[0], lane));  // L = {}: a dead class
        }
        if constexpr (S > 1) {
            if (two) {
                const int c = lane + 32;
                if (c < nc) {
                    const Cls<W> x = s.hi.lvl[c];
                    const int pl = Bits<W>::popc(x.l), pr = Bits<W>::popc(x.r);
                    sm += unsigned(min(pl, pr));
                    if (pl) key = min(key, class_key<W, TOP, sizeof(W) == 4>(pl, pr, x.l, c));
                }
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

    // (c is warp-uniform)
    __device__ __forceinline__ W class_l(int c) const {
        if constexpr (S > 1) {
            if (c >= 32) return s.hi.lvl[c].l;
            return __shfl_sync(kFull, L[0], c & 31);
        }
        return __shfl_sync(kFull, L[0], c);
    }
    __device__ __forceinline__ W class_r(int c) const {
        if constexpr (S > 1) {
            if (c >= 32) return s.hi.lvl[c].r;
            return __shfl_sync(kFull, R[0], c & 31);
        }
        return __shfl_sync(kFull, R[0], c);
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
    __device__ __forceinline__ void h_parts(int u, HParts& hp) const {
        W* h = hp.h;
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
        LX[0] = L[0] & ~vb;
        rs[0] = Bits<W>::popc(R[0]) - (lane == sel ? 1 : 0);
        if constexpr (!DIR) {
            const int a = Bits<W>::popc(LX[0] & g[1]);
            lc[0][1] = a;
            lc[0][0] = Bits<W>::popc(LX[0]) - a;
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) lc[0][q] = Bits<W>::popc(LX[0] & g[q]);
        }
        if constexpr (S > 1) {
            if (two) {  // (uniform stores)
                s.hi.v = v;
                s.hi.sel = sel;
            }
        }
    }

    // Bound of the child (v,u) minus |M|+1: Σ_c Σ_parts min(|L_part|, |R_part|).
    // u is in no adjacency row of its own, so it only ever sits in part 0 of
    // the selected class: |R\{u} ∩ part_q| = |R ∩ part_q| for q > 0, and part
    // 0 follows from rs = |R| - [selected] by subtraction (no per-u masking).
    __device__ __forceinline__ unsigned child_sum(int u, const HParts& hp) const {
        (void)u;
        const W* h = hp.h;
        unsigned sm = part_sum(R[0], lc[0], rs[0], h);
        if constexpr (S > 1) {
            if (two) {
                W g[P];
                g_parts(s.hi.v, g);
                const HiCls x = hi_cls(g);
                sm += part_sum(x.r, x.lc, x.rs, h);
            }
        }
        return __reduce_add_sync(kFull, sm);
    }
    __device__ static __forceinline__ unsigned part_sum(W r, const int lcq[P], int rsq, const W* h) {
        unsigned sm = 0;
        if constexpr (!DIR) {
            const int b = Bits<W>::popc(r & h[1]);
            sm += unsigned(min(lcq[0], rsq - b) + min(lcq[1], b));
        } else {
            int rest = rsq;
#pragma unroll
            for (int q = 1; q < P; ++q) {
                const int b = Bits<W>::popc(r & h[q]);
                rest -= b;
                sm += unsigned(min(lcq[q], b));
            }
            sm += unsigned(min(lcq[0], rest));
        }
        return sm;
    }

    // filter_classes (label_classes.cpp:80-108): split every class by the
    // codes toward (v,u), drop one-sided parts, compact into the next level
    // with ballots; returns the child's class count and its best class key.
    template <bool TOP>
    __device__ __forceinline__ int split(int u, int v, const HParts& hp, int cbase, unsigned* key_out) {
        if (in_smem(cbase)) return split_into<TOP>(u, v, hp.h, scls + cbase, key_out);
        return split_into<TOP>(u, v, hp.h, gcls + (cbase - cap), key_out);
    }

    template <bool TOP>
    __device__ __forceinline__ int split_into(int u, int v, const W h[P], Cls<W>* q, unsigned* key_out) {
        W g[P];
        g_parts(v, g);
        const W ub = W(1) << u;
        int total = 0;
        unsigned key = kNoKey;
        split_parts<TOP>(LX[0], R[0] & ~ub, lc[0], g, h, q, total, key);
        if constexpr (S > 1) {
            if (two) {
                const HiCls x = hi_cls(g);
                split_parts<TOP>(x.lx, x.r & ~ub, x.lc, g, h, q, total, key);
            }
        }
        *key_out = __reduce_min_sync(kFull, key);
        return total;
    }
    template <bool TOP>
    __device__ __forceinline__ void split_parts(W lx, W rx, const int lcq[P], const W g[P], const W h[P], Cls<W>* q,
                                                int& total, unsigned& key) const {
#pragma unroll
        for (int pp = 0; pp < P; ++pp) {
            const W lp = lx & g[pp], rp = rx & h[pp];
            const bool keep = (lp != 0) & (rp != 0);
            const unsigned m = __ballot_sync(kFull, keep);
            // branch-free: every lane computes its slot and key, the kept
            // ones store (one predicated store, no reconvergence block)
            const int pos = total + __popc(m & lt);
            const unsigned ck = class_key<W, TOP, sizeof(W) == 4>(lcq[pp], Bits<W>::popc(rp), lp, pos);
            if (keep) q[pos] = Cls<W>{lp, rp};
            key = keep ? min(key, ck) : key;
            total += __popc(m);
        }
    }

    // "v unmatched" (search_core.hpp:201-212): the bound drops by
    // [|L*| <= |R*|] (decided at select: kContDec) and v leaves L*. The lane
    // owning class sel already holds L* \ {v} (LX, prep_v) and writes it to
    // the level's stack copy. A class emptied this way stays in its slot,
    // dead: it adds 0 to every bound and is never selected (scan_key), which
    // is what dropping it does (label_classes.cpp:95-105).
    __device__ __forceinline__ void cont_step(int sel, int cbits, int base, int& bound) {
        bound -= (cbits & kContDec) ? 1 : 0;
        Cls<W>* lvl = at(base);
        if (lane == sel) {
            L[0] = LX[0];
            lvl[sel].l = LX[0];
        }
        if constexpr (S > 1) {
            // second slot: its owner lane (the one that reads it back) writes
            if (lane + 32 == sel) lvl[sel].l &= ~(W(1) << s.hi.v);
        }
    }
};

// ------------------------------------------------------- compacted subtrees --
// The 64-bit kernel runs a subtree whose live vertex sets fit 32 bits with
// the 32-bit policy on renumbered vertices: compact id j is the j-th live
// vertex (ascending original id, so every selection rule, being an order on
// ids, picks the same vertex and class as the 64-bit policy would). Rows are
// rebuilt for the live vertices (CompactArea), the class stack is the 64-bit
// stack's free memory above the enclosing level, seen as 8-byte classes (at
// most nc + s0(s0-1)/2 + 32 of them for the enclosing level's nc entries,
// dead ones included, and s0 = min(|∪L|, |∪R|, Σ min(|L|,|R|)): a nested level
// k matches deep holds at most s0 - k classes), and ids are mapped back wherever
// they leave the subtree: offered mappings, donated subtrees (in the 64-bit
// format, so any warp can take them).
template <bool DIR>
struct CompactSearch : Search<uint32_t, DIR, CompactRows<DIR>> {
    using Base = Search<uint32_t, DIR, CompactRows<DIR>>;
    using Set = uint32_t;
    using Desc = InstanceDesc;
    using Slot = TaskSlot;
    using KSm = WarpSmem<uint64_t, DIR>;
    static constexpr bool kNest = false;

    KSm& ks;  // the kernel's (64-bit) per-warp memory: mapping prefix, maps

    __device__ __forceinline__ CompactSearch(KSm& ks_, Cls<uint32_t>* scls_, int cap_, int lane_, unsigned lt_)
        : Base(ks_.ca.img, scls_, nullptr, cap_, lane_, lt_), ks(ks_) {}

    __device__ __forceinline__ int g_orig(int v) const { return ks.ca.gid[v]; }
    __device__ __forceinline__ int h_orig(int u) const { return ks.ca.hid[u]; }
    __device__ __forceinline__ int g_local(int v) const { return __popcll(ks.ca.lg & ((1ull << v) - 1)); }
    __device__ __forceinline__ int stack_limit(const KernelParams&) const { return this->cap; }

    // compact image of x ⊆ the live set of side w (0 = G, 2 = H): PEXT
    // with the nest's move masks (3 instructions per step, 5 steps per half)
    __device__ __forceinline__ uint32_t pext(uint64_t x, int w) const {
        uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
        const uint4 a0 = *reinterpret_cast<const uint4*>(&ks.ca.mv[w][0]);
        const uint4 a1 = *reinterpret_cast<const uint4*>(&ks.ca.mv[w][4]);
        const uint4 b0 = *reinterpret_cast<const uint4*>(&ks.ca.mv[w + 1][0]);
        const uint4 b1 = *reinterpret_cast<const uint4*>(&ks.ca.mv[w + 1][4]);
        const uint32_t ma[5] = {a0.x, a0.y, a0.z, a0.w, a1.x};
        const uint32_t mb[5] = {b0.x, b0.y, b0.z, b0.w, b1.x};
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t t = lo & ma[i], u = hi & mb[i];
            lo = (lo ^ t) | (t >> (1 << i));
            hi = (hi ^ u) | (u >> (1 << i));
        }
        // a1.y = the live low half's size; the whole set has at most 32 bits
        return lo | uint32_t(uint64_t(hi) << a1.y);
    }

    // Builds the compact area for live sets lg (G) and lh (H) from the
    // instance's 64-bit rows in the kernel's shared memory. (Siblings
    // rarely share live sets: reusing the last area hit 2% of C4's nests.)
    __device__ __forceinline__ void build(uint64_t lg, uint64_t lh) {
        const int lane = this->lane;
        if (lane < 4) {  // the move masks of one 32-bit half per lane (HD §7-4)
            const uint64_t mm = lane < 2 ? lg : lh;
            uint32_t m = (lane & 1) ? uint32_t(mm >> 32) : uint32_t(mm);
            const uint32_t n0 = __popc(m);
            uint32_t mk = ~m << 1;
            uint32_t o[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                uint32_t mp = mk ^ (mk << 1);
                mp ^= mp << 2;
                mp ^= mp << 4;
                mp ^= mp << 8;
                mp ^= mp << 16;
                const uint32_t mvi = mp & m;
                o[i] = mvi;
                m = (m ^ mvi) | (mvi >> (1 << i));
                mk &= ~mp;
            }
            *reinterpret_cast<uint4*>(&ks.ca.mv[lane][0]) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint2*>(&ks.ca.mv[lane][4]) = make_uint2(o[4], n0);
        }
        if (lane == 4) {
            ks.ca.lg = lg;
            ks.ca.lh = lh;
        }
        for (int x = lane; x < 64; x += 32) {
            if ((lg >> x) & 1) ks.ca.gid[__popcll(lg & ((1ull << x) - 1))] = uint8_t(x);
            if ((lh >> x) & 1) ks.ca.hid[__popcll(lh & ((1ull << x) - 1))] = uint8_t(x);
        }
        __syncwarp();
        // lane j builds row j: bit k = code bit toward the k-th live vertex
        const int ng = __popcll(lg), nh = __popcll(lh);
        auto& img = ks.ca.img;
        uint32_t og = 0, oh = 0, ig = 0, ih = 0;
        if (lane < ng) {
            const int xg = ks.ca.gid[lane];
            og = pext(ks.out_g[xg] & lg, 0);
            if constexpr (DIR) ig = pext(ks.in_g[xg] & lg, 0);
        }
        if (lane < nh) {
            const int xh = ks.ca.hid[lane];
            oh = pext(ks.out_h[xh] & lh, 2);
            if constexpr (DIR) ih = pext(ks.in_h[xh] & lh, 2);
        }
        img.out_g[lane] = og;
        img.out_h[lane] = oh;
        if constexpr (DIR) {
            img.in_g[lane] = ig;
            img.in_h[lane] = ih;
        }
        __syncwarp();
    }

    __device__ __forceinline__ uint32_t pack_g(uint64_t x) const { return pext(x, 0); }
    __device__ __forceinline__ uint32_t pack_h(uint64_t x) const { return pext(x, 2); }
    __device__ __forceinline__ uint64_t unpack_g(uint32_t x) const {
        uint64_t r = 0;
        for (; x; x &= x - 1) r |= 1ull << ks.ca.gid[__ffs(x) - 1];
        return r;
    }
    __device__ __forceinline__ uint64_t unpack_h(uint32_t x) const {
        uint64_t r = 0;
        for (; x; x &= x - 1) r |= 1ull << ks.ca.hid[__ffs(x) - 1];
        return r;
    }

    // the enclosing 64-bit level (lane = class, registers) as the compact
    // stack's level 0
    __device__ __forceinline__ void put_level(uint64_t l, uint64_t r, int nc) {
        if (this->lane < nc) this->scls[this->lane] = Cls<uint32_t>{pack_g(l), pack_h(r)};
    }
    __device__ __forceinline__ void store_task(Slot& sl, int fbase, int fnc) const {
        const Cls<uint32_t>* fp = this->at(fbase);
        for (int i = this->lane; i < fnc; i += 32) {
            const Cls<uint32_t> c = fp[i];
            sl.cls_l[i] = unpack_g(c.l);
            sl.cls_r[i] = unpack_h(c.r);
        }
    }
    __device__ __forceinline__ void put_cand(Slot&, TaskHeader& h, uint32_t give) const { h.cand = unpack_h(give); }
};

// ------------------------------------------------------------- wide graphs --
// 64 < n <= 255: a bitset is NW 64-bit words (NW = 2: n <= 128, NW = 4:
// n <= 255). A class no longer fits a lane's registers, and a level can hold
// up to 255 classes, so the wide policy keeps every level in memory (the
// per-warp shared-memory stack, spilling to HBM) and walks it 32 classes per
// pass, lane = class. The per-class counts that every u candidate of a level
// reuses (|LX ∩ part|, |R| - [selected]) are computed once per level into a
// shared-memory scratch. Adjacency rows are read through the read-only data
// path (L1), not staged: 255 rows × 32 B × 4 row sets would leave no room
// for resident warps.
template <int NW, bool DIR>
struct WideSmem {
    static constexpr int NB = NW >= 4 ? kMaxWideN : NW * 64;  // vertex capacity
    static constexpr int P = DIR ? 4 : 2;
    unsigned long long f_word[NB + 1];
    alignas(16) uint32_t pf[24];
    unsigned long long polled;
    unsigned long long st_nodes, st_splits, st_split_cls, st_donations, st_tasks, st_spills;
    unsigned long long st_idle, st_busy;
    unsigned long long deadline;
    long long t_mark;
    TaskCold tc;
    WSet<NW> f_cand[NB + 1];
    uint32_t vkey[NB];
    uint8_t map_v[NB + 1];
    uint8_t map_u[NB + 1];
    uint8_t lcs[NB][P];  // |LX ∩ part_q(v)| of each class of the current level
    uint8_t rss[NB];     // |R| - [class == selected]
};

template <int NW, bool DIR>
struct WideSearch {
    using Set = WSet<NW>;
    using C = Cls<Set>;
    using Sm = WideSmem<NW, DIR>;
    using Desc = WideDesc;
    using Slot = WideSlot;
    static constexpr int NB = Sm::NB;
    static constexpr int P = DIR ? 4 : 2;
    static constexpr int kMinBlocks = 2;
    static constexpr bool kSpill = true;
    static constexpr bool kBoundedStack = false;
    static constexpr bool kContSync = true;  // cont_step's write is read by other lanes at once (scan_key)
    static constexpr bool kColdSmem = true;
    __device__ static __forceinline__ int top(const Set& x) { return set_top(x); }
    static constexpr bool kNest = false;
    struct HParts {
        Set o, i;  // H rows of u (out; in when directed)
    };

    Sm& s;
    C* scls;
    C* gcls;
    int cap;
    int lane;
    unsigned lt;
    const Desc* dsc = nullptr;
    C* lvl = nullptr;  // current level
    int lnc = 0;
    Set vb, go, gi;    // bit of v, G rows of v

    __device__ __forceinline__ WideSearch(Sm& s_, C* scls_, C* gcls_, int cap_, int lane_, unsigned lt_)
        : s(s_), scls(scls_), gcls(gcls_), cap(cap_), lane(lane_), lt(lt_) {}

    __device__ static __forceinline__ const Desc* descs(const KernelParams& p) { return p.winst; }
    __device__ static __forceinline__ Slot* slots(const KernelParams& p) { return p.wslots; }
    __device__ static __forceinline__ int key_slot(unsigned key) { return int(key & 255u); }
    // vertex-id hooks (identity: the 32-bit compacted policy maps ids) and
    // the class-stack limit of the level placement
    __device__ __forceinline__ int g_orig(int v) const { return v; }
    __device__ __forceinline__ int h_orig(int u) const { return u; }
    __device__ __forceinline__ int g_local(int v) const { return v; }
    __device__ __forceinline__ int stack_limit(const KernelParams& p) const { return p.smem_classes + p.spill_classes; }

    // select_label_class key: (max, min, lowest left id, slot), 8 bits each
    template <bool TOP>
    __device__ static __forceinline__ unsigned class_key(int pl, int pr, const Set& l, int slot) {
        const unsigned mx = max(pl, pr), mn = min(pl, pr);
        return (mx << 24) | (mn << 16) | (unsigned(TOP ? 255 - set_top(l) : set_ctz(l)) << 8) | unsigned(slot);
    }

    __device__ static __forceinline__ Set row(const uint64_t (*rows)[kWideWords], int v) {
        Set x;
#pragma unroll
        for (int i = 0; i < NW; ++i) x.w[i] = __ldg(&rows[v][i]);
        return x;
    }
    // part q of a vertex's code row: undirected {¬adj, adj}; directed by
    // (out bit, in bit): {neither, out only, in only, both}
    __device__ static __forceinline__ Set part(int q, const Set& o, const Set& in) {
        Set r;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            const uint64_t a = o.w[i], b = DIR ? in.w[i] : 0ull;
            r.w[i] = q == 0 ? ~(a | b) : q == 1 ? (a & ~b) : q == 2 ? (b & ~a) : (a & b);
        }
        return r;
    }

    __device__ __forceinline__ bool in_smem(int base) const { return base < cap; }
    __device__ __forceinline__ C* at(int base) const { return in_smem(base) ? scls + base : gcls + (base - cap); }

    template <bool PAR>
    __device__ __forceinline__ void load_instance(const Desc& d) {
        dsc = &d;
        if constexpr (PAR)
            for (int i = lane; i < NB; i += 32) s.vkey[i] = d.vkey[i];
    }
    __device__ static __forceinline__ C from_words(const uint64_t* l, const uint64_t* r) {
        C c;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            c.l.w[i] = l[i];
            c.r.w[i] = r[i];
        }
        return c;
    }
    // the host keeps every level-0 level in shared memory (cap > NB)
    __device__ __forceinline__ void load_root(const Desc& d, int nc) {
        for (int i = lane; i < nc; i += 32) scls[i] = from_words(d.init_l[i], d.init_r[i]);
    }
    __device__ __forceinline__ void load_task(const Slot& sl, int nc, int d) {
        for (int i = lane; i < nc; i += 32) scls[i] = from_words(sl.cls[i][0], sl.cls[i][1]);
        for (int i = lane; i < d; i += 32) {
            s.map_v[i] = sl.map_v[i];
            s.map_u[i] = sl.map_u[i];
        }
    }
    __device__ static __forceinline__ Set slot_cand(const Slot& sl) {
        Set x;
#pragma unroll
        for (int i = 0; i < NW; ++i) x.w[i] = sl.cand[i];
        return x;
    }
    __device__ __forceinline__ void store_task(Slot& sl, int fbase, int fnc) const {
        const C* fp = at(fbase);
        for (int i = lane; i < fnc; i += 32) {
            const C c = fp[i];
#pragma unroll
            for (int k = 0; k < kWideWords; ++k) {
                sl.cls[i][0][k] = k < NW ? c.l.w[k < NW ? k : 0] : 0ull;
                sl.cls[i][1][k] = k < NW ? c.r.w[k < NW ? k : 0] : 0ull;
            }
        }
    }
    __device__ static __forceinline__ void put_cand(Slot& sl, TaskHeader& h, const Set& give) {
        h.cand = 0;
#pragma unroll
        for (int k = 0; k < kWideWords; ++k) sl.cand[k] = k < NW ? give.w[k < NW ? k : 0] : 0ull;
    }

    __device__ __forceinline__ void load_level(int base, int nc) {
        lvl = at(base);
        lnc = nc;
    }

    // compute_bound + select_label_class over the level
    template <bool TOP>
    __device__ __forceinline__ unsigned scan_key(int nc, unsigned* sum) const {
        unsigned key = kNoKey, sm = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) {
            const int c = c0 + lane;
            if (c < nc) {
                const C x = lvl[c];
                const int pl = set_popc(x.l), pr = set_popc(x.r);
                sm += unsigned(min(pl, pr));
                if (pl) key = min(key, class_key<TOP>(pl, pr, x.l, c));  // L = {}: a dead class
            }
        }
        if (sum) *sum = __reduce_add_sync(kFull, sm);
        return __reduce_min_sync(kFull, key);
    }

    // select_vertex (label_classes.cpp:69-78) over the vertex keys of L*
    __device__ __forceinline__ int select_vertex(const Set& lsel) const {
        unsigned k = kNoKey;
#pragma unroll
        for (int i = 0; i < NW; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int xb = lane + 32 * h, id = 64 * i + xb;
                if (id < NB && ((lsel.w[i] >> xb) & 1ull)) k = min(k, s.vkey[id]);
            }
        return int(__reduce_min_sync(kFull, k) & 255u);
    }

    __device__ __forceinline__ Set class_l(int c) const { return lvl[c].l; }
    __device__ __forceinline__ Set class_r(int c) const { return lvl[c].r; }

    __device__ __forceinline__ void prep_v(int v, int sel) {
        go = row(dsc->out_g, v);
        if constexpr (DIR) gi = row(dsc->in_g, v);
        vb = set_bit<NW>(v);
        for (int c0 = 0; c0 < lnc; c0 += 32) {
            const int c = c0 + lane;
            if (c < lnc) {
                const C x = lvl[c];
                const Set lx = set_andnot(x.l, vb);
                if constexpr (!DIR) {
                    const int a = set_popc(set_and(lx, go));
                    s.lcs[c][1] = uint8_t(a);
                    s.lcs[c][0] = uint8_t(set_popc(lx) - a);
                } else {
#pragma unroll
                    for (int q = 0; q < P; ++q) s.lcs[c][q] = uint8_t(set_popc(set_and(lx, part(q, go, gi))));
                }
                s.rss[c] = uint8_t(set_popc(x.r) - (c == sel ? 1 : 0));
            }
        }
        __syncwarp();
    }

    __device__ __forceinline__ void h_parts(int u, HParts& h) const {
        h.o = row(dsc->out_h, u);
        if constexpr (DIR) h.i = row(dsc->in_h, u);
    }

    // bound of the child minus |M|+1 (see Search::child_sum)
    __device__ __forceinline__ unsigned child_sum(int u, const HParts& h) const {
        (void)u;
        unsigned sm = 0;
        for (int c0 = 0; c0 < lnc; c0 += 32) {
            const int c = c0 + lane;
            if (c < lnc) {
                const Set r = lvl[c].r;
                const int rs = s.rss[c];
                if constexpr (!DIR) {
                    const int b = set_popc(set_and(r, h.o));
                    sm += unsigned(min(int(s.lcs[c][0]), rs - b) + min(int(s.lcs[c][1]), b));
                } else {
                    int rest = rs;
#pragma unroll
                    for (int q = 1; q < P; ++q) {
                        const int b = set_popc(set_and(r, part(q, h.o, h.i)));
                        rest -= b;
                        sm += unsigned(min(int(s.lcs[c][q]), b));
                    }
                    sm += unsigned(min(int(s.lcs[c][0]), rest));
                }
            }
        }
        return __reduce_add_sync(kFull, sm);
    }

    // filter_classes (label_classes.cpp:80-108) into the next level at cbase
    template <bool TOP>
    __device__ __forceinline__ int split(int u, int v, const HParts& h, int cbase, unsigned* key_out) {
        (void)v;
        C* q = at(cbase);
        const Set ub = set_bit<NW>(u);
        int total = 0;
        unsigned key = kNoKey;
        for (int c0 = 0; c0 < lnc; c0 += 32) {
            const int c = c0 + lane;
            C x{};
            if (c < lnc) x = lvl[c];
            const Set lx = set_andnot(x.l, vb), rx = set_andnot(x.r, ub);
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                const Set lp = set_and(lx, part(pp, go, gi)), rp = set_and(rx, part(pp, h.o, h.i));
                const bool keep = set_any(lp) & set_any(rp);
                const unsigned m = __ballot_sync(kFull, keep);
                if (keep) {
                    const int pos = total + __popc(m & lt);
                    q[pos] = C{lp, rp};
                    key = min(key, class_key<TOP>(set_popc(lp), set_popc(rp), lp, pos));
                }
                total += __popc(m);
            }
        }
        *key_out = __reduce_min_sync(kFull, key);
        return total;
    }

    // "v unmatched" (search_core.hpp:201-212), in the level's memory (an
    // emptied class stays in its slot, dead; see Search::cont_step)
    __device__ __forceinline__ void cont_step(int sel, int cbits, int base, int& bound) {
        (void)base;
        bound -= (cbits & kContDec) ? 1 : 0;
        if (lane == 0) lvl[sel].l = set_andnot(lvl[sel].l, vb);
    }
};

}  // namespace mcsg
