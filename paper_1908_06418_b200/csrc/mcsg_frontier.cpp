// Host-side frontier expansion for sharding ONE instance across devices.
//
// The top of the McSplit tree is expanded on the host into frozen subtrees
// (the same "branch" tasks the kernel donates: a node's classes, its mapping,
// the selected class and vertex, the u candidates left, and whether the
// v-unmatched continuation belongs to it). Every generated task is a disjoint
// part of the search tree and together they cover all of it, so dealing them
// to devices round-robin gives exactly-once coverage independent of the
// (racy) incumbent. Mirrors the reference's delegation of shallow nodes as
// SearchTasks (engine_parallel.cpp:86-117, task_queue.hpp:27-48) and the
// node rules of search_core.hpp:120-213 / label_classes.cpp:41-108.
#include <algorithm>
#include <array>
#include <tuple>
#include <cstring>
#include <deque>

#include "mcsg_frontier.hpp"

namespace mcsg {
namespace {

// Host bitset over up to 256 vertices (one word when n <= 64).
using HSet = std::array<uint64_t, kWideWords>;

inline int popc(const HSet& x) {
    int c = 0;
    for (uint64_t w : x) c += __builtin_popcountll(w);
    return c;
}
inline int ctz(const HSet& x) {
    for (int i = 0; i < kWideWords; ++i)
        if (x[i]) return 64 * i + __builtin_ctzll(x[i]);
    return -1;
}
inline int top(const HSet& x) {
    for (int i = kWideWords - 1; i >= 0; --i)
        if (x[i]) return 64 * i + 63 - __builtin_clzll(x[i]);
    return -1;
}
inline bool any(const HSet& x) { return (x[0] | x[1] | x[2] | x[3]) != 0; }
inline HSet band(const HSet& a, const HSet& b) { return {a[0] & b[0], a[1] & b[1], a[2] & b[2], a[3] & b[3]}; }
inline HSet bnot(const HSet& a) { return {~a[0], ~a[1], ~a[2], ~a[3]}; }
inline HSet without(HSet a, int v) {
    a[v >> 6] &= ~(1ull << (v & 63));
    return a;
}

// Rows and vertex keys of either description, as host sets.
inline HSet set_of(uint64_t x) { return {x, 0, 0, 0}; }
inline HSet set_of(const uint64_t (&x)[kWideWords]) { return {x[0], x[1], x[2], x[3]}; }

struct Node {
    std::vector<std::pair<HSet, HSet>> cls;
    std::vector<uint8_t> mv, mu;
    int bound = 0;
};

struct Branch {
    Node node;
    int sel = 0, v = 0;
    HSet cand{};
    int cont = 1;
};

int bound_of(const Node& n) {
    int b = int(n.mv.size());
    for (const auto& c : n.cls) b += std::min(popc(c.first), popc(c.second));
    return b;
}

// select_label_class + select_vertex (label_classes.cpp:47-78) on a node that
// survived its prune test; false when no class remains. Same rule as the
// throughput kernel: G is relabelled in REVERSE select_vertex order, so the
// class order is (max(|L|,|R|), min, highest left id, slot) and v is the
// highest id of the class.
template <class D>
bool enter(Node n, const D& d, Branch* out) {
    (void)d;
    std::tuple<int, int, int, int> best{1 << 30, 0, 0, 0};
    int sel = -1;
    for (int i = 0; i < int(n.cls.size()); ++i) {
        const int pl = popc(n.cls[i].first), pr = popc(n.cls[i].second);
        const std::tuple<int, int, int, int> k{std::max(pl, pr), std::min(pl, pr), -top(n.cls[i].first), i};
        if (k < best) best = k, sel = i;
    }
    if (sel < 0) return false;
    const int v = top(n.cls[sel].first);
    out->v = v;
    out->sel = sel;
    out->cand = n.cls[sel].second;
    // the kernel's continuation byte: owned | [|L*| <= |R*|] (kContDec)
    out->cont = 1 | (popc(n.cls[sel].first) <= popc(n.cls[sel].second) ? 2 : 0);
    out->node = std::move(n);
    return true;
}

// filter_classes (label_classes.cpp:80-108) for the child (v,u).
template <class D>
Node child_of(const Branch& b, int u, const D& d, bool directed) {
    Node c;
    c.mv = b.node.mv;
    c.mu = b.node.mu;
    c.mv.push_back(uint8_t(b.v));
    c.mu.push_back(uint8_t(u));
    const HSet ao = set_of(d.out_g[b.v]), ai = set_of(d.in_g[b.v]);
    const HSet bo = set_of(d.out_h[u]), bi = set_of(d.in_h[u]);
    HSet gp[4], hp[4];
    int parts = 2;
    if (!directed) {
        gp[0] = bnot(ao), gp[1] = ao, hp[0] = bnot(bo), hp[1] = bo;
    } else {
        parts = 4;
        gp[0] = band(bnot(ao), bnot(ai)), gp[1] = band(ao, bnot(ai)), gp[2] = band(ai, bnot(ao)), gp[3] = band(ao, ai);
        hp[0] = band(bnot(bo), bnot(bi)), hp[1] = band(bo, bnot(bi)), hp[2] = band(bi, bnot(bo)), hp[3] = band(bo, bi);
    }
    for (const auto& cl : b.node.cls) {
        const HSet l = without(cl.first, b.v), r = without(cl.second, u);
        for (int q = 0; q < parts; ++q) {
            const HSet lp = band(l, gp[q]), rp = band(r, hp[q]);
            if (any(lp) && any(rp)) c.cls.push_back({lp, rp});
        }
    }
    c.bound = bound_of(c);
    return c;
}

// v left unmatched (search_core.hpp:201-212).
Node continuation_of(const Branch& b) {
    Node c = b.node;
    const auto cl = c.cls[b.sel];
    c.bound -= popc(cl.first) <= popc(cl.second) ? 1 : 0;
    const HSet nl = without(cl.first, b.v);
    if (any(nl)) {
        c.cls[b.sel].first = nl;
    } else {
        c.cls[b.sel] = c.cls.back();
        c.cls.pop_back();
    }
    return c;
}

template <class S>
void fill_header(S& s, const Branch& b, int inst) {
    s.hdr.inst = inst;
    s.hdr.kind = kTaskBranch;
    s.hdr.depth = uint8_t(b.node.mv.size());
    s.hdr.nc = uint8_t(b.node.cls.size());
    s.hdr.sel = uint8_t(b.sel);
    s.hdr.v = uint8_t(b.v);
    s.hdr.bound = uint8_t(b.node.bound);
    s.hdr.cont = uint8_t(b.cont);
    for (size_t k = 0; k < b.node.mv.size(); ++k) {
        s.map_v[k] = b.node.mv[k];
        s.map_u[k] = b.node.mu[k];
    }
}

void push_slot(const Branch& b, int inst, Frontier* f, const InstanceDesc&) {
    TaskSlot s;
    std::memset(&s, 0, sizeof(s));
    fill_header(s, b, inst);
    s.hdr.cand = b.cand[0];
    for (size_t i = 0; i < b.node.cls.size(); ++i) {
        s.cls_l[i] = b.node.cls[i].first[0];
        s.cls_r[i] = b.node.cls[i].second[0];
    }
    f->tasks.push_back(s);
}

void push_slot(const Branch& b, int inst, Frontier* f, const WideDesc&) {
    f->wtasks.emplace_back();
    WideSlot& s = f->wtasks.back();
    std::memset(&s, 0, sizeof(s));
    fill_header(s, b, inst);
    for (int w = 0; w < kWideWords; ++w) s.cand[w] = b.cand[w];
    for (size_t i = 0; i < b.node.cls.size(); ++i)
        for (int w = 0; w < kWideWords; ++w) {
            s.cls[i][0][w] = b.node.cls[i].first[w];
            s.cls[i][1][w] = b.node.cls[i].second[w];
        }
}

template <class D>
Frontier expand(const D& d, bool directed, int target, int inst) {
    Frontier f;
    Node root;
    for (int i = 0; i < d.n_init; ++i) root.cls.push_back({set_of(d.init_l[i]), set_of(d.init_r[i])});
    root.bound = bound_of(root);
    f.nodes = 1;
    // The host keeps its own incumbent from the mappings it passes through:
    // pruning with it is exactly the kernel's rule (bound <= best).
    int best = 0;
    std::deque<Branch> open;
    {
        Branch b;
        if (d.prune && root.bound <= std::max(d.floor, d.goal - 1)) return f;
        if (!enter(root, d, &b)) return f;
        open.push_back(std::move(b));
    }
    while (!open.empty() && int(open.size()) < target) {
        Branch b = std::move(open.front());
        open.pop_front();
        const int depth = int(b.node.mv.size());
        for (HSet m = b.cand; any(m); m = without(m, ctz(m))) {
            const int u = ctz(m);
            Node c = child_of(b, u, d, directed);
            ++f.nodes;
            if (depth + 1 > best) {
                best = depth + 1;
                f.best_v = c.mv;
                f.best_u = c.mu;
                if (d.prune && d.goal == 0 && best >= d.maxp) {  // search_core.hpp:151-154
                    f.max_reached = true;
                    f.best_size = best;
                    return f;
                }
            }
            const int thr = d.prune ? std::max({best, d.floor, d.goal - 1}) : -1;
            if (c.bound <= thr) continue;
            Branch cb;
            if (enter(std::move(c), d, &cb)) open.push_back(std::move(cb));
        }
        if (b.cont) {
            Node c = continuation_of(b);
            ++f.nodes;
            const int thr = d.prune ? std::max({best, d.floor, d.goal - 1}) : -1;
            if (c.bound > thr) {
                Branch cb;
                if (enter(std::move(c), d, &cb)) open.push_back(std::move(cb));
            }
        }
    }
    f.best_size = best;
    for (const Branch& b : open) push_slot(b, inst, &f, d);
    return f;
}

}  // namespace

Frontier expand_frontier(const InstanceDesc& d, bool directed, int target, int inst) {
    return expand(d, directed, target, inst);
}

Frontier expand_frontier(const WideDesc& d, bool directed, int target, int inst) {
    return expand(d, directed, target, inst);
}

}  // namespace mcsg
