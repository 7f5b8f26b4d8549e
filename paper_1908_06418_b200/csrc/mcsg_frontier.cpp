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
#include <cstring>
#include <deque>

#include "mcsg_frontier.hpp"

namespace mcsg {
namespace {

inline int popc(uint64_t x) { return __builtin_popcountll(x); }
inline int ctz(uint64_t x) { return __builtin_ctzll(x); }

struct Node {
    std::vector<std::pair<uint64_t, uint64_t>> cls;
    std::vector<uint8_t> mv, mu;
    int bound = 0;
};

struct Branch {
    Node node;
    int sel = 0, v = 0;
    uint64_t cand = 0;
    int cont = 1;
};

unsigned class_key(int pl, int pr, uint64_t l, int slot) {
    const unsigned mx = std::max(pl, pr), mn = std::min(pl, pr);
    return (mx << 20) | (mn << 13) | (unsigned(ctz(l)) << 7) | unsigned(slot);
}

int bound_of(const Node& n) {
    int b = int(n.mv.size());
    for (const auto& c : n.cls) b += std::min(popc(c.first), popc(c.second));
    return b;
}

// select_label_class + select_vertex (label_classes.cpp:47-78) on a node that
// survived its prune test; false when no class remains.
bool enter(Node n, const InstanceDesc& d, Branch* out) {
    unsigned best = ~0u;
    int sel = -1;
    for (int i = 0; i < int(n.cls.size()); ++i) {
        const unsigned k = class_key(popc(n.cls[i].first), popc(n.cls[i].second), n.cls[i].first, i);
        if (k < best) best = k, sel = i;
    }
    if (sel < 0) return false;
    const uint64_t l = n.cls[sel].first;
    unsigned vk = ~0u;
    for (uint64_t m = l; m; m &= m - 1) vk = std::min(vk, unsigned(d.vkey[ctz(m)]));
    out->v = int(vk & 63u);
    out->sel = sel;
    out->cand = n.cls[sel].second;
    out->cont = 1;
    out->node = std::move(n);
    return true;
}

// filter_classes (label_classes.cpp:80-108) for the child (v,u).
Node child_of(const Branch& b, int u, const InstanceDesc& d, bool directed) {
    Node c;
    c.mv = b.node.mv;
    c.mu = b.node.mu;
    c.mv.push_back(uint8_t(b.v));
    c.mu.push_back(uint8_t(u));
    const uint64_t ao = d.out_g[b.v], ai = d.in_g[b.v], bo = d.out_h[u], bi = d.in_h[u];
    uint64_t gp[4], hp[4];
    int parts = 2;
    if (!directed) {
        gp[0] = ~ao, gp[1] = ao, hp[0] = ~bo, hp[1] = bo;
    } else {
        parts = 4;
        gp[0] = ~(ao | ai), gp[1] = ao & ~ai, gp[2] = ai & ~ao, gp[3] = ao & ai;
        hp[0] = ~(bo | bi), hp[1] = bo & ~bi, hp[2] = bi & ~bo, hp[3] = bo & bi;
    }
    const uint64_t vb = 1ull << b.v, ub = 1ull << u;
    for (const auto& cl : b.node.cls) {
        const uint64_t l = cl.first & ~vb, r = cl.second & ~ub;
        for (int q = 0; q < parts; ++q) {
            const uint64_t lp = l & gp[q], rp = r & hp[q];
            if (lp && rp) c.cls.push_back({lp, rp});
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
    const uint64_t nl = cl.first & ~(1ull << b.v);
    if (nl) {
        c.cls[b.sel].first = nl;
    } else {
        c.cls[b.sel] = c.cls.back();
        c.cls.pop_back();
    }
    return c;
}

TaskSlot to_slot(const Branch& b, int inst) {
    TaskSlot s;
    std::memset(&s, 0, sizeof(s));
    s.hdr.inst = inst;
    s.hdr.kind = kTaskBranch;
    s.hdr.depth = uint8_t(b.node.mv.size());
    s.hdr.nc = uint8_t(b.node.cls.size());
    s.hdr.sel = uint8_t(b.sel);
    s.hdr.v = uint8_t(b.v);
    s.hdr.bound = uint8_t(b.node.bound);
    s.hdr.cont = uint8_t(b.cont);
    s.hdr.cand = b.cand;
    for (size_t k = 0; k < b.node.mv.size(); ++k) {
        s.map_v[k] = b.node.mv[k];
        s.map_u[k] = b.node.mu[k];
    }
    for (size_t i = 0; i < b.node.cls.size(); ++i) {
        s.cls_l[i] = b.node.cls[i].first;
        s.cls_r[i] = b.node.cls[i].second;
    }
    return s;
}

}  // namespace

Frontier expand_frontier(const InstanceDesc& d, bool directed, int target, int inst) {
    Frontier f;
    Node root;
    for (int i = 0; i < d.n_init; ++i) root.cls.push_back({d.init_l[i], d.init_r[i]});
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
        for (uint64_t m = b.cand; m; m &= m - 1) {
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
    for (const Branch& b : open) f.tasks.push_back(to_slot(b, inst));
    return f;
}

}  // namespace mcsg
