// Graph core and loader of the drop-in (host side, C++17).
//
// Restates the reference's graph layer (/root/reference/proj):
//   storage + codes        include/mcs/graph.hpp:31-62   (n*n byte codes, mirror-consistent)
//   degree                 src/graph.cpp:17-29           (directed: out + in)
//   random_graph           src/graph.cpp:136-161         (std::mt19937, fixed-point threshold)
//   random_permutation     src/graph.cpp:163-173
//   orderings              src/heuristics.cpp:30-101
//   verify                 src/oracle.cpp:8-24
//   MIVIA / text loaders   src/graph_io.cpp:35-166
// and packs graphs into the 64-bit adjacency rows the kernel stages in
// shared memory (the "graph loader" of the north star).
#include "mcsg_graph.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>
#include <sstream>

namespace mcsg {

HostGraph HostGraph::from_abi(const mcsg_graph* g) {
    if (!g) throw Error("null graph");
    if (g->n < 0) throw Error("negative vertex count");
    HostGraph out;
    out.n = g->n;
    out.directed = (g->flags & MCSG_DIRECTED) != 0;
    const size_t nn = size_t(out.n) * size_t(out.n);
    if (nn && !g->codes) throw Error("null code matrix");
    out.codes.assign(g->codes, g->codes + nn);
    if (g->flags & MCSG_LABELED) {
        if (out.n && !g->labels) throw Error("labeled graph without labels");
        out.labels.assign(g->labels, g->labels + out.n);
        out.labeled = true;
    }
    // mirror consistency (graph.hpp:13-16): code(u,v) forward <=> code(v,u) backward
    for (int u = 0; u < out.n; ++u) {
        if (out.code(u, u) != 0) throw Error("self-loop on vertex " + std::to_string(u));
        for (int v = u + 1; v < out.n; ++v) {
            const uint8_t a = out.code(u, v), b = out.code(v, u);
            const uint8_t lim = out.directed ? 3 : 1;
            if (a > lim || b > lim) throw Error("adjacency code out of range");
            const uint8_t mir = out.directed ? (a == 1 ? 2 : a == 2 ? 1 : a) : a;
            if (b != mir) throw Error("code matrix is not mirror-consistent");
        }
    }
    return out;
}

int HostGraph::degree(int v) const {
    int d = 0;
    for (int u = 0; u < n; ++u) {
        const uint8_t c = code(v, u);
        if (!directed) d += c != 0;
        else d += ((c & 1u) != 0) + ((c & 2u) != 0);
    }
    return d;
}

HostGraph HostGraph::permuted(const std::vector<int>& p) const {
    HostGraph out = *this;
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) out.codes[size_t(p[u]) * n + p[v]] = code(u, v);
    if (labeled)
        for (int v = 0; v < n; ++v) out.labels[p[v]] = labels[v];
    return out;
}

void random_graph(int n, double density, uint64_t seed, bool directed, int label_count,
                  uint8_t* codes, int32_t* labels) {
    if (n < 0) throw Error("negative vertex count");
    if (density < 0.0 || density > 1.0) throw Error("density must be in [0,1]");
    std::mt19937 gen(static_cast<uint32_t>(seed));
    const uint64_t thr = static_cast<uint64_t>(density * 4294967296.0);
    std::memset(codes, 0, size_t(n) * size_t(n));
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v) {
            if (static_cast<uint64_t>(gen()) >= thr) continue;
            uint8_t c = 1, m = 1;
            if (directed) {
                c = static_cast<uint8_t>(1 + gen() % 3);
                m = c == 1 ? 2 : c == 2 ? 1 : 3;
            }
            codes[size_t(u) * n + v] = c;
            codes[size_t(v) * n + u] = m;
        }
    if (label_count > 0 && labels)
        for (int v = 0; v < n; ++v) labels[v] = static_cast<int32_t>(gen() % unsigned(label_count));
}

std::vector<int> random_permutation(int n, uint64_t seed) {
    std::mt19937 gen(static_cast<uint32_t>(seed));
    std::vector<int> f(n);
    std::iota(f.begin(), f.end(), 0);
    for (int i = n - 1; i > 0; --i) std::swap(f[i], f[gen() % unsigned(i + 1)]);
    return f;
}

namespace {

std::vector<int> to_forward(const std::vector<int>& order) {
    std::vector<int> fwd(order.size());
    for (size_t pos = 0; pos < order.size(); ++pos) fwd[order[pos]] = int(pos);
    return fwd;
}

void by_degree(const HostGraph& g, std::vector<int>& members) {
    std::vector<int> deg(g.n);
    for (int v = 0; v < g.n; ++v) deg[v] = g.degree(v);
    std::stable_sort(members.begin(), members.end(), [&](int a, int b) {
        return deg[a] != deg[b] ? deg[a] > deg[b] : a < b;
    });
}

}  // namespace

// heuristics.cpp:30-101 (degree / components / block-triangular).
std::vector<int> make_ordering(const HostGraph& g, int strategy) {
    const int n = g.n;
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    switch (strategy) {
        case MCSG_ORDER_NONE: return order;
        case MCSG_ORDER_DEGREE: by_degree(g, order); return to_forward(order);
        case MCSG_ORDER_COMPONENTS: {
            std::vector<int> comp(n, -1);
            std::vector<std::vector<int>> comps;
            for (int s = 0; s < n; ++s) {
                if (comp[s] != -1) continue;
                const int id = int(comps.size());
                comps.emplace_back();
                std::vector<int> stack{s};
                comp[s] = id;
                while (!stack.empty()) {
                    const int v = stack.back();
                    stack.pop_back();
                    comps[id].push_back(v);
                    for (int u = 0; u < n; ++u)
                        if (comp[u] == -1 && g.code(v, u) != 0) {
                            comp[u] = id;
                            stack.push_back(u);
                        }
                }
                std::sort(comps[id].begin(), comps[id].end());
            }
            std::stable_sort(comps.begin(), comps.end(), [](const auto& a, const auto& b) {
                return a.size() != b.size() ? a.size() > b.size() : a[0] < b[0];
            });
            order.clear();
            for (auto& c : comps) {
                by_degree(g, c);
                order.insert(order.end(), c.begin(), c.end());
            }
            return to_forward(order);
        }
        case MCSG_ORDER_BLOCK: {
            std::vector<char> col(n, 0), row(n, 0), placed(n, 0);
            for (int v = 0; v < n; ++v)
                if (g.degree(v) > 0) col[v] = row[v] = 1;
            order.clear();
            std::vector<int> len(n);
            for (;;) {
                int minlen = -1;
                for (int r = 0; r < n; ++r) {
                    len[r] = 0;
                    if (!row[r]) continue;
                    for (int c = 0; c < n; ++c) len[r] += col[c] && g.code(r, c) != 0;
                    if (len[r] == 0) {
                        row[r] = 0;
                        continue;
                    }
                    if (minlen < 0 || len[r] < minlen) minlen = len[r];
                }
                if (minlen < 0) break;
                int best = -1, hits_best = -1;
                for (int c = 0; c < n; ++c) {
                    if (!col[c]) continue;
                    int hits = 0;
                    for (int r = 0; r < n; ++r) hits += row[r] && len[r] == minlen && g.code(r, c) != 0;
                    if (hits > hits_best) hits_best = hits, best = c;
                }
                order.push_back(best);
                placed[best] = 1;
                col[best] = 0;
            }
            for (int v = 0; v < n; ++v)
                if (!placed[v]) order.push_back(v);
            return to_forward(order);
        }
    }
    throw Error("unknown ordering strategy");
}

int verify(const HostGraph& g, const HostGraph& h, const int32_t* pairs, int k) {
    std::vector<char> ug(g.n, 0), uh(h.n, 0);
    for (int i = 0; i < k; ++i) {
        const int v = pairs[2 * i], u = pairs[2 * i + 1];
        if (v < 0 || v >= g.n || u < 0 || u >= h.n) throw Error("verify: vertex out of range");
    }
    for (int i = 0; i < k; ++i) {
        const int v = pairs[2 * i], u = pairs[2 * i + 1];
        if (ug[v] || uh[u]) return 0;
        ug[v] = uh[u] = 1;
        if (g.labeled != h.labeled) return 0;
        if (g.labeled && g.labels[v] != h.labels[u]) return 0;
    }
    for (int i = 0; i < k; ++i)
        for (int j = i + 1; j < k; ++j)
            if (g.code(pairs[2 * i], pairs[2 * j]) != h.code(pairs[2 * i + 1], pairs[2 * j + 1])) return 0;
    return 1;
}

// ---------------------------------------------------------------- loaders --
namespace {

HostGraph build(int n, bool directed, const std::vector<std::array<int, 3>>& edges,
                const std::vector<int32_t>* labels) {
    if (n < 0) throw Error("negative vertex count");
    HostGraph g;
    g.n = n;
    g.directed = directed;
    g.codes.assign(size_t(n) * n, 0);
    if (labels) {
        g.labeled = true;
        g.labels = *labels;
    }
    for (const auto& e : edges) {
        const int u = e[0], v = e[1];
        if (u < 0 || u >= n || v < 0 || v >= n)
            throw Error("edge endpoint out of range: (" + std::to_string(u) + "," + std::to_string(v) + ")");
        if (u == v) throw Error("self-loop on vertex " + std::to_string(u));
        uint8_t f = 1, b = 1;
        if (directed) {
            if (e[2] < 1 || e[2] > 3) throw Error("directed edge with code none");
            f = uint8_t(e[2]);
            b = f == 1 ? 2 : f == 2 ? 1 : 3;
        }
        uint8_t& cell = g.codes[size_t(u) * n + v];
        if (cell != 0 && cell != f)
            throw Error("conflicting duplicate edge (" + std::to_string(u) + "," + std::to_string(v) + ")");
        cell = f;
        g.codes[size_t(v) * n + u] = b;
    }
    return g;
}

}  // namespace

// MIVIA ARG binary (graph_io.cpp:35-67): u16 LE node count, then per node a
// u16 edge count and that many u16 targets; undirected.
HostGraph load_mivia(const std::vector<uint8_t>& bytes) {
    size_t pos = 0;
    auto u16 = [&]() -> int {
        if (pos + 2 > bytes.size()) throw ParseErr("truncated MIVIA stream");
        const int v = bytes[pos] | (bytes[pos + 1] << 8);
        pos += 2;
        return v;
    };
    const int n = u16();
    std::vector<std::array<int, 3>> edges;
    for (int i = 0; i < n; ++i) {
        const int k = u16();
        for (int j = 0; j < k; ++j) {
            const int t = u16();
            if (t >= n) throw ParseErr("target id " + std::to_string(t) + " >= n=" + std::to_string(n));
            if (t == i) throw ParseErr("self-loop on vertex " + std::to_string(i));
            edges.push_back({std::min(i, t), std::max(i, t), 1});
        }
    }
    if (pos != bytes.size()) throw ParseErr("trailing bytes after MIVIA graph");
    return build(n, false, edges, nullptr);
}

std::vector<uint8_t> save_mivia(const HostGraph& g) {
    if (g.directed) throw Error("MIVIA writer supports undirected graphs only");
    if (g.n > 0xffff) throw Error("graph too large for 16-bit MIVIA format");
    std::vector<uint8_t> out;
    auto put = [&](int v) {
        out.push_back(uint8_t(v & 0xff));
        out.push_back(uint8_t((v >> 8) & 0xff));
    };
    put(g.n);
    for (int i = 0; i < g.n; ++i) {
        int k = 0;
        for (int t = 0; t < g.n; ++t) k += g.code(i, t) != 0;
        put(k);
        for (int t = 0; t < g.n; ++t)
            if (g.code(i, t) != 0) put(t);
    }
    return out;
}

// Text format (graph_io.cpp:69-137): "n [directed] [labeled]", n label lines
// when labeled, then "u v [code]" edge lines.
HostGraph load_text(const std::string& text) {
    std::istringstream in(text);
    std::string header;
    while (std::getline(in, header))
        if (header.find_first_not_of(" \t\r") != std::string::npos) break;
    std::istringstream hl(header);
    int n;
    if (!(hl >> n)) throw ParseErr("text graph: missing vertex count");
    bool directed = false, labeled = false;
    std::string w;
    while (hl >> w) {
        if (w == "directed") directed = true;
        else if (w == "labeled") labeled = true;
        else throw ParseErr("text graph: unknown header word '" + w + "'");
    }
    std::vector<int32_t> labels;
    if (labeled) {
        if (n < 0) throw Error("negative vertex count");
        labels.assign(n, -1);
        for (int i = 0; i < n; ++i) {
            int v, lab;
            if (!(in >> v >> lab)) throw ParseErr("text graph: missing label line");
            if (v < 0 || v >= n) throw ParseErr("text graph: label vertex out of range");
            labels[v] = lab;
        }
        for (int v = 0; v < n; ++v)
            if (labels[v] < 0) throw ParseErr("text graph: vertex " + std::to_string(v) + " has no label");
    }
    std::vector<std::array<int, 3>> edges;
    std::string line;
    while (std::getline(in, line)) {
        std::istringstream el(line);
        int u, v;
        if (!(el >> u)) {
            if (line.find_first_not_of(" \t\r") != std::string::npos)
                throw ParseErr("text graph: malformed edge line '" + line + "'");
            continue;
        }
        if (!(el >> v)) throw ParseErr("text graph: malformed edge line '" + line + "'");
        int c = 1;
        el >> c;
        if (c < 1 || c > 3) throw ParseErr("text graph: edge code out of range");
        edges.push_back({u, v, c});
    }
    return build(n, directed, edges, labeled ? &labels : nullptr);
}

std::string save_text(const HostGraph& g) {
    std::ostringstream out;
    out << g.n;
    if (g.directed) out << " directed";
    if (g.labeled) out << " labeled";
    out << "\n";
    if (g.labeled)
        for (int v = 0; v < g.n; ++v) out << v << " " << g.labels[v] << "\n";
    for (int u = 0; u < g.n; ++u)
        for (int v = u + 1; v < g.n; ++v) {
            const uint8_t c = g.code(u, v);
            if (!c) continue;
            out << u << " " << v;
            if (g.directed) out << " " << int(c);
            out << "\n";
        }
    return out.str();
}

HostGraph load_graph_file(const std::string& path, int format) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseErr("cannot open '" + path + "'");
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (format == 2) format = (!bytes.empty() && bytes[0] >= '0' && bytes[0] <= '9') ? 1 : 0;
    if (format == 1) return load_text(std::string(bytes.begin(), bytes.end()));
    return load_mivia(bytes);
}

void save_graph_file(const HostGraph& g, const std::string& path, int format) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write '" + path + "'");
    if (format == 1) {
        const std::string s = save_text(g);
        out.write(s.data(), std::streamsize(s.size()));
    } else {
        const auto b = save_mivia(g);
        out.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
    }
}

// ------------------------------------------------------------------ packer --
// The loader's device form: per vertex one 64-bit row of the code matrix
// (bit x of out[v] = code(v,x) & 1, of in[v] = code(v,x) & 2), the
// select_vertex key (255 - degree) << 6 | id, and the initial classes
// (label_classes.cpp:8-39: all vertices, or one class per shared label in
// ascending label order).
void pack_instance(const HostGraph& g, const HostGraph& h, int goal, bool prune, int floor_size,
                   int group, InstanceDesc* d) {
    if (g.directed != h.directed) throw Error("solve: graphs must share a kind");
    if (g.labeled != h.labeled) throw Error("cannot mix a labeled graph with an unlabeled one");
    if (g.n > kMaxN || h.n > kMaxN)
        throw Error("graphs above " + std::to_string(kMaxN) + " vertices are not supported (n=" +
                    std::to_string(std::max(g.n, h.n)) + ")");
    std::memset(d, 0, sizeof(*d));
    d->n_g = g.n;
    d->n_h = h.n;
    d->maxp = std::min(g.n, h.n);
    d->goal = goal;
    d->prune = prune ? 1 : 0;
    d->floor = floor_size;
    d->group = group;
    auto rows = [](const HostGraph& x, uint64_t* out, uint64_t* in) {
        for (int v = 0; v < x.n; ++v) {
            uint64_t o = 0, i = 0;
            for (int u = 0; u < x.n; ++u) {
                const uint8_t c = x.code(v, u);
                if (c & 1u) o |= 1ull << u;
                if (c & 2u) i |= 1ull << u;
            }
            out[v] = o;
            in[v] = i;
        }
    };
    rows(g, d->out_g, d->in_g);
    rows(h, d->out_h, d->in_h);
    for (int v = 0; v < kMaxN; ++v) d->vkey[v] = 0xffff;
    for (int v = 0; v < g.n; ++v) d->vkey[v] = uint16_t(((255 - g.degree(v)) << 6) | v);
    int nc = 0;
    if (!g.labeled) {
        if (g.n > 0 && h.n > 0) {
            d->init_l[0] = g.n == 64 ? ~0ull : ((1ull << g.n) - 1);
            d->init_r[0] = h.n == 64 ? ~0ull : ((1ull << h.n) - 1);
            nc = 1;
        }
    } else {
        std::vector<int32_t> labs(g.labels.begin(), g.labels.end());
        std::sort(labs.begin(), labs.end());
        labs.erase(std::unique(labs.begin(), labs.end()), labs.end());
        for (int32_t lab : labs) {
            uint64_t l = 0, r = 0;
            for (int v = 0; v < g.n; ++v)
                if (g.labels[v] == lab) l |= 1ull << v;
            for (int u = 0; u < h.n; ++u)
                if (h.labels[u] == lab) r |= 1ull << u;
            if (l && r) {
                d->init_l[nc] = l;
                d->init_r[nc] = r;
                ++nc;
            }
        }
    }
    d->n_init = nc;
}

// The same device form for 64 < n <= 255: rows of kWideWords words (bit x%64
// of word x/64), vertex key (1023 - degree) << 8 | id (a directed degree
// reaches 2 * 254).
void pack_wide(const HostGraph& g, const HostGraph& h, int goal, bool prune, int floor_size, int group,
               WideDesc* d) {
    if (g.directed != h.directed) throw Error("solve: graphs must share a kind");
    if (g.labeled != h.labeled) throw Error("cannot mix a labeled graph with an unlabeled one");
    if (g.n > kMaxWideN || h.n > kMaxWideN)
        throw Error("graphs above " + std::to_string(kMaxWideN) + " vertices are not supported (n=" +
                    std::to_string(std::max(g.n, h.n)) + ")");
    std::memset(d, 0, sizeof(*d));
    d->n_g = g.n;
    d->n_h = h.n;
    d->maxp = std::min(g.n, h.n);
    d->goal = goal;
    d->prune = prune ? 1 : 0;
    d->floor = floor_size;
    d->group = group;
    auto set = [](uint64_t* row, int x) { row[x >> 6] |= 1ull << (x & 63); };
    auto rows = [&](const HostGraph& x, uint64_t (*out)[kWideWords], uint64_t (*in)[kWideWords]) {
        for (int v = 0; v < x.n; ++v)
            for (int u = 0; u < x.n; ++u) {
                const uint8_t c = x.code(v, u);
                if (c & 1u) set(out[v], u);
                if (c & 2u) set(in[v], u);
            }
    };
    rows(g, d->out_g, d->in_g);
    rows(h, d->out_h, d->in_h);
    for (int v = 0; v <= kMaxWideN; ++v) d->vkey[v] = 0xffffffffu;
    for (int v = 0; v < g.n; ++v) d->vkey[v] = uint32_t(((1023 - g.degree(v)) << 8) | v);
    int nc = 0;
    if (!g.labeled) {
        if (g.n > 0 && h.n > 0) {
            for (int v = 0; v < g.n; ++v) set(d->init_l[0], v);
            for (int u = 0; u < h.n; ++u) set(d->init_r[0], u);
            nc = 1;
        }
    } else {
        std::vector<int32_t> labs(g.labels.begin(), g.labels.end());
        std::sort(labs.begin(), labs.end());
        labs.erase(std::unique(labs.begin(), labs.end()), labs.end());
        for (int32_t lab : labs) {
            bool l = false, r = false;
            for (int v = 0; v < g.n; ++v) l |= g.labels[v] == lab;
            for (int u = 0; u < h.n; ++u) r |= h.labels[u] == lab;
            if (!(l && r)) continue;
            for (int v = 0; v < g.n; ++v)
                if (g.labels[v] == lab) set(d->init_l[nc], v);
            for (int u = 0; u < h.n; ++u)
                if (h.labels[u] == lab) set(d->init_r[nc], u);
            ++nc;
        }
    }
    d->n_init = nc;
}

}  // namespace mcsg
