/* TEST INFRASTRUCTURE ONLY — CPU oracle for the McSplit search path.
 *
 * Plain-C restatement of the reference's sequential branch-and-bound
 * (/root/reference/proj). Every function cites the reference file:line it
 * restates. It is the checker for the CUDA path (tests/, smoke()) and the
 * "port" CPU baseline; the product library never links or calls it.
 *
 * Representation follows the reference: label classes are windows
 * (start, length) into two shared vertex buffers that each recursion level
 * re-partitions in place (label_classes.hpp:12-27). The split is a stable
 * counting partition by adjacency code instead of std::sort; the reference's
 * sort is unstable and window order never influences which node comes next
 * (every selection rule is a total order on vertex ids), so node counts match.
 */
#define _POSIX_C_SOURCE 199309L
#include "mcs_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------ mt19937 -- */
/* std::mt19937 (32-bit Mersenne twister) as used by random_graph,
 * graph.cpp:138 and random_permutation, graph.cpp:164. */
typedef struct {
    uint32_t s[624];
    int i;
} mt32;

static void mt_seed(mt32* m, uint32_t seed) {
    m->s[0] = seed;
    for (int k = 1; k < 624; ++k)
        m->s[k] = 1812433253u * (m->s[k - 1] ^ (m->s[k - 1] >> 30)) + (uint32_t)k;
    m->i = 624;
}

static uint32_t mt_next(mt32* m) {
    if (m->i >= 624) {
        for (int k = 0; k < 624; ++k) {
            uint32_t y = (m->s[k] & 0x80000000u) | (m->s[(k + 1) % 624] & 0x7fffffffu);
            uint32_t x = m->s[(k + 397) % 624] ^ (y >> 1);
            if (y & 1u) x ^= 0x9908b0dfu;
            m->s[k] = x;
        }
        m->i = 0;
    }
    uint32_t y = m->s[m->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* random_graph, graph.cpp:136-161: one raw draw per unordered pair (u<v)
 * against a fixed-point threshold, one extra draw for the directed code,
 * then one draw per vertex label. */
void orc_random_graph(int n, double density, uint64_t seed, int directed, int label_count,
                      uint8_t* codes_out, int32_t* labels_out) {
    mt32 m;
    mt_seed(&m, (uint32_t)seed);
    const uint64_t thr = (uint64_t)(density * 4294967296.0);
    memset(codes_out, 0, (size_t)n * (size_t)n);
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v) {
            if ((uint64_t)mt_next(&m) < thr) {
                uint8_t c = 1;
                if (directed) c = (uint8_t)(1 + mt_next(&m) % 3u);
                codes_out[(size_t)u * n + v] = c;
                /* mirror: forward <-> backward, both stays (graph.cpp:9-15,57-68) */
                codes_out[(size_t)v * n + u] = (uint8_t)(c == 1 ? (directed ? 2 : 1) : c == 2 ? 1 : c);
            }
        }
    if (label_count > 0 && labels_out)
        for (int v = 0; v < n; ++v) labels_out[v] = (int32_t)(mt_next(&m) % (uint32_t)label_count);
}

/* random_permutation, graph.cpp:163-173 (Fisher-Yates on raw draws). */
void orc_random_permutation(int n, uint64_t seed, int32_t* f) {
    mt32 m;
    mt_seed(&m, (uint32_t)seed);
    for (int i = 0; i < n; ++i) f[i] = i;
    for (int i = n - 1; i > 0; --i) {
        int j = (int)(mt_next(&m) % (uint32_t)(i + 1));
        int32_t t = f[i];
        f[i] = f[j];
        f[j] = t;
    }
}

static inline uint8_t code(const orc_graph* g, int u, int v) {
    return g->codes[(size_t)u * g->n + v];
}

/* Graph::degree, graph.cpp:17-29: out+in for directed ('both' counts twice). */
int orc_degree(const orc_graph* g, int v) {
    int d = 0;
    for (int u = 0; u < g->n; ++u) {
        uint8_t c = code(g, v, u);
        if (!g->directed) d += c != 0;
        else d += ((c & 1u) != 0) + ((c & 2u) != 0);
    }
    return d;
}

/* ---------------------------------------------------------- orderings -- */
static int* g_sort_deg; /* qsort context (single-threaded oracle) */

static int cmp_deg_desc(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    if (g_sort_deg[x] != g_sort_deg[y]) return g_sort_deg[x] > g_sort_deg[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

static void to_forward(const int* order, int n, int32_t* fwd) {
    for (int pos = 0; pos < n; ++pos) fwd[order[pos]] = pos;
}

/* order_by_degree, heuristics.cpp:30-34 (stable: degree desc, id asc). */
static void order_degree(const orc_graph* g, int32_t* fwd) {
    int n = g->n;
    int* deg = malloc(sizeof(int) * (n + 1));
    int* ord = malloc(sizeof(int) * (n + 1));
    for (int v = 0; v < n; ++v) deg[v] = orc_degree(g, v), ord[v] = v;
    g_sort_deg = deg;
    qsort(ord, n, sizeof(int), cmp_deg_desc);
    to_forward(ord, n, fwd);
    free(deg);
    free(ord);
}

/* order_by_components, heuristics.cpp:36-48 over connected_components,
 * graph.cpp:111-134: components largest first (ties: smallest member), each
 * internally degree-ordered. */
static void order_components(const orc_graph* g, int32_t* fwd) {
    int n = g->n;
    int* comp = malloc(sizeof(int) * (n + 1));
    int* deg = malloc(sizeof(int) * (n + 1));
    int* stack = malloc(sizeof(int) * (n + 1));
    int* csize = calloc(n + 1, sizeof(int));
    int* cfirst = malloc(sizeof(int) * (n + 1));
    int* ord = malloc(sizeof(int) * (n + 1));
    int nc = 0;
    for (int v = 0; v < n; ++v) comp[v] = -1, deg[v] = orc_degree(g, v);
    for (int s = 0; s < n; ++s) {
        if (comp[s] != -1) continue;
        int sp = 0;
        comp[s] = nc;
        stack[sp++] = s;
        cfirst[nc] = s;
        while (sp) {
            int v = stack[--sp];
            csize[nc]++;
            for (int u = 0; u < n; ++u)
                if (comp[u] == -1 && code(g, v, u) != 0) comp[u] = nc, stack[sp++] = u;
        }
        nc++;
    }
    /* component order: size desc, then smallest member asc (insertion sort, stable) */
    int* corder = malloc(sizeof(int) * (nc + 1));
    for (int c = 0; c < nc; ++c) {
        int j = c;
        while (j > 0 && (csize[corder[j - 1]] < csize[c] ||
                         (csize[corder[j - 1]] == csize[c] && cfirst[corder[j - 1]] > cfirst[c]))) {
            corder[j] = corder[j - 1];
            --j;
        }
        corder[j] = c;
    }
    int k = 0;
    g_sort_deg = deg;
    for (int ci = 0; ci < nc; ++ci) {
        int c = corder[ci];
        int start = k;
        for (int v = 0; v < n; ++v)
            if (comp[v] == c) ord[k++] = v;
        qsort(ord + start, k - start, sizeof(int), cmp_deg_desc);
    }
    to_forward(ord, n, fwd);
    free(comp), free(deg), free(stack), free(csize), free(cfirst), free(ord), free(corder);
}

/* order_block_triangular, heuristics.cpp:50-91: repeatedly move to the border
 * the column hitting the most shortest active rows (ties: lowest id). */
static void order_block(const orc_graph* g, int32_t* fwd) {
    int n = g->n;
    char* col = calloc(n + 1, 1);
    char* row = calloc(n + 1, 1);
    char* placed = calloc(n + 1, 1);
    int* rlen = malloc(sizeof(int) * (n + 1));
    int* ord = malloc(sizeof(int) * (n + 1));
    int k = 0;
    for (int v = 0; v < n; ++v)
        if (orc_degree(g, v) > 0) col[v] = row[v] = 1;
    for (;;) {
        int minlen = -1;
        for (int r = 0; r < n; ++r) {
            rlen[r] = 0;
            if (!row[r]) continue;
            for (int c = 0; c < n; ++c)
                if (col[c] && code(g, r, c) != 0) rlen[r]++;
            if (rlen[r] == 0) {
                row[r] = 0;
                continue;
            }
            if (minlen == -1 || rlen[r] < minlen) minlen = rlen[r];
        }
        if (minlen == -1) break;
        int best = -1, hits_best = -1;
        for (int c = 0; c < n; ++c) {
            if (!col[c]) continue;
            int hits = 0;
            for (int r = 0; r < n; ++r)
                if (row[r] && rlen[r] == minlen && code(g, r, c) != 0) hits++;
            if (hits > hits_best) hits_best = hits, best = c;
        }
        ord[k++] = best;
        placed[best] = 1;
        col[best] = 0;
    }
    for (int v = 0; v < n; ++v)
        if (!placed[v]) ord[k++] = v;
    to_forward(ord, n, fwd);
    free(col), free(row), free(placed), free(rlen), free(ord);
}

/* make_ordering, heuristics.cpp:93-101. */
int orc_ordering(const orc_graph* g, int strategy, int32_t* fwd) {
    switch (strategy) {
        case 0:
            for (int v = 0; v < g->n; ++v) fwd[v] = v;
            return 0;
        case 1: order_degree(g, fwd); return 0;
        case 2: order_components(g, fwd); return 0;
        case 3: order_block(g, fwd); return 0;
    }
    return -1;
}

/* permute, graph.cpp:94-109: adjacency(p(u),p(v)) of the result equals
 * adjacency(u,v) of g; labels follow. Caller owns the buffers. */
static void permute_into(const orc_graph* g, const int32_t* p, uint8_t* codes, int32_t* labels,
                         orc_graph* out) {
    int n = g->n;
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) codes[(size_t)p[u] * n + p[v]] = code(g, u, v);
    if (g->labels)
        for (int v = 0; v < n; ++v) labels[p[v]] = g->labels[v];
    out->n = n;
    out->directed = g->directed;
    out->codes = codes;
    out->labels = g->labels ? labels : NULL;
}

/* ------------------------------------------------------ search state -- */
typedef struct {
    int ls, rs, ll, rl;
} cls_t; /* LabelClass window, label_classes.hpp:12-20 (adjacent flag unused by search) */

typedef struct {
    const orc_graph* g;
    const orc_graph* h;
    int* deg;
    int* left;
    int* right;
    int prune;
    int64_t goal, maxp, floor_size;
    struct timespec deadline;
    int unlimited;
    const volatile int32_t* cancel;
    /* incumbent (LocalIncumbent, search_core.hpp:21-36) */
    int best_n;
    int* best_pairs;
    int cur_n;
    int* cur_pairs;
    uint64_t nodes;
    int reason; /* 0 none, 1 timeout, 2 cancelled, 3 goal reached, 4 max reached */
    /* class arena: each recursion level owns a slice */
    cls_t* arena;
    int arena_top;
    orc_result* stats;
} ctx_t;

static int now_past(const struct timespec* dl) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec > dl->tv_sec || (t.tv_sec == dl->tv_sec && t.tv_nsec >= dl->tv_nsec);
}

static void set_deadline(ctx_t* c, double budget) {
    c->unlimited = budget >= 1e8; /* budget_deadline, solve.cpp:51-55 */
    clock_gettime(CLOCK_MONOTONIC, &c->deadline);
    if (!c->unlimited) {
        double s = (double)c->deadline.tv_sec + c->deadline.tv_nsec * 1e-9 + budget;
        c->deadline.tv_sec = (time_t)s;
        c->deadline.tv_nsec = (long)((s - (double)(time_t)s) * 1e9);
    }
}

/* SearchCtx::poll, search_core.hpp:109-115. */
static void poll(ctx_t* c) {
    if (c->cancel && *c->cancel) {
        c->reason = 2;
        return;
    }
    if ((c->nodes & 0xffu) == 1 && !c->unlimited && now_past(&c->deadline)) c->reason = 1;
}

/* compute_bound, label_classes.cpp:41-45. */
static int64_t bound_of(int64_t m, const cls_t* cs, int nc) {
    int64_t b = m;
    for (int i = 0; i < nc; ++i) b += cs[i].ll < cs[i].rl ? cs[i].ll : cs[i].rl;
    return b;
}

/* select_label_class, label_classes.cpp:47-67: min max(|L|,|R|), then min
 * min(|L|,|R|), then lowest left vertex id. */
static int select_class(const cls_t* cs, int nc, const int* left) {
    int best = -1, bmax = 0, bmin = 0, blow = 0;
    for (int i = 0; i < nc; ++i) {
        const cls_t* c = &cs[i];
        if (c->ll == 0 || c->rl == 0) continue;
        int mx = c->ll > c->rl ? c->ll : c->rl;
        int mn = c->ll < c->rl ? c->ll : c->rl;
        int low = left[c->ls];
        for (int j = 1; j < c->ll; ++j)
            if (left[c->ls + j] < low) low = left[c->ls + j];
        if (best == -1 || mx < bmax || (mx == bmax && mn < bmin) ||
            (mx == bmax && mn == bmin && low < blow))
            best = i, bmax = mx, bmin = mn, blow = low;
    }
    return best;
}

/* select_vertex, label_classes.cpp:69-78: max degree, lowest id on ties. */
static int select_vertex(const cls_t* c, const int* left, const int* deg) {
    int best = -1;
    for (int j = 0; j < c->ll; ++j) {
        int v = left[c->ls + j];
        if (best == -1 || deg[v] > deg[best] || (deg[v] == deg[best] && v < best)) best = v;
    }
    return best;
}

/* Stable partition of a window by adjacency code toward w (codes 0..3). */
static void partition4(int* buf, int start, int len, const orc_graph* g, int w, int cnt[4]) {
    int tmp[512];
    int* t = len <= 512 ? tmp : malloc(sizeof(int) * len);
    int pos[4];
    cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0;
    for (int j = 0; j < len; ++j) cnt[code(g, w, buf[start + j])]++;
    pos[0] = 0, pos[1] = cnt[0], pos[2] = pos[1] + cnt[1], pos[3] = pos[2] + cnt[2];
    for (int j = 0; j < len; ++j) t[pos[code(g, w, buf[start + j])]++] = buf[start + j];
    memcpy(buf + start, t, sizeof(int) * len);
    if (t != tmp) free(t);
}

/* filter_classes, label_classes.cpp:80-108: split every class by its code
 * toward (v,u), ascending code, dropping one-sided parts. Writes children to
 * out and returns their count. */
static int filter(ctx_t* c, const cls_t* cs, int nc, int v, int u, cls_t* out) {
    int k = 0;
    for (int i = 0; i < nc; ++i) {
        int lc[4], rc[4];
        partition4(c->left, cs[i].ls, cs[i].ll, c->g, v, lc);
        partition4(c->right, cs[i].rs, cs[i].rl, c->h, u, rc);
        int lo = 0, ro = 0;
        for (int code_ = 0; code_ < 4; ++code_) {
            if (lc[code_] && rc[code_]) {
                out[k].ls = cs[i].ls + lo;
                out[k].rs = cs[i].rs + ro;
                out[k].ll = lc[code_];
                out[k].rl = rc[code_];
                ++k;
            }
            lo += lc[code_];
            ro += rc[code_];
        }
    }
    c->stats->sum_splits += (uint64_t)nc;
    c->stats->children_built++;
    return k;
}

/* search_node, search_core.hpp:120-213. `cs` is this node's own copy of its
 * classes (placed in the arena by the caller); buffers are shared. */
static void search(ctx_t* c, cls_t* cs, int nc, int depth) {
    if (c->reason) return;
    ++c->nodes; /* :130 */
    poll(c);    /* :131 */
    if (c->reason) return;
    c->stats->sum_classes += (uint64_t)nc;
    if (depth > c->stats->max_depth) c->stats->max_depth = depth;
    if (c->arena_top > c->stats->max_stack_classes) c->stats->max_stack_classes = c->arena_top;

    /* inc.offer (:145): strict improvement over the local best only */
    if (c->cur_n > c->best_n) {
        c->best_n = c->cur_n;
        memcpy(c->best_pairs, c->cur_pairs, sizeof(int) * 2 * c->cur_n);
        if (c->goal > 0 && c->cur_n >= c->goal) { /* :147-150 */
            c->reason = 3;
            return;
        }
        if (c->prune && c->goal == 0 && c->cur_n >= c->maxp) { /* :151-154 */
            c->reason = 4;
            return;
        }
    }
    int64_t bound = bound_of(c->cur_n, cs, nc); /* :157 */
    int64_t inc = c->best_n > c->floor_size ? c->best_n : c->floor_size;
    int64_t thr = inc > c->goal - 1 ? inc : c->goal - 1;
    if (c->prune && bound <= thr) { /* :166 */
        c->stats->pruned_at_entry++;
        return;
    }
    int bi = select_class(cs, nc, c->left); /* :168 */
    if (bi < 0) return;
    cls_t* bd = &cs[bi];
    int v = select_vertex(bd, c->left, c->deg); /* :171 */
    for (int j = 0; j < bd->ll; ++j) /* :173-178 swap v out */
        if (c->left[bd->ls + j] == v) {
            int t = c->left[bd->ls + bd->ll - 1];
            c->left[bd->ls + bd->ll - 1] = v;
            c->left[bd->ls + j] = t;
            break;
        }
    bd->ll--;
    const int total = bd->rl;
    bd->rl--;
    int last_u = -1;
    cls_t* child = c->arena + c->arena_top;
    for (int it = 0; it < total && !c->reason; ++it) { /* :183-200 ascending u */
        int pos = -1;
        for (int j = 0; j < total; ++j) {
            int cand = c->right[bd->rs + j];
            if (cand > last_u && (pos == -1 || cand < c->right[bd->rs + pos])) pos = j;
        }
        int u = c->right[bd->rs + pos];
        last_u = u;
        c->right[bd->rs + pos] = c->right[bd->rs + total - 1];
        c->right[bd->rs + total - 1] = u;
        int k = filter(c, cs, nc, v, u, child);
        c->cur_pairs[2 * c->cur_n] = v;
        c->cur_pairs[2 * c->cur_n + 1] = u;
        c->cur_n++;
        c->arena_top += k;
        search(c, child, k, depth + 1);
        c->arena_top -= k;
        c->cur_n--;
    }
    bd->rl++; /* :201 */
    if (c->reason) return;
    if (bd->ll == 0) { /* :205-208 drop emptied class */
        cs[bi] = cs[nc - 1];
        nc--;
    }
    /* :210-212 v left unmatched: a counted node of its own, with its own copy */
    cls_t* rest = c->arena + c->arena_top;
    memcpy(rest, cs, sizeof(cls_t) * nc);
    c->arena_top += nc;
    search(c, rest, nc, depth + 1);
    c->arena_top -= nc;
}

static int check_graphs(const orc_graph* g, const orc_graph* h) {
    if (g->directed != h->directed) return -1;                /* solve.cpp:94 */
    if ((g->labels == NULL) != (h->labels == NULL)) return -1; /* label_classes.cpp:18-19 */
    return 0;
}

/* initial_classes, label_classes.cpp:8-39: one class of everything, or one
 * per label present on both sides in ascending label order. */
static int initial(ctx_t* c, cls_t* out) {
    const orc_graph* g = c->g;
    const orc_graph* h = c->h;
    if (!g->labels) {
        if (g->n == 0 || h->n == 0) return 0;
        for (int v = 0; v < g->n; ++v) c->left[v] = v;
        for (int u = 0; u < h->n; ++u) c->right[u] = u;
        out[0].ls = out[0].rs = 0;
        out[0].ll = g->n;
        out[0].rl = h->n;
        return 1;
    }
    int nc = 0, lp = 0, rp = 0;
    /* ascending distinct labels of G that also occur in H */
    int* labs = malloc(sizeof(int) * (g->n + 1));
    int nl = 0;
    for (int v = 0; v < g->n; ++v) {
        int lab = g->labels[v], seen = 0;
        for (int j = 0; j < nl; ++j) seen |= labs[j] == lab;
        if (!seen) labs[nl++] = lab;
    }
    for (int i = 1; i < nl; ++i)
        for (int j = i; j > 0 && labs[j - 1] > labs[j]; --j) {
            int t = labs[j];
            labs[j] = labs[j - 1];
            labs[j - 1] = t;
        }
    for (int i = 0; i < nl; ++i) {
        int lab = labs[i], inh = 0;
        for (int u = 0; u < h->n; ++u) inh |= h->labels[u] == lab;
        if (!inh) continue;
        int ls = lp, rs = rp;
        for (int v = 0; v < g->n; ++v)
            if (g->labels[v] == lab) c->left[lp++] = v;
        for (int u = 0; u < h->n; ++u)
            if (h->labels[u] == lab) c->right[rp++] = u;
        out[nc].ls = ls, out[nc].rs = rs, out[nc].ll = lp - ls, out[nc].rl = rp - rs;
        nc++;
    }
    free(labs);
    return nc;
}

/* One search over (g,h) in already-permuted ids: shared by solve and the
 * goal probes (solve.cpp:57-75 probe_goal, :92-129 solve_monitored). */
static void run_search(const orc_graph* g, const orc_graph* h, int prune, int64_t goal,
                       int64_t floor_size, const struct timespec* dl, int unlimited,
                       const volatile int32_t* cancel, orc_result* r, int* best_n,
                       int* best_pairs, uint64_t* nodes, int* reason) {
    ctx_t c;
    memset(&c, 0, sizeof(c));
    c.g = g;
    c.h = h;
    c.prune = prune;
    c.goal = goal;
    c.floor_size = floor_size;
    c.maxp = g->n < h->n ? g->n : h->n;
    c.deadline = *dl;
    c.unlimited = unlimited;
    c.cancel = cancel;
    c.stats = r;
    int n = g->n > h->n ? g->n : h->n;
    c.deg = malloc(sizeof(int) * (g->n + 1));
    for (int v = 0; v < g->n; ++v) c.deg[v] = orc_degree(g, v);
    c.left = malloc(sizeof(int) * (g->n + 1));
    c.right = malloc(sizeof(int) * (h->n + 1));
    c.best_pairs = best_pairs;
    c.cur_pairs = malloc(sizeof(int) * 2 * (n + 1));
    /* arena bound: every level holds at most min(nG,nH) classes, depth <= nG+1 */
    size_t cap = (size_t)(g->n + 2) * (size_t)(c.maxp + 1) + 4;
    c.arena = malloc(sizeof(cls_t) * cap);
    int nc = initial(&c, c.arena);
    c.arena_top = nc;
    search(&c, c.arena, nc, 0);
    *best_n = c.best_n;
    *nodes = c.nodes;
    *reason = c.reason;
    free(c.deg), free(c.left), free(c.right), free(c.cur_pairs), free(c.arena);
}

typedef struct {
    uint8_t* gc;
    int32_t* gl;
    uint8_t* hc;
    int32_t* hl;
    int32_t* pg;
    int32_t* ph;
    orc_graph g2, h2;
} ordered_t;

/* with_ordering, search_core.hpp:72-81: permute both inputs, solve, map back. */
static void order_begin(const orc_graph* g, const orc_graph* h, int order, ordered_t* o) {
    memset(o, 0, sizeof(*o));
    if (order == 0) {
        o->g2 = *g;
        o->h2 = *h;
        return;
    }
    o->pg = malloc(sizeof(int32_t) * (g->n + 1));
    o->ph = malloc(sizeof(int32_t) * (h->n + 1));
    orc_ordering(g, order, o->pg);
    orc_ordering(h, order, o->ph);
    o->gc = malloc((size_t)g->n * g->n + 1);
    o->hc = malloc((size_t)h->n * h->n + 1);
    o->gl = malloc(sizeof(int32_t) * (g->n + 1));
    o->hl = malloc(sizeof(int32_t) * (h->n + 1));
    permute_into(g, o->pg, o->gc, o->gl, &o->g2);
    permute_into(h, o->ph, o->hc, o->hl, &o->h2);
}

static void order_end(ordered_t* o, int32_t* pairs, int k) {
    if (o->pg) {
        int ng = o->g2.n, nh = o->h2.n;
        int32_t* ig = malloc(sizeof(int32_t) * (ng + 1));
        int32_t* ih = malloc(sizeof(int32_t) * (nh + 1));
        for (int v = 0; v < ng; ++v) ig[o->pg[v]] = v;
        for (int u = 0; u < nh; ++u) ih[o->ph[u]] = u;
        for (int i = 0; i < k; ++i) pairs[2 * i] = ig[pairs[2 * i]], pairs[2 * i + 1] = ih[pairs[2 * i + 1]];
        free(ig), free(ih);
    }
    free(o->gc), free(o->hc), free(o->gl), free(o->hl), free(o->pg), free(o->ph);
}

static double elapsed(const struct timespec* t0) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)(t.tv_sec - t0->tv_sec) + (t.tv_nsec - t0->tv_nsec) * 1e-9;
}

int orc_solve(const orc_graph* g, const orc_graph* h, const orc_options* o, orc_result* r) {
    memset(r, 0, sizeof(*r));
    if (check_graphs(g, h)) {
        r->status = -1;
        return -1;
    }
    if (o->budget_s <= 0) { /* solve.cpp:95 */
        r->status = 1;
        return 0;
    }
    struct timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    ordered_t ord;
    order_begin(g, h, o->order, &ord);
    ctx_t dlc;
    set_deadline(&dlc, o->budget_s);
    int best_n = 0, reason = 0;
    uint64_t nodes = 0;
    run_search(&ord.g2, &ord.h2, o->prune, 0, o->floor_size, &dlc.deadline, dlc.unlimited,
               o->cancel, r, &best_n, r->pairs, &nodes, &reason);
    order_end(&ord, r->pairs, best_n);
    r->size = best_n;
    r->nodes = nodes;
    r->status = reason == 1 ? 1 : reason == 2 ? 2 : 0; /* solve.cpp:118-126 */
    r->wall_s = elapsed(&t0);
    return 0;
}

/* solve_goal_directed, solve.cpp:131-168: goals n_G, n_G-1, ... over the
 * smaller graph; the first reachable goal is optimal. */
int orc_solve_goal_directed(const orc_graph* g, const orc_graph* h, const orc_options* o,
                            orc_result* r) {
    memset(r, 0, sizeof(*r));
    if (check_graphs(g, h)) {
        r->status = -1;
        return -1;
    }
    if (o->budget_s <= 0) {
        r->status = 1;
        return 0;
    }
    if (g->n > h->n) {
        int rc = orc_solve_goal_directed(h, g, o, r);
        for (int i = 0; i < r->size; ++i) {
            int32_t t = r->pairs[2 * i];
            r->pairs[2 * i] = r->pairs[2 * i + 1];
            r->pairs[2 * i + 1] = t;
        }
        return rc;
    }
    struct timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    ordered_t ord;
    order_begin(g, h, o->order, &ord);
    ctx_t dlc;
    set_deadline(&dlc, o->budget_s);
    int32_t* wit = malloc(sizeof(int32_t) * 2 * 258);
    int best = 0;
    r->status = 0;
    for (int64_t goal = ord.g2.n; goal >= 1; --goal) {
        int bn = 0, reason = 0;
        uint64_t nodes = 0;
        run_search(&ord.g2, &ord.h2, 1, goal, 0, &dlc.deadline, dlc.unlimited, o->cancel, r,
                   &bn, wit, &nodes, &reason);
        r->probes++;
        r->nodes += nodes;
        if (bn > best) {
            best = bn;
            memcpy(r->pairs, wit, sizeof(int32_t) * 2 * bn);
        }
        if (reason == 1 || reason == 2) {
            r->status = reason;
            break;
        }
        if (reason == 3) break; /* reached */
    }
    free(wit);
    order_end(&ord, r->pairs, best);
    r->size = best;
    r->wall_s = elapsed(&t0);
    return 0;
}

/* bound_jump_search, heuristics.cpp:114-185: raise the target (+1 or x2)
 * until a probe fails, then binary-search the bracket; finally recover a
 * witness for a caller-supplied lower bound. */
int orc_bound_jump(const orc_graph* g, const orc_graph* h, int current_best, int doubling,
                   const orc_options* o, orc_result* r) {
    memset(r, 0, sizeof(*r));
    if (check_graphs(g, h)) {
        r->status = -1;
        return -1;
    }
    if (o->budget_s <= 0) {
        r->status = 1;
        return 0;
    }
    struct timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    ordered_t ord;
    order_begin(g, h, o->order, &ord);
    ctx_t dlc;
    set_deadline(&dlc, o->budget_s);
    int64_t lower = current_best;
    int64_t upper = ord.g2.n < ord.h2.n ? ord.g2.n : ord.h2.n;
    int32_t* wit = malloc(sizeof(int32_t) * 2 * 258);
    int best = 0;
    r->status = 0;
    int stopped = 0;
#define PROBE(goal_, reached_)                                                                 \
    do {                                                                                       \
        int bn = 0, reason = 0;                                                                \
        uint64_t nodes = 0;                                                                    \
        run_search(&ord.g2, &ord.h2, 1, (goal_), 0, &dlc.deadline, dlc.unlimited, o->cancel, r, \
                   &bn, wit, &nodes, &reason);                                                 \
        r->probes++;                                                                           \
        r->nodes += nodes;                                                                     \
        if (bn > best) {                                                                       \
            best = bn;                                                                         \
            memcpy(r->pairs, wit, sizeof(int32_t) * 2 * bn);                                   \
        }                                                                                      \
        if (reason == 1 || reason == 2) {                                                      \
            r->status = reason;                                                                \
            stopped = 1;                                                                       \
        }                                                                                      \
        (reached_) = reason == 3;                                                              \
    } while (0)
    while (lower < upper) {
        int64_t target = doubling ? (lower * 2 > 1 ? lower * 2 : 1) : lower + 1;
        if (target > upper) target = upper;
        int reached;
        PROBE(target, reached);
        if (stopped) break;
        if (reached) lower = target;
        else upper = target - 1;
    }
    while (!stopped && lower < upper) {
        int64_t mid = lower + (upper - lower + 1) / 2;
        int reached;
        PROBE(mid, reached);
        if (stopped) break;
        if (reached) lower = mid;
        else upper = mid - 1;
    }
    if (!stopped && best < lower && lower > 0) {
        int reached;
        PROBE(lower, reached);
        (void)reached;
    }
#undef PROBE
    free(wit);
    order_end(&ord, r->pairs, best);
    r->size = best;
    r->wall_s = elapsed(&t0);
    return 0;
}

/* oracle::verify, oracle.cpp:8-24. */
int orc_verify(const orc_graph* g, const orc_graph* h, const int32_t* pairs, int k) {
    char* ug = calloc(g->n + 1, 1);
    char* uh = calloc(h->n + 1, 1);
    int ok = 1;
    for (int i = 0; i < k && ok; ++i) {
        int v = pairs[2 * i], u = pairs[2 * i + 1];
        if (v < 0 || v >= g->n || u < 0 || u >= h->n) {
            ok = -1;
            break;
        }
        if (ug[v] || uh[u]) ok = 0;
        ug[v] = uh[u] = 1;
        if ((g->labels == NULL) != (h->labels == NULL)) ok = 0;
        if (ok && g->labels && g->labels[v] != h->labels[u]) ok = 0;
    }
    for (int i = 0; i < k && ok == 1; ++i)
        for (int j = i + 1; j < k && ok == 1; ++j)
            if (code(g, pairs[2 * i], pairs[2 * j]) != code(h, pairs[2 * i + 1], pairs[2 * j + 1]))
                ok = 0;
    free(ug), free(uh);
    return ok;
}

/* mcs_bruteforce, oracle.cpp:33-86: for k from min side down, enumerate
 * k-subsets of V_G (lexicographic) and injections into V_H (ascending). */
static int bf_extend(const orc_graph* g, const orc_graph* h, const int* chosen, int k, int pos,
                     int32_t* part, char* used) {
    if (pos == k) return 1;
    int v = chosen[pos];
    for (int u = 0; u < h->n; ++u) {
        if (used[u]) continue;
        if (g->labels && g->labels[v] != h->labels[u]) continue;
        int ok = 1;
        for (int i = 0; i < pos && ok; ++i)
            if (code(g, part[2 * i], v) != code(h, part[2 * i + 1], u)) ok = 0;
        if (!ok) continue;
        part[2 * pos] = v;
        part[2 * pos + 1] = u;
        used[u] = 1;
        if (bf_extend(g, h, chosen, k, pos + 1, part, used)) return 1;
        used[u] = 0;
    }
    return 0;
}

static int bf_subsets(const orc_graph* g, const orc_graph* h, int* chosen, int nch, int next,
                      int k, int32_t* out) {
    if (nch == k) {
        char used[64] = {0};
        return bf_extend(g, h, chosen, k, 0, out, used);
    }
    for (int v = next; v < g->n; ++v) {
        if (g->n - v < k - nch) break;
        chosen[nch] = v;
        if (bf_subsets(g, h, chosen, nch + 1, v + 1, k, out)) return 1;
    }
    return 0;
}

int orc_bruteforce(const orc_graph* g, const orc_graph* h, int32_t* pairs_out) {
    int ceil_ = g->n < h->n ? g->n : h->n;
    if (ceil_ > 10) return -1;
    int chosen[16];
    for (int k = ceil_; k >= 1; --k)
        if (bf_subsets(g, h, chosen, 0, 0, k, pairs_out)) return k;
    return 0;
}

/* --------------------------------------------------------- restarts -- */
/* std::mt19937_64 (the segment draw of solve_with_restarts, restarts.cpp:213). */
typedef struct {
    uint64_t s[312];
    int i;
} mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
    m->s[0] = seed;
    for (int k = 1; k < 312; ++k)
        m->s[k] = 6364136223846793005ull * (m->s[k - 1] ^ (m->s[k - 1] >> 62)) + (uint64_t)k;
    m->i = 312;
}

static uint64_t mt64_next(mt64* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (m->s[k] & 0xFFFFFFFF80000000ull) | (m->s[(k + 1) % 312] & 0x7FFFFFFFull);
            uint64_t x = m->s[(k + 156) % 312] ^ (y >> 1);
            if (y & 1u) x ^= 0xB5026F5AA96619E9ull;
            m->s[k] = x;
        }
        m->i = 0;
    }
    uint64_t y = m->s[m->i++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* PositionKey (heuristics.hpp:77) without the depth field (it equals the
 * index): the iteration taken at each depth. */
typedef struct {
    int32_t* it;
    int len;
} pkey;

static pkey key_dup(const int32_t* it, int len, int extra) {
    pkey k;
    k.it = malloc(sizeof(int32_t) * (size_t)(len + extra + 1));
    if (len) memcpy(k.it, it, sizeof(int32_t) * (size_t)len);
    k.len = len;
    return k;
}

/* extend / successor, restarts.cpp:13-24 */
static pkey key_extend(const int32_t* it, int len, int x) {
    pkey k = key_dup(it, len, 1);
    k.it[k.len++] = x;
    return k;
}

static pkey key_successor(const int32_t* it, int len) {
    if (len == 0) {
        pkey k = key_dup(it, 0, 1);
        k.it[k.len++] = 2147483647;
        return k;
    }
    pkey k = key_dup(it, len, 0);
    k.it[len - 1] += 1;
    return k;
}

/* Segment (restarts.cpp:26-33): a frozen node's state plus the first
 * iteration still to run. */
typedef struct {
    int* left;
    int* right;
    cls_t* dom;
    int nd;
    int32_t* map; /* (v,u) pairs */
    int nmap;
    pkey pos;
    int from;
} rseg;

typedef struct {
    const orc_graph* g;
    const orc_graph* h;
    int* deg;
    int ng, nh;
    int prune;
    int64_t maxp, floor_size;
    struct timespec deadline;
    int unlimited;
    const volatile int32_t* cancel;
    double mult;
    int best_n;
    int32_t* best_pairs;
    int cur_n;
    int32_t* cur_pairs;
    uint64_t nodes, restarts, at;
    int rflag;
    int reason; /* 0 none, 1 timeout, 2 cancelled, 4 max reached */
    rseg* pool;
    int npool, cappool;
    pkey* rlo;
    pkey* rhi;
    int nranges, capranges;
} rctx;

static void r_add_range(rctx* c, pkey lo, pkey hi) {
    if (c->nranges == c->capranges) {
        c->capranges = c->capranges ? 2 * c->capranges : 64;
        c->rlo = realloc(c->rlo, sizeof(pkey) * (size_t)c->capranges);
        c->rhi = realloc(c->rhi, sizeof(pkey) * (size_t)c->capranges);
    }
    c->rlo[c->nranges] = lo;
    c->rhi[c->nranges] = hi;
    c->nranges++;
}

static void r_push(rctx* c, const int* left, const int* right, const cls_t* dom, int nd, const int32_t* pos,
                   int npos, int from) {
    if (c->npool == c->cappool) {
        c->cappool = c->cappool ? 2 * c->cappool : 64;
        c->pool = realloc(c->pool, sizeof(rseg) * (size_t)c->cappool);
    }
    rseg* s = &c->pool[c->npool++];
    s->left = malloc(sizeof(int) * (size_t)(c->ng + 1));
    s->right = malloc(sizeof(int) * (size_t)(c->nh + 1));
    memcpy(s->left, left, sizeof(int) * (size_t)c->ng);
    memcpy(s->right, right, sizeof(int) * (size_t)c->nh);
    s->dom = malloc(sizeof(cls_t) * (size_t)(nd + 1));
    memcpy(s->dom, dom, sizeof(cls_t) * (size_t)nd);
    s->nd = nd;
    s->map = malloc(sizeof(int32_t) * (size_t)(2 * c->cur_n + 1));
    memcpy(s->map, c->cur_pairs, sizeof(int32_t) * (size_t)(2 * c->cur_n));
    s->nmap = c->cur_n;
    s->pos = key_dup(pos, npos, 0);
    s->from = from;
}

static void r_poll(rctx* c) { /* RestartDriver::poll, restarts.cpp:61-66 */
    if (c->cancel && *c->cancel)
        c->reason = 2;
    else if ((c->nodes & 0xffu) == 1 && !c->unlimited && now_past(&c->deadline))
        c->reason = 1;
}

static int r_restart_due(const rctx* c) { /* restarts.cpp:68-72 */
    uint64_t delta = c->nodes - c->at;
    return (double)delta >= c->mult * (double)(c->at > 1 ? c->at : 1);
}

/* RestartDriver::node, restarts.cpp:80-190. `dom` is this node's own copy. */
static void r_node(rctx* c, cls_t* dom, int nd, int* left, int* right, const int32_t* pos, int npos, int from,
                   int is_root) {
    if (c->reason) return;
    ++c->nodes;
    r_poll(c);
    if (c->reason) return;
    if (c->mult > 0 && !c->rflag && r_restart_due(c)) { /* :87-91 */
        c->rflag = 1;
        ++c->restarts;
        c->at = c->nodes;
    }
    if (c->rflag) { /* :92-95 freeze this whole node */
        r_push(c, left, right, dom, nd, pos, npos, from);
        return;
    }
    if (c->cur_n > c->best_n) { /* :97 inc.offer */
        c->best_n = c->cur_n;
        memcpy(c->best_pairs, c->cur_pairs, sizeof(int32_t) * 2 * (size_t)c->cur_n);
        c->at = c->nodes;
    }
    int64_t bound = bound_of(c->cur_n, dom, nd);
    /* lo = from == 0 ? pos : extend(pos, from)   (:107) */
    pkey lo = from == 0 ? key_dup(pos, npos, 0) : key_extend(pos, npos, from);
    if (c->prune && c->cur_n >= c->maxp) { /* :108-111 */
        c->reason = 4;
        free(lo.it);
        return;
    }
    int64_t inc = c->best_n > c->floor_size ? c->best_n : c->floor_size;
    if (c->prune && bound <= inc) { /* :112-115 */
        if (is_root)
            r_add_range(c, lo, key_successor(pos, npos));
        else
            free(lo.it);
        return;
    }
    int bi = select_class(dom, nd, left); /* :117-121 */
    if (bi < 0) {
        if (is_root)
            r_add_range(c, lo, key_successor(pos, npos));
        else
            free(lo.it);
        return;
    }
    cls_t* entry = NULL; /* :124-125 entry state, for freezing */
    if (c->mult > 0) {
        entry = malloc(sizeof(cls_t) * (size_t)(nd + 1));
        memcpy(entry, dom, sizeof(cls_t) * (size_t)nd);
    }
    cls_t* bd = &dom[bi];
    int v = select_vertex(bd, left, c->deg); /* :128-134 */
    for (int j = 0; j < bd->ll; ++j)
        if (left[bd->ls + j] == v) {
            int t = left[bd->ls + bd->ll - 1];
            left[bd->ls + bd->ll - 1] = v;
            left[bd->ls + j] = t;
            break;
        }
    bd->ll--;
    const int total = bd->rl;
    const int n_iters = total + 1;
    bd->rl--;
    int last_u = -1;
    for (int skip = 0; skip < (from < total ? from : total); ++skip) { /* :140-147 */
        int next = -1;
        for (int j = 0; j < total; ++j) {
            int cand = right[bd->rs + j];
            if (cand > last_u && (next == -1 || cand < next)) next = cand;
        }
        last_u = next;
    }
    /* children get their own class copies; filter() partitions the windows */
    ctx_t fc;
    memset(&fc, 0, sizeof(fc));
    fc.g = c->g;
    fc.h = c->h;
    fc.left = left;
    fc.right = right;
    orc_result dummy;
    memset(&dummy, 0, sizeof(dummy));
    fc.stats = &dummy;
    cls_t* child = malloc(sizeof(cls_t) * (size_t)(4 * nd + 4));
    for (int it = from; it < n_iters; ++it) { /* :149-187 */
        if (it < total) {
            int pj = -1;
            for (int j = 0; j < total; ++j) {
                int cand = right[bd->rs + j];
                if (cand > last_u && (pj == -1 || cand < right[bd->rs + pj])) pj = j;
            }
            int u = right[bd->rs + pj];
            last_u = u;
            right[bd->rs + pj] = right[bd->rs + total - 1];
            right[bd->rs + total - 1] = u;
            int k = filter(&fc, dom, nd, v, u, child);
            cls_t* cc = malloc(sizeof(cls_t) * (size_t)(k + 1));
            memcpy(cc, child, sizeof(cls_t) * (size_t)k);
            c->cur_pairs[2 * c->cur_n] = v;
            c->cur_pairs[2 * c->cur_n + 1] = u;
            c->cur_n++;
            pkey ep = key_extend(pos, npos, it);
            r_node(c, cc, k, left, right, ep.it, ep.len, 0, 0);
            free(ep.it);
            free(cc);
            c->cur_n--;
        } else { /* :165-175 v left unmatched */
            bd->rl++;
            cls_t* rest = malloc(sizeof(cls_t) * (size_t)(nd + 1));
            memcpy(rest, dom, sizeof(cls_t) * (size_t)nd);
            int nr = nd;
            if (rest[bi].ll == 0) {
                rest[bi] = rest[nr - 1];
                nr--;
            }
            pkey ep = key_extend(pos, npos, it);
            r_node(c, rest, nr, left, right, ep.it, ep.len, 0, 0);
            free(ep.it);
            free(rest);
            bd->rl--;
        }
        if (c->rflag || c->reason) { /* :176-186 */
            if (c->rflag) {
                r_push(c, left, right, entry, nd, pos, npos, it + 1);
                r_add_range(c, lo, key_extend(pos, npos, it));
                lo.it = NULL;
            }
            bd->rl++;
            free(lo.it);
            free(entry);
            free(child);
            return;
        }
    }
    bd->rl++;
    free(entry);
    free(child);
    if (is_root)
        r_add_range(c, lo, key_successor(pos, npos));
    else
        free(lo.it);
}

/* solve_with_restarts, restarts.cpp:195-246. */
int orc_solve_with_restarts(const orc_graph* g, const orc_graph* h, const orc_options* o, uint64_t seed,
                            double multiplier, orc_result* r, uint64_t* restarts, int32_t* ranges_out,
                            int64_t ranges_cap, int64_t* ranges_len) {
    memset(r, 0, sizeof(*r));
    if (restarts) *restarts = 0;
    if (ranges_len) *ranges_len = 0;
    if (check_graphs(g, h)) {
        r->status = -1;
        return -1;
    }
    if (o->budget_s <= 0) {
        r->status = 1;
        return 0;
    }
    struct timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    ordered_t ord;
    order_begin(g, h, o->order, &ord);
    rctx c;
    memset(&c, 0, sizeof(c));
    c.g = &ord.g2;
    c.h = &ord.h2;
    c.ng = ord.g2.n;
    c.nh = ord.h2.n;
    c.prune = o->prune;
    c.maxp = c.ng < c.nh ? c.ng : c.nh;
    c.floor_size = o->floor_size;
    c.cancel = o->cancel;
    c.mult = multiplier;
    {
        ctx_t dl;
        set_deadline(&dl, o->budget_s);
        c.deadline = dl.deadline;
        c.unlimited = dl.unlimited;
    }
    c.deg = malloc(sizeof(int) * (size_t)(c.ng + 1));
    for (int v = 0; v < c.ng; ++v) c.deg[v] = orc_degree(c.g, v);
    c.best_pairs = r->pairs;
    c.cur_pairs = malloc(sizeof(int32_t) * (size_t)(2 * (c.ng + c.nh) + 2));
    /* the initial segment (restarts.cpp:214-216) */
    {
        ctx_t ic;
        memset(&ic, 0, sizeof(ic));
        ic.g = c.g;
        ic.h = c.h;
        int* left = malloc(sizeof(int) * (size_t)(c.ng + 1));
        int* right = malloc(sizeof(int) * (size_t)(c.nh + 1));
        ic.left = left;
        ic.right = right;
        cls_t* init = malloc(sizeof(cls_t) * (size_t)(c.ng + 1));
        int nc = initial(&ic, init);
        r_push(&c, left, right, init, nc, NULL, 0, 0);
        free(left), free(right), free(init);
    }
    mt64 rng;
    mt64_seed(&rng, seed);
    while (c.npool > 0 && !c.reason) { /* :218-228 */
        int idx = c.npool == 1 ? 0 : (int)(mt64_next(&rng) % (uint64_t)c.npool);
        rseg s = c.pool[idx];
        memmove(&c.pool[idx], &c.pool[idx + 1], sizeof(rseg) * (size_t)(c.npool - idx - 1));
        c.npool--;
        c.rflag = 0;
        memcpy(c.cur_pairs, s.map, sizeof(int32_t) * 2 * (size_t)s.nmap);
        c.cur_n = s.nmap;
        r_node(&c, s.dom, s.nd, s.left, s.right, s.pos.it, s.pos.len, s.from, 1);
        free(s.left), free(s.right), free(s.dom), free(s.map), free(s.pos.it);
    }
    for (int i = 0; i < c.npool; ++i)
        free(c.pool[i].left), free(c.pool[i].right), free(c.pool[i].dom), free(c.pool[i].map),
            free(c.pool[i].pos.it);
    free(c.pool);
    int64_t w = 0;
    for (int i = 0; i < c.nranges; ++i)
        for (int side = 0; side < 2; ++side) {
            const pkey* k = side ? &c.rhi[i] : &c.rlo[i];
            if (ranges_out && w < ranges_cap) ranges_out[w] = k->len;
            ++w;
            for (int d = 0; d < k->len; ++d) {
                if (ranges_out && w < ranges_cap) ranges_out[w] = k->it[d];
                ++w;
            }
        }
    if (ranges_len) *ranges_len = w;
    for (int i = 0; i < c.nranges; ++i) free(c.rlo[i].it), free(c.rhi[i].it);
    free(c.rlo), free(c.rhi);
    order_end(&ord, r->pairs, c.best_n);
    r->size = c.best_n;
    r->nodes = c.nodes;
    r->status = c.reason == 1 ? 1 : c.reason == 2 ? 2 : 0;
    r->probes = (uint64_t)c.nranges; /* (visited_ranges travels in probes) */
    if (restarts) *restarts = c.restarts;
    r->wall_s = elapsed(&t0);
    free(c.deg), free(c.cur_pairs);
    return 0;
}
