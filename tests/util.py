"""Shared fixtures mirroring the reference's tests/test_util.hpp."""
import oracle as O
import paper_1908_06418_b200 as M

DENSITIES = (0.2, 0.5, 0.8)


def random_pairs(count, n_lo, n_hi, seed0):
    """testutil::random_pairs (test_util.hpp:30-40): sizes cycle n_lo..n_hi,
    densities cycle {.2,.5,.8}, seed = seed0 + 977 i, H seed + 1."""
    out = []
    for i in range(count):
        n = n_lo + (i % (n_hi - n_lo + 1) if n_hi > n_lo else 0)
        d = DENSITIES[i % 3]
        s = seed0 + 977 * i
        out.append((n, d, s))
    return out


def pair(n, d, s, directed=False, labels=0, seed_h=None):
    """(product Graph G, product Graph H, oracle G, oracle H) for the same seeds."""
    sh = s + 1 if seed_h is None else seed_h
    g = M.random_graph(n, d, s, directed, labels)
    h = M.random_graph(n, d, sh, directed, labels)
    return g, h, to_oracle(g), to_oracle(h)


def to_oracle(g):
    return O.G(g.n(), g.codes.copy(), g.directed(), None if g.labels is None else g.labels.copy())


def diamond():
    return M.from_edge_list(4, [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3)])


def k4():
    return M.from_edge_list(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
