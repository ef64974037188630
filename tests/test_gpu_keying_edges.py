"""Keying (CellIndex) on constructed edge points, GPU against the oracle, bit-exact (-m gpu).

Random inputs almost never land on the places where the keying has to break a tie, so these
points are built on them:
  * quadtree: the grid lines x, y = k 2^-L (Morton P:79, reading D7) including the root's far
    edge x = 1 / y = 1 (clamped to the last cell, D11) and one ulp either side of them, and points
    one ulp outside the root;
  * septree: the vertices and edge midpoints of leaf hexagons, where two or three lattice points
    are equidistant (nearest-lattice selection over four candidates; strict <, first
    candidate wins, D11), on interior and island-boundary leaves, including points that fall
    outside the island;
  * triangle-quadtree: every vertex of the leaf subdivision and the midpoints of its edges (the
    nearest-of-4 descent), the root edges, and points pushed off the root by 0.5 and 2
    times the 1e-12 R0 closure slack (D11).
Both sides evaluate the same binary64 expression sequence (D11), so the keys of every point --
and which points are out of the domain -- must agree exactly."""
import math

import numpy as np
import pytest

import fmm_inputs as fi

pytestmark = pytest.mark.gpu

H = 0.8660254037844386  # sqrt(3)/2 rounded to binary64 (D11)


def gpu_keys(w, xy):
    import torch

    from paper_1204_3105_b200 import Config, Tree, X

    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    t = Tree(cfg, torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.ones(len(xy), dtype=torch.float64).cuda())
    k = t.export(X.SRC_KEYS)
    t.close()
    return k


def oracle_keys(w, xy):
    import oracle

    cfg = oracle.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    return oracle.keys_all(cfg, xy)


def compare(w, xy):
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    K = (7 if w.tiling == "sept" else 4) ** w.depth
    g = gpu_keys(w, xy)
    o = oracle_keys(w, xy)
    o_ood = o == 0xFFFFFFFF
    assert np.array_equal(g == K, o_ood), "out-of-domain points differ"
    assert np.array_equal(g[~o_ood], o[~o_ood])
    return o_ood.sum()


def ulp_ring(pts):
    """each point and its one-ulp neighbours in x and y"""
    out = [pts]
    for ax in (0, 1):
        for d in (-np.inf, np.inf):
            q = pts.copy()
            q[:, ax] = np.nextafter(q[:, ax], d)
            out.append(q)
    return np.concatenate(out)


@pytest.mark.parametrize("name", ["C4q"])
def test_quad_grid_lines(name):
    w = fi.get(name)
    n = 2 ** w.depth
    ks = np.array([0, 1, 2, 3, n // 2 - 1, n // 2, n // 2 + 1, n - 2, n - 1, n])
    g = np.array([(i / n, j / n) for i in ks for j in ks])  # exact in binary64
    rng = np.random.default_rng(0)
    lines = np.concatenate([np.stack([np.full(200, k / n), rng.random(200)], 1) for k in ks] +
                           [np.stack([rng.random(200), np.full(200, k / n)], 1) for k in ks])
    pts = ulp_ring(np.concatenate([g, lines]))
    extra = np.array([[1.0, 1.0], [0.0, 0.0], [-0.0, 0.5], [0.5, -0.0], [-1e-300, 0.5], [0.5, 1.0 + 2.0 ** -52]])
    ood = compare(w, np.concatenate([pts, extra]))
    assert ood > 0  # the one-ulp-outside points are out of the domain on both sides


@pytest.mark.parametrize("name", ["C1", "C4s"])
def test_septree_hexagon_vertices_and_edges(name):
    import oracle

    w = fi.get(name)
    L = w.depth
    cfg = oracle.config(w.tiling, L, w.p, w.root_x, w.root_y, w.root_size, True)
    K = 7 ** L
    rng = np.random.default_rng(1)
    leaves = np.unique(np.concatenate([np.arange(min(K, 400)), rng.choice(K, size=min(K, 1200), replace=False),
                                       K - 1 - np.arange(min(K, 400))]))
    r = w.root_size / (7 ** (L // 2) * (math.sqrt(7.0) if L % 2 else 1.0))  # leaf circumradius (D8)
    cen = np.array([oracle.cell_center(cfg, L, int(c)) for c in leaves])
    vx = np.array([1.0, 0.5, -0.5, -1.0, -0.5, 0.5])
    vy = np.array([0.0, H, H, 0.0, -H, -H])
    verts = (cen[:, None, :] + r * np.stack([vx, vy], -1)[None]).reshape(-1, 2)
    mids = (cen[:, None, :] + 0.5 * r * np.stack([vx + np.roll(vx, -1), vy + np.roll(vy, -1)], -1)[None]).reshape(-1, 2)
    pts = ulp_ring(np.concatenate([verts, mids]))
    compare(w, pts)


@pytest.mark.parametrize("name", ["C2", "C4t"])
def test_triangle_subdivision_vertices_and_edges(name):
    w = fi.get(name)
    L = w.depth
    R = w.root_size
    # root vertices of the upright triangle (centroid root_x, root_y, circumradius R)
    A = np.array([w.root_x + R * math.cos(math.pi / 2 + 2 * math.pi * k / 3) for k in range(3)])
    B = np.array([w.root_y + R * math.sin(math.pi / 2 + 2 * math.pi * k / 3) for k in range(3)])
    V = np.stack([A, B], 1)
    n = 2 ** L
    step = max(1, n // 128)
    ii, jj = np.meshgrid(np.arange(0, n + 1, step), np.arange(0, n + 1, step), indexing="ij")
    keep = ii + jj <= n
    a, b = ii[keep] / n, jj[keep] / n
    lat = V[0] + a[:, None] * (V[1] - V[0]) + b[:, None] * (V[2] - V[0])
    h = 1.0 / n
    mids = np.concatenate([lat + 0.5 * h * (V[1] - V[0]), lat + 0.5 * h * (V[2] - V[0]),
                           lat + 0.5 * h * (V[2] - V[1])])
    # the root edges, pushed outward by 0.5 and 2 slack widths (1e-12 R0, D11)
    t = np.linspace(0.0, 1.0, 257)
    edges, normals = [], []
    for e in range(3):
        p0, p1 = V[e], V[(e + 1) % 3]
        mid = 0.5 * (p0 + p1)
        nrm = mid - np.array([w.root_x, w.root_y])
        nrm /= np.linalg.norm(nrm)
        seg = p0 + t[:, None] * (p1 - p0)
        edges.append(seg)
        normals.append(np.repeat(nrm[None], len(t), 0))
    edges, normals = np.concatenate(edges), np.concatenate(normals)
    pushed = np.concatenate([edges + 0.5e-12 * R * normals, edges + 2e-12 * R * normals])
    pts = np.concatenate([ulp_ring(lat), mids, ulp_ring(edges), pushed])
    ood = compare(w, pts)
    assert ood >= len(t) * 3 - 3  # the points 2 slack widths outside (corners may differ) are out on both sides
