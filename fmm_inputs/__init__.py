"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle tests, the GPU tests and bench.py.  It holds
none of the FMM's arithmetic: no keys, no addresses, no lists, no expansions.  It
only draws points with numpy's PCG64 and places them with plain geometry:

* regular-polygon point picking of the paper's Fig. 12: an edge
  isosceles triangle chosen by a uniform selector z, a uniform point of the
  rectangle formed by its two rearranged halves;
* the septree domain (reading D8) is the union of the 7^L leaf hexagons of the
  island; leaf hexagon centres are placed with the paper's polar CellCenter
  formula in floating point -- a sampling recipe only, never
  compared against anything;
* config 5's "rejected if outside" test (reading D8) = "inside the hexagon of
  the nearest island leaf centre" (a k-d tree query plus a hexagon test).

Draw order per config: source positions, source strengths, then target
positions (distinct-target configs only).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SQRT3 = math.sqrt(3.0)


@dataclass
class Workload:
    name: str
    tiling: str            # "quad" | "sept" | "triq"
    depth: int
    p: int
    root_x: float
    root_y: float
    root_size: float
    n: int
    m: int
    self_mode: bool
    seed: int
    dist: str = "uniform"  # "uniform" | "clustered"
    note: str = ""
    extra: dict = field(default_factory=dict)

    def scaled(self, n: int, m: int | None = None, name: str | None = None) -> "Workload":
        """Same domain / tree / p, fewer points (parity cases the oracle finishes in seconds)."""
        w = Workload(**{**self.__dict__})
        w.n = n
        w.m = n if self.self_mode else (m if m is not None else n)
        w.name = name or f"{self.name}@{n}"
        return w


def sept_r0_equal_area() -> float:
    """circumradius of the hexagon of area 1: (3 sqrt3 / 2) R0^2 = 1."""
    return math.sqrt(2.0 / (3.0 * SQRT3))


def _tri_frame(side: float):
    """triangle with vertices 0, side, side*e^{i pi/3}: centroid and circumradius."""
    return side / 2.0, side * SQRT3 / 6.0, side / SQRT3


_C2 = _tri_frame(1.0)
_C4T = _tri_frame(2.0 * 3.0 ** -0.25)

WORKLOADS = {
    "C1": Workload("C1", "sept", 3, 20, 0.0, 0.0, 1.0, 4096, 4096, False, 0,
                   note="septree L3, R0=1, 4096/4096 distinct, p=20"),
    "C2": Workload("C2", "triq", 5, 20, _C2[0], _C2[1], _C2[2], 65536, 65536, True, 1,
                   note="triangle-quadtree L5, triangle 0,1,e^{i pi/3}, 65536 self, p=20"),
    "C3": Workload("C3", "sept", 6, 16, 0.0, 0.0, 1.0, 4194304, 4194304, False, 2,
                   note="septree L6, R0=1, 4.19M/4.19M distinct, p=16"),
    "C4q": Workload("C4q", "quad", 9, 24, 0.0, 0.0, 1.0, 16777216, 16777216, True, 3,
                    note="quadtree L9 unit square, 16.8M self, p=24"),
    "C4s": Workload("C4s", "sept", 6, 24, 0.0, 0.0, sept_r0_equal_area(), 16777216, 16777216, True, 3,
                    note="septree L6 island of area 1, 16.8M self, p=24"),
    "C4t": Workload("C4t", "triq", 9, 24, _C4T[0], _C4T[1], _C4T[2], 16777216, 16777216, True, 3,
                    note="triangle-quadtree L9 triangle of area 1, 16.8M self, p=24"),
    "C5": Workload("C5", "sept", 7, 20, 0.0, 0.0, 1.0, 16777216, 16777216, True, 4, dist="clustered",
                   note="septree L7 R0=1, 64 Gaussian clusters, 16.8M self, u~N(0,1), p=20"),
}


# ---------------------------------------------------------------- polygon point picking (Fig. 12)
def polygon_points(rng: np.random.Generator, n: int, nsides: int, circumradius: float, angle0: float):
    """n uniform points in the regular polygon (centre 0) with vertices at angle0 + 2 pi k / nsides.

    Each edge forms an isosceles triangle with the centre; its two halves (split by
    the apothem) are rearranged into a rectangle (half-edge x apothem).  (s, t) is
    uniform in that rectangle, z selects the edge triangle (Fig. 12)."""
    s = rng.random(n)
    t = rng.random(n)
    z = rng.integers(0, nsides, n)
    half_edge = circumradius * math.sin(math.pi / nsides)
    apothem = circumradius * math.cos(math.pi / nsides)
    left = s > t  # lower-right half of the rectangle -> the other half of the triangle
    X = np.where(left, (s - 1.0) * half_edge, s * half_edge)
    Y = np.where(left, (1.0 - t) * apothem, t * apothem)
    # local frame: apothem direction of edge k is at angle0 + (2k+1) pi / nsides
    phi = angle0 + (2 * z + 1) * math.pi / nsides
    # local (X along the edge, Y towards the edge) -> rotate so +Y points along phi
    c, sn = np.cos(phi), np.sin(phi)
    px = Y * c + X * sn
    py = Y * sn - X * c
    return px, py


# ---------------------------------------------------------------- septree island sampling (D8)
def sept_leaf_r(R0: float, L: int) -> float:
    return R0 / (7.0 ** (L // 2) * (math.sqrt(7.0) if L % 2 else 1.0))


def island_leaf_centres(R0: float, L: int) -> np.ndarray:
    """Centres of all 7^L leaf hexagons, leaf order, by the polar formula P:192-197 (float64)."""
    r = sept_leaf_r(R0, L)
    theta = math.atan(SQRT3 / 2.0)
    idx = np.arange(7 ** L, dtype=np.int64)
    x = np.zeros(len(idx))
    y = np.zeros(len(idx))
    for i in range(1, L + 1):
        ti = (idx // 7 ** (L - i)) % 7
        j = L - i
        th = j * theta + ti * math.pi / 3.0 - math.pi / 6.0
        R = r * SQRT3 * math.sqrt(7.0) ** j
        nz = ti != 0
        x = x + np.where(nz, R * np.cos(th), 0.0)
        y = y + np.where(nz, R * np.sin(th), 0.0)
    return np.stack([x, y], axis=1)


def sample_island(rng, n, R0, L, centres=None):
    """uniform over the island: uniform leaf, uniform point in its hexagon (flat-top, circumradius r)."""
    if centres is None:
        centres = island_leaf_centres(R0, L)
    leaf = rng.integers(0, len(centres), n)
    px, py = polygon_points(rng, n, 6, sept_leaf_r(R0, L), 0.0)
    return np.stack([centres[leaf, 0] + px, centres[leaf, 1] + py], axis=1)


def inside_island(xy, R0, L, centres, kdtree=None):
    """inside the flat-top hexagon of the nearest island leaf centre (with a 1e-9 r inner margin)."""
    from scipy.spatial import cKDTree

    kd = kdtree if kdtree is not None else cKDTree(centres)
    _, nearest = kd.query(xy, k=1)
    r = sept_leaf_r(R0, L)
    d = xy - centres[nearest]
    ax, ay = np.abs(d[:, 0]), np.abs(d[:, 1])
    m = 1e-9 * r
    return (ay <= 0.5 * SQRT3 * r - m) & (SQRT3 * ax + ay <= SQRT3 * r - m)


# ---------------------------------------------------------------- per-tiling uniform sampling
def _uniform_positions(w: Workload, rng, n, centres=None):
    if w.tiling == "quad":
        u = rng.random((n, 2))
        return np.stack([w.root_x + u[:, 0] * w.root_size, w.root_y + u[:, 1] * w.root_size], axis=1)
    if w.tiling == "triq":
        px, py = polygon_points(rng, n, 3, w.root_size, math.pi / 2.0)
        return np.stack([w.root_x + px, w.root_y + py], axis=1)
    xy = sample_island(rng, n, w.root_size, w.depth, centres)
    return xy + np.array([w.root_x, w.root_y])


def _clustered_positions(w: Workload, rng, n, centres):
    """64 isotropic Gaussians, centres uniform over the island, sigma log-uniform in
    [0.005, 0.05] (x R0), n/64 points each, rejected if outside the island (D8)."""
    from scipy.spatial import cKDTree

    kd = cKDTree(centres)
    ncl = int(w.extra.get("clusters", 64))
    cen = sample_island(rng, ncl, w.root_size, w.depth, centres)
    sig = np.exp(rng.uniform(math.log(0.005), math.log(0.05), ncl)) * w.root_size
    per = [n // ncl + (1 if k < n % ncl else 0) for k in range(ncl)]
    out = []
    for k in range(ncl):
        need, got = per[k], []
        while need > 0:
            cand = cen[k] + sig[k] * rng.standard_normal((max(2 * need, 64), 2))
            ok = inside_island(cand, w.root_size, w.depth, centres, kd)
            cand = cand[ok][:need]
            got.append(cand)
            need -= len(cand)
        out.append(np.concatenate(got))
    return np.concatenate(out) + np.array([w.root_x, w.root_y])


def generate(w: Workload):
    """-> dict(src_xy (n,2) f64, u (n,) f64, tgt_xy (m,2) f64 or None in self mode)."""
    rng = np.random.Generator(np.random.PCG64(w.seed))
    centres = island_leaf_centres(w.root_size, w.depth) if w.tiling == "sept" else None
    if w.dist == "clustered":
        src = _clustered_positions(w, rng, w.n, centres)
        u = rng.standard_normal(w.n)
    else:
        src = _uniform_positions(w, rng, w.n, centres)
        u = rng.uniform(-1.0, 1.0, w.n)
    tgt = None
    if not w.self_mode:
        tgt = (_clustered_positions(w, rng, w.m, centres) if w.dist == "clustered"
               else _uniform_positions(w, rng, w.m, centres))
    return {"src_xy": np.ascontiguousarray(src, np.float64), "u": np.ascontiguousarray(u, np.float64),
            "tgt_xy": None if tgt is None else np.ascontiguousarray(tgt, np.float64)}


def get(name: str) -> Workload:
    return WORKLOADS[name]


# ---------------------------------------------------------------- section-9 sweeps (NEXT-1)
# "S_opt uniformly random source and target points fitted to each cell ... to modify the total
# number of source and target points, the total number of occupied cells is reduced".
# Leaf cells are enumerated geometrically (a sampling recipe; no CellIndex arithmetic here).
def s_opt(tiling: str, p: int) -> float:
    """Table 2 optimal points per cell at N = M: p (P2'/P4)^0.5."""
    return p * {"quad": 116.0 / 27.0, "sept": 308.0 / 42.0, "triq": 164.0 / 39.0}[tiling] ** 0.5


def leaf_cells(tiling: str, depth: int, root_x: float, root_y: float, root_size: float):
    """-> (centres (K, 2), circumradius, nsides, angle0 (K,)) of every leaf polygon."""
    if tiling == "quad":
        n = 2 ** depth
        s = root_size / n
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        c = np.stack([root_x + (i.ravel() + 0.5) * s, root_y + (j.ravel() + 0.5) * s], axis=1)
        return c, s / math.sqrt(2.0), 4, np.full(len(c), math.pi / 4.0)
    if tiling == "sept":
        c = island_leaf_centres(root_size, depth) + np.array([root_x, root_y])
        return c, sept_leaf_r(root_size, depth), 6, np.zeros(len(c))
    # triangle: midpoint subdivision of the upright root (centroid root_x, root_y, circumradius)
    R = root_size
    v = np.array([[root_x + R * math.cos(math.pi / 2 + 2 * math.pi * k / 3),
                   root_y + R * math.sin(math.pi / 2 + 2 * math.pi * k / 3)] for k in range(3)])[None]
    for _ in range(depth):
        a, b, c3 = v[:, 0], v[:, 1], v[:, 2]
        ab, bc, ca = 0.5 * (a + b), 0.5 * (b + c3), 0.5 * (c3 + a)
        v = np.concatenate([np.stack(t, axis=1) for t in ((a, ab, ca), (ab, b, bc), (ca, bc, c3), (bc, ca, ab))])
    cen = v.mean(axis=1)
    up = v[:, 0, 1] > cen[:, 1]  # first vertex above the centroid: upright
    return cen, R * 2.0 ** -depth, 3, np.where(up, math.pi / 2.0, -math.pi / 2.0)


def sweep_generate(tiling: str, depth: int, root_x: float, root_y: float, root_size: float, per_cell: int,
                   n_cells: int, seed: int):
    """n_cells occupied leaves (a seeded random subset), per_cell uniform sources and as many
    distinct uniform targets in each; strengths U[-1, 1).  -> dict like generate()."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cen, rad, ns, ang = leaf_cells(tiling, depth, root_x, root_y, root_size)
    occ = rng.choice(len(cen), size=min(n_cells, len(cen)), replace=False)

    def pts():
        cell = np.repeat(occ, per_cell)
        px, py = polygon_points(rng, len(cell), ns, rad, 0.0)
        a = ang[cell]  # polygon_points puts a vertex at angle 0: rotate to the cell's orientation
        ca, sa = np.cos(a), np.sin(a)
        return np.stack([cen[cell, 0] + ca * px - sa * py, cen[cell, 1] + sa * px + ca * py], axis=1)

    src = pts()
    u = rng.uniform(-1.0, 1.0, len(src))
    tgt = pts()
    return {"src_xy": np.ascontiguousarray(src, np.float64), "u": np.ascontiguousarray(u, np.float64),
            "tgt_xy": np.ascontiguousarray(tgt, np.float64)}
