"""Oracle pins (-m "not gpu") for the NEXT-4 regular-polygon point picking
(Fig. 12; reading D22): oracle.sample_cells draws per_cell
points uniformly in each leaf polygon from counter-based draws.

Pinned against things other than the sampler itself:
* CellIndex (independently pinned in test_oracle_tiling.py): every point lies in its cell;
* closed forms of the uniform distribution on a regular n-gon of circumradius R:
  mean = centre, E|x - c|^2 = (R^2 / 6)(2 + cos(2 pi / n)) (sum over the n isosceles triangles
  of the triangle second moment (|v1|^2 + |v2|^2 + |v1 + v2|^2) / 12 with v0 = 0), equal mass
  1 / (2n) in each of the 2n half-triangles, and mass pi rho^2 / (n a b) inside a small
  disc of radius rho about the centre;
* the support: no point beyond R, points reach within 1% of R;
* the draws: bit balance, uniform mean / variance, lag-1 correlation, counter addressing."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
import oracle as orc

SQ3 = math.sqrt(3.0)


def cfg_for(tiling, L):
    if tiling == "quad":
        return orc.config("quad", L, 4, 0.0, 0.0, 1.0)
    if tiling == "sept":
        return orc.config("sept", L, 4, 0.0, 0.0, 1.0)
    w = fi.get("C2")
    return orc.config("triq", L, 4, w.root_x, w.root_y, w.root_size)


def polygon(cfg):
    """(nsides, circumradius) of a leaf, from the tiling's definition (D7, D8, reading of P:358)"""
    L = cfg.depth
    if cfg.tiling == 0:
        return 4, cfg.root_size * 2.0 ** -L / math.sqrt(2.0)
    if cfg.tiling == 1:
        return 6, fi.sept_leaf_r(cfg.root_size, L)
    return 3, cfg.root_size * 2.0 ** -L


def leaf_centres(cfg, cells):
    return np.array([orc.cell_center(cfg, cfg.depth, int(c)) for c in cells])


@pytest.mark.parametrize("tiling,L", [("quad", 3), ("sept", 2), ("sept", 3), ("triq", 3), ("quad", 5)])
def test_points_lie_in_their_cells(tiling, L):
    cfg = cfg_for(tiling, L)
    K = orc.num_cells(cfg, L)
    xy, u = orc.sample_cells(cfg, None, 40, seed=11)
    keys = orc.keys(cfg, xy)
    assert np.array_equal(keys.astype(np.int64), np.repeat(np.arange(K), 40))
    assert np.all((u >= -1.0) & (u < 1.0))


@pytest.mark.parametrize("tiling", ["quad", "sept", "triq"])
def test_uniform_on_the_polygon(tiling):
    cfg = cfg_for(tiling, 3)
    K = orc.num_cells(cfg, 3)
    cells = np.array([1, K // 2, K - 1] + ([int(K * 0.37) + 2] if tiling != "quad" else []), np.int64)
    pc = 60000
    xy, _ = orc.sample_cells(cfg, cells, pc, seed=5, want_u=False)
    n, R = polygon(cfg)
    a, b = R * math.sin(math.pi / n), R * math.cos(math.pi / n)
    cen = leaf_centres(cfg, cells)
    for i, c in enumerate(cells):
        d = xy[i * pc:(i + 1) * pc] - cen[i]
        r2 = (d ** 2).sum(1)
        # support: inside the circumcircle, and reaching it
        assert r2.max() <= R * R * (1 + 1e-12)
        assert math.sqrt(r2.max()) > 0.99 * R
        # mean = centre; E r^2 closed form
        for k in range(2):
            assert abs(d[:, k].mean()) < 5 * d[:, k].std() / math.sqrt(pc)
        m2 = R * R / 6.0 * (2.0 + math.cos(2 * math.pi / n))
        assert abs(r2.mean() - m2) < 5 * r2.std() / math.sqrt(pc), (r2.mean(), m2)
        # mass pi rho^2 / (n a b) in the disc of radius b / 2
        frac = (r2 < (0.5 * b) ** 2).mean()
        p0 = math.pi * (0.5 * b) ** 2 / (n * a * b)
        assert abs(frac - p0) < 5 * math.sqrt(p0 * (1 - p0) / pc)
        # equal mass in the 2n half-triangles (angular sectors between a vertex and an
        # apothem direction; the vertex directions follow the leaf orientation)
        v0 = vertex_angle(cfg, int(c))
        ang = np.mod(np.arctan2(d[:, 1], d[:, 0]) - v0, 2 * math.pi)
        sector = np.minimum((ang / (math.pi / n)).astype(int), 2 * n - 1)
        cnt = np.bincount(sector, minlength=2 * n)
        e = pc / (2 * n)
        chi2 = ((cnt - e) ** 2 / e).sum()
        assert chi2 < 2 * n - 1 + 6 * math.sqrt(2 * (2 * n - 1)), cnt


def vertex_angle(cfg, cell):
    """direction of one polygon vertex: square pi/4, hexagon 0 (D8), triangle +-pi/2 (isUp)"""
    if cfg.tiling == 0:
        return math.pi / 4
    if cfg.tiling == 1:
        return 0.0
    return math.pi / 2 if orc.triq_isup(cell, cfg.depth, cfg.depth) > 0 else -math.pi / 2


def test_draws_statistics():
    h = np.array([orc.draw(2024, c) for c in range(1 << 15)], dtype=np.uint64)
    bits = ((h[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(float)
    n = len(h)
    assert np.all(np.abs(bits.mean(0) - 0.5) < 5 * 0.5 / math.sqrt(n))
    x = (h >> np.uint64(11)).astype(float) * 2.0 ** -53
    assert abs(x.mean() - 0.5) < 5 * math.sqrt(1 / 12 / n)
    assert abs(x.var() - 1 / 12) < 0.01
    assert abs(np.corrcoef(x[:-1], x[1:])[0, 1]) < 5 / math.sqrt(n)
    # counter addressing: the state after c + 1 increments of seed is the state after c
    # increments of seed + phi
    phi = 0x9E3779B97F4A7C15
    for c in (1, 7, 1000):
        assert orc.draw(2024, c) == orc.draw((2024 + phi) % 2 ** 64, c - 1)
    assert orc.draw(1, 0) != orc.draw(2, 0)


def test_first_offset_slices_and_domain():
    cfg = cfg_for("sept", 3)
    cells = np.array([3, 100, 7, 342, 0, 55], np.int64)
    xy, u = orc.sample_cells(cfg, cells, 9, seed=3)
    xy2, u2 = orc.sample_cells(cfg, cells[2:5], 9, seed=3, first=2 * 9)
    assert np.array_equal(xy2, xy[18:45]) and np.array_equal(u2, u[18:45])
    xy3, _ = orc.sample_cells(cfg, cells, 9, seed=4)
    assert not np.array_equal(xy3, xy)
    with pytest.raises(orc.OracleError):
        orc.sample_cells(cfg, np.array([343], np.int64), 2, seed=1)
    with pytest.raises(orc.OracleError):
        orc.sample_cells(cfg, np.array([-1], np.int64), 2, seed=1)
