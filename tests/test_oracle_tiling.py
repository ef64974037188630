"""Oracle pins: tilings, addressing and interaction lists (PAPER.md sections 4-7, Tables 1-2).

Independent references used here (none of them calls the oracle's formulas):
* the paper's printed examples (tests/golden/);
* a geometric triangle-quadtree built in this file by recursive subdivision of
  the root triangle into (centre, vertical, left, right) children;
* leaf hexagon centres of fmm_inputs (polar formula, floating point) for the
  septree, and brute-force nearest-lattice / vertex-sharing geometry;
* Morton order written out for the quadtree;
* Table 2 counts and separation ratios."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
from conftest import golden_lines

S3 = math.sqrt(3.0)


def b7(s):
    return int(str(s), 7)


def b4(s):
    return int(str(s), 4)


# ------------------------------------------------------------------ configs
def sept_cfg(orc, L, R0=1.0, p=8):
    return orc.config("sept", L, p, 0.0, 0.0, R0)


def triq_cfg(orc, L, p=8):
    w = fi.get("C2")
    return orc.config("triq", L, p, w.root_x, w.root_y, w.root_size)


def quad_cfg(orc, L, p=8):
    return orc.config("quad", L, p, 0.0, 0.0, 1.0)


# ------------------------------------------------------------------ septree
def test_septree_neighbors_fig7a(orc):
    cfg = sept_cfg(orc, 3)
    for line in golden_lines("septree_neighbors.txt"):
        lhs, rhs = line.split(":")
        lvl, cell = lhs.split()
        want = [b7(v) for v in rhs.split()]
        assert orc.neighbors(cfg, int(lvl), b7(cell)) == want


def test_septree_level1_lists(orc):
    # reading D2: Neighbors(1,1) = {2,0,6} (table row 1 filtered by < 7), E4(1) = {3,4,5}
    cfg = sept_cfg(orc, 3)
    assert sorted(orc.neighbors(cfg, 1, 1)) == [0, 2, 6]
    assert orc.neighbors_e4(cfg, 1, 1) == [3, 4, 5]
    assert orc.neighbors(cfg, 1, 0) == [1, 2, 3, 4, 5, 6]
    assert orc.neighbors_e4(cfg, 1, 0) == []


def test_septree_center_example_342(orc):
    # CellCenter(342_7) = sum of the centres of {300, 40, 2}_7 (leaf level 3)
    cfg = sept_cfg(orc, 3)
    c = orc.cell_center(cfg, 3, b7(342))
    s = orc.cell_center(cfg, 3, b7(300)) + orc.cell_center(cfg, 3, b7(40)) + orc.cell_center(cfg, 3, b7(2))
    assert np.allclose(c, s, atol=1e-15)


def test_septree_centres_vs_generator_polar(orc):
    # exact-lattice centres (D12) vs the polar formula evaluated independently in fmm_inputs
    for L, R0 in [(3, 1.0), (4, 0.7)]:
        cfg = sept_cfg(orc, L, R0)
        ref = fi.island_leaf_centres(R0, L)
        for n in range(7 ** L):
            c = orc.cell_center(cfg, L, n)
            assert np.abs(c - ref[n]).max() < 1e-13 * R0
            cp = orc.cell_center_polar(cfg, L, n)
            assert np.abs(cp - c).max() < 1e-13 * R0


def test_septree_roundtrip_all_levels(orc):
    cfg = sept_cfg(orc, 4)
    for l in range(1, 5):
        for n in range(7 ** l):
            x, y = orc.cell_center(cfg, l, n)
            assert orc.cell_index(cfg, x, y, l) == n


def test_septree_keys_vs_generated_leaf(orc):
    # points drawn inside a known leaf hexagon (0.995 r) must key to that leaf
    rng = np.random.default_rng(11)
    for L, R0 in [(3, 1.0), (5, fi.sept_r0_equal_area())]:
        cen = fi.island_leaf_centres(R0, L)
        leaf = rng.integers(0, 7 ** L, 20000)
        px, py = fi.polygon_points(rng, len(leaf), 6, 0.995 * fi.sept_leaf_r(R0, L), 0.0)
        xy = np.stack([cen[leaf, 0] + px, cen[leaf, 1] + py], axis=1)
        k = orc.keys(sept_cfg(orc, L, R0), xy)
        assert np.array_equal(k.astype(np.int64), leaf)


def test_septree_duality(orc):
    L = 4
    cfg = sept_cfg(orc, L)
    rnd = np.random.default_rng(3)
    checked = 0
    for _ in range(400):
        a, b = (int(v) for v in rnd.integers(0, 7 ** L, 2))
        s = orc.gbt_add(int(np.base_repr(a, 7)), int(np.base_repr(b, 7)))
        sv = b7(s)
        if sv >= 7 ** L:
            continue
        ca, cb, cs = (orc.cell_center(cfg, L, v) for v in (a, b, sv))
        assert np.abs(ca + cb - cs).max() < 1e-12
        checked += 1
    assert checked > 100


def test_septree_neighbors_geometric(orc):
    L = 3
    cfg = sept_cfg(orc, L)
    r = fi.sept_leaf_r(1.0, L)
    cen = np.array([orc.cell_center(cfg, L, n) for n in range(7 ** L)])
    d = np.hypot(*(cen[:, None, :] - cen[None, :, :]).transpose(2, 0, 1))
    for n in range(7 ** L):
        want = set(np.nonzero(np.abs(d[n] - S3 * r) < 1e-9)[0].tolist())
        assert set(orc.neighbors(cfg, L, n)) == want


# ------------------------------------------------------------------ triangle-quadtree
def tri_tree(L, G, R0):
    """geometric triangle-quadtree: {level: {index: (apex, left, right)}} (apex = vertical vertex)."""
    apex = np.array([G[0], G[1] + R0])
    left = np.array([G[0] - R0 * S3 / 2, G[1] - R0 / 2])
    right = np.array([G[0] + R0 * S3 / 2, G[1] - R0 / 2])
    levels = {0: {0: (apex, left, right)}}
    for l in range(1, L + 1):
        cur = {}
        for idx, (a, lf, rt) in levels[l - 1].items():
            mal, mar, mlr = (a + lf) / 2, (a + rt) / 2, (lf + rt) / 2
            cur[4 * idx + 0] = (mlr, mal, mar)  # centre: flipped
            cur[4 * idx + 1] = (a, mal, mar)  # vertical
            cur[4 * idx + 2] = (mal, lf, mlr)  # left
            cur[4 * idx + 3] = (mar, mlr, rt)  # right
        levels[l] = cur
    return levels


def test_triangle_golden_examples(orc):
    for line in golden_lines("triangle_examples.txt"):
        f = line.split()
        if f[0] == "adj":
            k = {"L": 0, "R": 1, "V": 2}[f[3]]
            assert orc.triq_adjacent(int(f[1]), b4(f[2]), k) == b4(f[4])
        elif f[0] == "isup":
            t = f[1]
            got = [orc.triq_isup(b4(t[:i]), i, i) for i in range(1, len(t) + 1)]
            assert got == [int(v) for v in f[2:]]
        elif f[0] == "table1":
            src = int(f[1])
            for k, ent in enumerate(f[2:]):
                # Table 1 is observable through a level-1 cell: starred -> the sibling itself
                res = orc.triq_adjacent(1, src, k)
                if ent.endswith("*"):
                    assert res == int(ent[:-1])
                else:
                    assert res == -1  # no ancestor above level 1: domain boundary
    assert orc.triq_isup(0, 1, 1) == -1 and orc.triq_isup(0, 2, 2) == 1


@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_triangle_centres_and_neighbors_geometric(orc, L):
    w = fi.get("C2")
    cfg = triq_cfg(orc, L)
    levels = tri_tree(L, (w.root_x, w.root_y), w.root_size)
    for l in range(1, L + 1):
        cells = levels[l]
        vmap = {}
        for idx, tri in cells.items():
            c = sum(tri) / 3
            assert np.abs(orc.cell_center(cfg, l, idx) - c).max() < 1e-13
            assert np.abs(orc.cell_center_polar(cfg, l, idx) - c).max() < 1e-13
            for v in tri:
                vmap.setdefault((round(v[0], 9), round(v[1], 9)), set()).add(idx)
        for idx, tri in cells.items():
            want = set()
            for v in tri:
                want |= vmap[(round(v[0], 9), round(v[1], 9))]
            want.discard(idx)
            got = orc.neighbors(cfg, l, idx)
            assert len(got) == len(set(got))
            assert set(got) == want, (l, idx)


def test_triangle_keys_point_in_triangle(orc):
    L = 4
    w = fi.get("C2")
    cfg = triq_cfg(orc, L)
    leaves = tri_tree(L, (w.root_x, w.root_y), w.root_size)[L]
    rng = np.random.default_rng(5)
    px, py = fi.polygon_points(rng, 20000, 3, w.root_size, math.pi / 2)
    xy = np.stack([w.root_x + px, w.root_y + py], 1)
    keys = orc.keys(cfg, xy)
    idx = np.array(sorted(leaves))
    A = np.array([leaves[i][0] for i in idx])
    B = np.array([leaves[i][1] for i in idx])
    Cc = np.array([leaves[i][2] for i in idx])

    def cross(o, a, b):
        return (a[..., 0] - o[..., 0]) * (b[..., 1] - o[..., 1]) - (a[..., 1] - o[..., 1]) * (b[..., 0] - o[..., 0])

    P = xy[:, None, :]
    s1, s2, s3 = cross(A[None], B[None], P), cross(B[None], Cc[None], P), cross(Cc[None], A[None], P)
    inside = ((s1 >= 0) & (s2 >= 0) & (s3 >= 0)) | ((s1 <= 0) & (s2 <= 0) & (s3 <= 0))
    margin = np.minimum(np.minimum(np.abs(s1), np.abs(s2)), np.abs(s3))
    for j in range(len(xy)):
        hit = np.nonzero(inside[j])[0]
        if len(hit) != 1 or margin[j, hit[0]] < 1e-12:
            continue
        assert keys[j] == idx[hit[0]]


def test_triangle_domain_error(orc):
    cfg = triq_cfg(orc, 3)
    with pytest.raises(orc.OracleError) as e:
        orc.keys(cfg, np.array([[0.5, 0.3], [2.0, 2.0]]))
    assert e.value.code == orc.EDOMAIN and e.value.index == 1


# ------------------------------------------------------------------ quadtree
def test_quad_morton_keys_and_centres(orc):
    L = 5
    cfg = quad_cfg(orc, L)
    rng = np.random.default_rng(2)
    xy = rng.random((5000, 2))
    k = orc.keys(cfg, xy)
    i = np.floor(xy[:, 0] * 2 ** L).astype(np.int64)
    j = np.floor(xy[:, 1] * 2 ** L).astype(np.int64)
    want = np.zeros(len(xy), np.int64)
    for b in range(L):
        want |= ((i >> b) & 1) << (2 * b) | ((j >> b) & 1) << (2 * b + 1)
    assert np.array_equal(k.astype(np.int64), want)
    # children order: digit = 2*ybit + xbit (D7): child 1 of the root is lower-right
    assert np.allclose(orc.cell_center(quad_cfg(orc, 1), 1, 1), [0.75, 0.25])
    assert np.allclose(orc.cell_center(quad_cfg(orc, 1), 1, 2), [0.25, 0.75])
    # closed far edge clamps
    assert orc.keys(cfg, np.array([[1.0, 1.0]]))[0] == 4 ** L - 1


def test_quad_neighbors_geometric(orc):
    L = 3
    cfg = quad_cfg(orc, L)
    cen = np.array([orc.cell_center(cfg, L, n) for n in range(4 ** L)])
    h = 2.0 ** -L
    for n in range(4 ** L):
        d = np.abs(cen - cen[n]).max(axis=1)
        want = set(np.nonzero(np.abs(d - h) < 1e-12)[0].tolist())
        assert set(orc.neighbors(cfg, L, n)) == want


# ------------------------------------------------------------------ lists: Table 2, partition, separation
def _interior(orc, cfg, l, n, B):
    full = {0: 8, 1: 6, 2: 12}[cfg.tiling]
    return len(orc.neighbors(cfg, l, n)) == full and len(orc.neighbors(cfg, l - 1, n // B)) == full


@pytest.mark.parametrize("tiling", ["quad", "sept", "triq"])
def test_table2_P4_P2(orc, tiling):
    rows = {r.split()[0]: r.split() for r in golden_lines("table2.txt")}
    P4, P2 = int(rows[tiling][1]), int(rows[tiling][2])
    cfg = {"quad": quad_cfg, "sept": sept_cfg, "triq": triq_cfg}[tiling](orc, 4)
    B = 7 if tiling == "sept" else 4
    l = 3
    seen = 0
    for n in range(B ** l):
        e4 = orc.neighbors_e4(cfg, l, n)
        assert len(e4) <= P4
        if _interior(orc, cfg, l, n, B):
            assert len(e4) == P4
            assert len(orc.neighbors(cfg, l, n)) + 1 == P2
            seen += 1
    assert seen > 0


@pytest.mark.parametrize("tiling,L", [("quad", 4), ("sept", 3), ("triq", 4)])
def test_near_far_exact_partition(orc, tiling, L):
    """every (target leaf, source leaf) pair is covered exactly once by
    near(t) U E4(anc_l(t)) for l = 1..L (D1, D2)"""
    cfg = {"quad": quad_cfg, "sept": sept_cfg, "triq": triq_cfg}[tiling](orc, L)
    B = 7 if tiling == "sept" else 4
    K = B ** L
    e4 = {(l, n): set(orc.neighbors_e4(cfg, l, n)) for l in range(1, L + 1) for n in range(B ** l)}
    for t in range(K):
        near = set(orc.neighbors(cfg, L, t)) | {t}
        for s in range(K):
            c = int(s in near)
            for l in range(1, L + 1):
                sh = B ** (L - l)
                c += int((s // sh) in e4[(l, t // sh)])
            assert c == 1, (t, s)


@pytest.mark.parametrize("tiling,L", [("quad", 4), ("sept", 3), ("triq", 4)])
def test_e4_symmetric_and_separated(orc, tiling, L):
    rows = {r.split()[0]: r.split() for r in golden_lines("table2.txt")}
    rho_over_r = eval(rows[tiling][4], {"sqrt": math.sqrt})
    cfg = {"quad": quad_cfg, "sept": sept_cfg, "triq": triq_cfg}[tiling](orc, L)
    B = 7 if tiling == "sept" else 4
    if tiling == "quad":
        r = 2.0 ** -L / math.sqrt(2)
    elif tiling == "sept":
        r = fi.sept_leaf_r(1.0, L)
    else:
        r = fi.get("C2").root_size * 2.0 ** -L
    dmin = np.inf
    for n in range(B ** L):
        e4 = orc.neighbors_e4(cfg, L, n)
        for s in e4:
            assert n in orc.neighbors_e4(cfg, L, s)
            d = np.hypot(*(orc.cell_center(cfg, L, s) - orc.cell_center(cfg, L, n)))
            dmin = min(dmin, d)
        for s in orc.neighbors(cfg, L, n):
            assert n in orc.neighbors(cfg, L, s)
    # D20: rho = (min E4 centre distance) - 2 r reproduces Table 2
    assert abs((dmin - 2 * r) / r - rho_over_r) < 1e-9


@pytest.mark.parametrize("tiling,L,total", [("sept", 3, 13170), ("triq", 5, 43680), ("quad", 4, 6900),
                                            ("triq", 4, 8940)])
def test_full_tree_e4_totals(orc, tiling, L, total):
    # SURVEY App. A.8c / A.17 full-tree totals (independent scratch computation by the survey)
    cfg = {"quad": quad_cfg, "sept": sept_cfg, "triq": triq_cfg}[tiling](orc, L)
    B = 7 if tiling == "sept" else 4
    got = sum(len(orc.neighbors_e4(cfg, l, n)) for l in range(1, L + 1) for n in range(B ** l))
    assert got == total
