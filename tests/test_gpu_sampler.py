"""GPU (-m gpu) tests of SURVEY §8(f) NEXT-4, device-side generation and geometry:

* fmm_sample_cells (regular-polygon point picking, Fig. 12; D22) is bit-identical
  to the oracle's sampler: every point and strength, all three tilings, all leaves or ragged
  cell subsets with an offset `first`; at BASELINE.json's full sizes on sampled cells;
* every device-sampled point keys (device CellIndex) to the cell it was drawn for, at full size;
* Table 2's separation ratios measured on device-built trees: the local separation
  ratio r/R from device-sampled points and the device near lists (r = max |x - c| over a
  cell's points, R = min distance from c_t to any point outside near(t)), and the WSPD ratio
  rho/r from the device E4 lists and cell centres of every level (D20: rho = min E4 centre
  distance - 2r)."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
import oracle as orc

pytestmark = pytest.mark.gpu

FRAMES = {"quad": (0.0, 0.0, 1.0), "sept": (0.0, 0.0, 1.0), "triq": (0.5, math.sqrt(3.0) / 6.0, 1.0 / math.sqrt(3.0))}
TABLE2 = {"quad": (math.sqrt(2) / 3, 2 * (math.sqrt(2) - 1)), "sept": (0.5, 1.0), "triq": (0.5, math.sqrt(7) - 2)}
P2 = {"quad": 9, "sept": 7, "triq": 13}


def cfgs(tiling, L, frame=None):
    from paper_1204_3105_b200 import Config

    rx, ry, rs = frame or FRAMES[tiling]
    return Config.make(tiling, L, 8, rx, ry, rs, True), orc.config(tiling, L, 8, rx, ry, rs, True)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("tiling,L,per_cell", [("quad", 4, 37), ("sept", 3, 29), ("triq", 4, 31), ("sept", 4, 5),
                                               ("triq", 1, 3), ("quad", 1, 1)])
def test_sampler_bit_exact_all_leaves(tiling, L, per_cell):
    from paper_1204_3105_b200 import sample_cells

    gc, oc = cfgs(tiling, L)
    xy, u = sample_cells(gc, None, per_cell, seed=77)
    oxy, ou = orc.sample_cells(oc, None, per_cell, seed=77)
    assert np.array_equal(bits(xy.cpu().numpy()), bits(oxy))
    assert np.array_equal(bits(u.cpu().numpy()), bits(ou))


@pytest.mark.parametrize("tiling", ["quad", "sept", "triq"])
def test_sampler_bit_exact_subset_offset(tiling):
    import torch

    from paper_1204_3105_b200 import sample_cells

    gc, oc = cfgs(tiling, 5 if tiling != "sept" else 4)
    K = (7 if tiling == "sept" else 4) ** gc.depth
    rng = np.random.default_rng(3)
    cells = rng.choice(K, size=K // 3 + 1, replace=False).astype(np.int64)
    xy, u = sample_cells(gc, torch.from_numpy(cells).cuda(), 13, seed=2 ** 63 + 5, first=123456789)
    oxy, ou = orc.sample_cells(oc, cells, 13, seed=2 ** 63 + 5, first=123456789)
    assert np.array_equal(bits(xy.cpu().numpy()), bits(oxy))
    assert np.array_equal(bits(u.cpu().numpy()), bits(ou))
    # no strengths requested: same points
    xy2, u2 = sample_cells(gc, torch.from_numpy(cells).cuda(), 13, seed=2 ** 63 + 5, first=123456789,
                           want_u=False)
    assert u2 is None and torch.equal(xy2, xy)


def test_sampler_edge_cases():
    import torch

    from paper_1204_3105_b200 import FmmError, lib, sample_cells

    gc, _ = cfgs("sept", 3)
    xy, u = sample_cells(gc, torch.zeros(0, dtype=torch.int64, device="cuda"), 10, seed=1)
    assert xy.shape == (0, 2) and u.shape == (0,)
    xy, u = sample_cells(gc, None, 0, seed=1, ncells=5)
    assert xy.shape == (0, 2)
    with pytest.raises(FmmError) as e:
        sample_cells(gc, torch.tensor([0, 5, 343, 2, 400], dtype=torch.int64, device="cuda"), 4, seed=1)
    assert e.value.code == 2  # FMM_EDOMAIN
    assert "index 2" in str(e.value)
    with pytest.raises(FmmError):
        sample_cells(gc, torch.tensor([-1], dtype=torch.int64, device="cuda"), 4, seed=1)
    with pytest.raises(FmmError):  # more leaves than the tree has
        sample_cells(gc, None, 4, seed=1, ncells=344)
    # host output pointer: FMM_EBADCFG
    import ctypes

    host = np.zeros(8)
    rc = lib().fmm_sample_cells(ctypes.byref(gc), None, 2, 2, ctypes.c_uint64(1), 0,
                                ctypes.c_void_p(host.ctypes.data), None, None)
    assert rc == 1


FULL = {"C4q": 64, "C4s": 143, "C4t": 64}


@pytest.mark.parametrize("name", list(FULL))
def test_sampler_fullsize(name):
    """BASELINE.json's C4 sizes (16.8M points, all leaves): sampled cells bit-exact against
    the oracle (drawn alone through `first`), and every point keyed to its own cell by the
    device tree build"""
    import torch

    from paper_1204_3105_b200 import Config, Tree, X, sample_cells

    w = fi.get(name)
    pc = FULL[name]
    gc = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    oc = orc.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    K = (7 if w.tiling == "sept" else 4) ** w.depth
    xy, u = sample_cells(gc, None, pc, seed=99)
    assert xy.shape[0] == K * pc >= 16_000_000
    rng = np.random.default_rng(1)
    hx = xy.cpu().numpy()
    hu = u.cpu().numpy()
    for c in np.concatenate([[0, K - 1], rng.choice(K, 200, replace=False)]):
        c = int(c)
        oxy, ou = orc.sample_cells(oc, np.array([c], np.int64), pc, seed=99, first=c * pc)
        assert np.array_equal(bits(hx[c * pc:(c + 1) * pc]), bits(oxy)), c
        assert np.array_equal(bits(hu[c * pc:(c + 1) * pc]), bits(ou)), c
    t = Tree(gc, xy, u)
    keys = t.export(X.SRC_KEYS)
    t.check()
    t.close()
    assert np.array_equal(keys.astype(np.int64), np.repeat(np.arange(K, dtype=np.int64), pc))
    del xy, u
    torch.cuda.empty_cache()


@pytest.mark.parametrize("tiling,L,per_cell", [("quad", 5, 300), ("sept", 3, 700), ("triq", 5, 300)])
def test_table2_local_separation_ratio(tiling, L, per_cell):
    """r/R of Table 2 (Fig. 2: circles circumscribing a tile and inscribed
    in it plus its adjacent neighbours), measured on device-sampled points and device lists"""
    from paper_1204_3105_b200 import Tree, X, sample_cells

    gc, _ = cfgs(tiling, L)
    K = (7 if tiling == "sept" else 4) ** L
    xy, u = sample_cells(gc, None, per_cell, seed=8)
    t = Tree(gc, xy, u)
    cen = t.export(X.CENTRES, L).reshape(-1, 2)
    ow, of, en = t.export(X.NEAR_OWNERS), t.export(X.NEAR_OFFSETS), t.export(X.NEAR_ENTRIES)
    t.check()
    t.close()
    near = {int(o): set(int(s) for s in en[of[i]:of[i + 1]]) for i, o in enumerate(ow)}
    pts = xy.cpu().numpy()
    cell = np.repeat(np.arange(K), per_cell)
    r_emp = float(np.sqrt(((pts - cen[cell]) ** 2).sum(1)).max())
    # interior targets: t and all its neighbours have complete neighbourhoods
    full = {c for c, s in near.items() if len(s) == P2[tiling]}
    inner = [c for c in full if near[c] <= full]
    assert len(inner) > 10
    rng = np.random.default_rng(4)
    R_emp = np.inf
    for c in rng.choice(inner, size=min(60, len(inner)), replace=False):
        mask = ~np.isin(cell, list(near[int(c)]))
        R_emp = min(R_emp, float(np.sqrt(((pts[mask] - cen[c]) ** 2).sum(1)).min()))
    ratio = r_emp / R_emp
    want = TABLE2[tiling][0]
    assert ratio <= want * (1 + 1e-12), (ratio, want)
    assert ratio > want * 0.97, (ratio, want)


@pytest.mark.parametrize("name", ["C4q", "C4s", "C4t"])
def test_table2_wspd_ratio_device_lists(name):
    """rho/r of Table 2 (D20) on the device E4 lists and centres of every level of
    the full-size trees"""
    from paper_1204_3105_b200 import Config, Tree, X, sample_cells

    w = fi.get(name)
    gc = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    xy, u = sample_cells(gc, None, 1, seed=5)  # one point per leaf: every cell non-empty
    t = Tree(gc, xy, u)
    B = 7 if w.tiling == "sept" else 4
    for l in range(2, w.depth + 1):
        cen = t.export(X.CENTRES, l).reshape(-1, 2)
        ow, of, en = t.export(X.E4_OWNERS, l), t.export(X.E4_OFFSETS, l), t.export(X.E4_ENTRIES, l)
        own = np.repeat(ow.astype(np.int64), np.diff(of))
        dmin = float(np.sqrt(((cen[own] - cen[en.astype(np.int64)]) ** 2).sum(1)).min())
        if w.tiling == "quad":
            r = w.root_size * 2.0 ** -l / math.sqrt(2)
        elif w.tiling == "sept":
            r = fi.sept_leaf_r(w.root_size, w.depth) * math.sqrt(7.0) ** (w.depth - l)
        else:
            r = w.root_size * 2.0 ** -l
        assert abs((dmin - 2 * r) / r - TABLE2[w.tiling][1]) < 1e-9, (l, (dmin - 2 * r) / r)
    t.check()
    t.close()
