"""Pins of the oracle's accumulated truncation bound B_j (orc_tree_bound, reading D14 of the
M2L bound P:403 with Table 2's rho/r) against hand-derived values
(tests/golden/bound_cases.txt): a quadtree case pins A_s = sum |u| over the E4 cell and the
exponent p + 1; a septree case pins the level of rho_l (level-1 E4 cells, D2, against leaf-level
ones).  Then a tightness window on the C1 workload: the FMM error is below B_j everywhere and
B_j is not vacuous (max err / B_j above 1e-7)."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
from conftest import golden_lines


def _golden():
    return {ln.split()[0]: float(ln.split()[1]) for ln in golden_lines("bound_cases.txt")}


def _tree(orc, tiling, depth, p, root, src, u, tgt):
    cfg = orc.config(tiling, depth, p, root[0], root[1], root[2], False)
    return cfg, orc.Tree(cfg, np.asarray(src, float), np.asarray(u, float), np.asarray(tgt, float))


def test_bound_quad_depth2(orc):
    src = [(0.9, 0.9), (0.6, 0.1), (0.62, 0.12), (0.3, 0.1)]
    u = [1.0, -1.0, 0.25, 0.5]
    cfg, T = _tree(orc, "quad", 2, 4, (0.0, 0.0, 1.0), src, u, [(0.1, 0.1)])
    sk, tk = T.keys()
    # Morton keys (D7): leaf (i, j) -> interleave, x bits even
    assert list(sk) == [15, 4, 4, 1] and list(tk) == [0]
    T.upward()
    b = T.bound(np.array([0]))[0]
    assert b == pytest.approx(_golden()["quadL2"], rel=1e-13)
    # and the bound holds for this target
    phi = T.evaluate(np.array([0]))[0]
    ref = orc.direct(np.asarray(src, float), np.asarray(u, float), np.array([(0.1, 0.1)]))[0]
    assert abs(phi.real - ref.real) <= b


def test_bound_septree_depth2_levels(orc):
    cfg = orc.config("sept", 2, 4, 0.0, 0.0, 1.0, False)
    r = 1.0 / 7.0
    c = {n: orc.cell_center(cfg, 2, n) for n in (7, 8, 14, 21, 22)}  # leaves 10, 11, 20, 30, 31 (base 7)
    tgt = [c[7] + 0.1 * r * np.array([1.0, 0.5])]
    src = [c[21], c[22] + np.array([0.1 * r, 0.0]), c[14], c[8]]
    u = [1.0, -0.5, 2.0, 3.0]
    cfg, T = _tree(orc, "sept", 2, 4, (0.0, 0.0, 1.0), src, u, tgt)
    sk, tk = T.keys()
    assert list(sk) == [21, 22, 14, 8] and list(tk) == [7]
    T.upward()
    b = T.bound(np.array([0]))[0]
    assert b == pytest.approx(_golden()["septL2"], rel=1e-13)
    phi = T.evaluate(np.array([0]))[0]
    ref = orc.direct(np.asarray(src, float), np.asarray(u, float), np.asarray(tgt))[0]
    assert abs(phi.real - ref.real) <= b


def test_bound_zero_without_far_sources(orc):
    """sources only in near leaves: no M2L term, B_j = 0, and the FMM is the direct sum"""
    src = [(0.3, 0.1), (0.12, 0.35)]
    cfg, T = _tree(orc, "quad", 2, 6, (0.0, 0.0, 1.0), src, [1.0, -2.0], [(0.1, 0.1)])
    T.upward()
    assert T.bound(np.array([0]))[0] == 0.0
    phi = T.evaluate(np.array([0]))[0]
    ref = orc.direct(np.asarray(src, float), np.array([1.0, -2.0]), np.array([(0.1, 0.1)]))[0]
    assert abs(phi - ref) <= 1e-15 * abs(ref)


def test_bound_tightness_window_c1(orc):
    """on C1 every target's Re error lies below B_j, and the largest ratio err / B_j is above
    1e-7 (the bound is not vacuous: the survey measured ~1.4e-5 at this scale)"""
    w = fi.get("C1")
    d = fi.generate(w)
    T = orc.Tree(orc.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode),
                 d["src_xy"], d["u"], d["tgt_xy"])
    ids = np.arange(w.m)
    phi = T.evaluate(ids)
    ref = orc.direct(d["src_xy"], d["u"], d["tgt_xy"], w.self_mode, ids)
    ratio = np.abs(phi.real - ref.real) / T.bound(ids)
    assert ratio.max() < 1.0
    assert ratio.max() > 1e-7
    # and the bound follows the decay 1/(1 + rho/r) = 1/2 per extra term (septree, Table 2)
    w2 = fi.get("C1")
    w2.p = w.p + 1
    T2 = orc.Tree(orc.config(w2.tiling, w2.depth, w2.p, w2.root_x, w2.root_y, w2.root_size, w2.self_mode),
                  d["src_xy"], d["u"], d["tgt_xy"])
    T2.upward()
    T.upward()
    b1, b2 = T.bound(ids[:64]), T2.bound(ids[:64])
    assert np.allclose(b2, 0.5 * b1, rtol=1e-13)
