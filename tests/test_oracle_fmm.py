"""Oracle pins: operators (the paper omits them P:43), direct sum
(P:29-42), and the whole FMM against direct summation within the paper's bounds
(P:392-406), plus closed forms, invariants and degenerate cases."""
import cmath
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import fmm_inputs as fi


# ------------------------------------------------------------------ kernel / log
def test_log_special_values(orc):
    assert orc.log(1.0, 0.0) == 0
    assert abs(orc.log(math.e, 0.0) - 1) < 1e-16
    assert abs(2 * orc.log(0.0, 1.0) - 1j * math.pi) < 1e-15
    # principal branch, zero imaginary part canonicalised to +0 (D13)
    assert orc.log(-1.0, 0.0).imag == math.pi
    assert orc.log(-1.0, -0.0).imag == math.pi
    assert abs(orc.log(-1.0, -1e-300).imag + math.pi) < 1e-15


def test_direct_vs_numpy_log(orc):
    rng = np.random.default_rng(1)
    x = rng.random((64, 2))
    y = rng.random((64, 2)) + 2.0
    u = rng.uniform(-1, 1, 64)
    phi = orc.direct(x, u, y)
    zx = x[:, 0] + 1j * x[:, 1]
    zy = y[:, 0] + 1j * y[:, 1]
    ref = np.array([np.sum(u * np.log(t - zx)) for t in zy])
    assert np.abs(phi - ref).max() < 1e-12
    # independent compensated re-summation (math.fsum) of the real part
    ref_re = np.array([math.fsum(u * np.log(np.abs(t - zx))) for t in zy])
    assert np.abs(phi.real - ref_re).max() < 1e-12


def test_direct_self_and_coincident(orc):
    x = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    u = np.array([1.0, 2.0, 3.0])
    phi = orc.direct(x, u, self_mode=True)
    assert abs(phi[0] - (2 * cmath.log(-1 + 0j) + 3 * cmath.log(-1j))) < 1e-15
    with pytest.raises(orc.OracleError) as e:
        orc.direct(x, u, np.array([[5.0, 5.0], [1.0, 0.0]]))
    assert e.value.code == orc.ECOINCIDENT and e.value.index == 1


# ------------------------------------------------------------------ operators
def mp_eval(mp, c, z):
    zc = z - complex(*c)
    return mp[0] * np.log(zc) + sum(mp[k] * zc ** (-k) for k in range(1, len(mp)))


def loc_eval(loc, c, z):
    zc = z - complex(*c)
    return sum(loc[k] * zc ** k for k in range(len(loc)))


def test_p2m_closed_forms(orc):
    mp = orc.p2m(np.array([[0.3, 0.2]]), np.array([1.7]), [0.3, 0.2], 12)
    assert mp[0] == 1.7 and np.all(mp[1:] == 0)
    d = np.array([[0.1, 0.05], [-0.1, -0.05]])
    mp = orc.p2m(d, np.array([1.0, 1.0]), [0.0, 0.0], 12)
    assert np.abs(mp[1::2]).max() < 1e-18  # odd a_k vanish for +-d
    # a_k = -(1/k) sum u (x-c)^k for one source
    mp = orc.p2m(np.array([[0.1, 0.2]]), np.array([2.0]), [0.0, 0.0], 6)
    z = 0.1 + 0.2j
    assert np.allclose(mp[1:], [-2.0 * z ** k / k for k in range(1, 7)], rtol=1e-14)


def test_p2m_far_field_bound(orc):
    rng = np.random.default_rng(3)
    c = np.array([0.5, 0.5])
    r = 0.1
    x = c + (rng.random((8, 2)) - 0.5) * r
    u = rng.uniform(-1, 1, 8)
    p = 12
    mp = orc.p2m(x, u, c, p)
    R = 0.5
    for ang in np.linspace(0, 2 * np.pi, 10, endpoint=False):
        z = complex(*c) + R * cmath.exp(1j * ang)
        direct = np.sum(u * np.log(np.abs(z - (x[:, 0] + 1j * x[:, 1]))))
        rmax = np.abs((x[:, 0] + 1j * x[:, 1]) - complex(*c)).max()
        bound = np.abs(u).sum() / (R - rmax) * (rmax / R) ** (p + 1)
        assert abs(mp_eval(mp, c, z).real - direct) <= bound


def test_m2m_exact_shift(orc):
    rng = np.random.default_rng(4)
    x = rng.random((10, 2)) * 0.1
    u = rng.uniform(-1, 1, 10)
    p = 20
    c1, c2 = np.array([0.05, 0.04]), np.array([0.13, -0.02])
    a = orc.m2m(orc.p2m(x, u, c1, p), c1, c2, p)
    b = orc.p2m(x, u, c2, p)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    assert np.array_equal(orc.m2m(b, c2, c2, p), b)  # shift by zero


def test_m2l_single_source_closed_form(orc):
    p = 20
    cm, cl = np.array([0.2, -0.1]), np.array([1.5, 0.7])
    mp = np.zeros(p + 1, complex)
    mp[0] = 1.0
    loc = orc.m2l(mp, cm, cl, p)
    d = complex(*cl) - complex(*cm)
    want = [cmath.log(d)] + [(-1) ** (l + 1) / (l * d ** l) for l in range(1, p + 1)]
    assert np.abs(loc - np.array(want)).max() < 1e-15
    assert np.all(orc.m2l(np.zeros(p + 1), cm, cl, p) == 0)
    # linearity
    rng = np.random.default_rng(2)
    a = rng.standard_normal(p + 1) + 1j * rng.standard_normal(p + 1)
    a[0] = a[0].real
    assert np.abs(orc.m2l(2 * a, cm, cl, p) - 2 * orc.m2l(a, cm, cl, p)).max() < 1e-12


def test_m2l_local_matches_direct_within_bound(orc):
    rng = np.random.default_rng(8)
    r = 0.1
    cm, cl = np.array([0.0, 0.0]), np.array([3 * r * 1.2, 0.0])
    x = cm + (rng.random((6, 2)) - 0.5) * r
    u = rng.uniform(-1, 1, 6)
    p = 16
    loc = orc.m2l(orc.p2m(x, u, cm, p), cm, cl, p)
    for _ in range(10):
        y = cl + (rng.random(2) - 0.5) * r
        z = complex(*y)
        direct = np.sum(u * np.log(np.abs(z - (x[:, 0] + 1j * x[:, 1]))))
        assert abs(loc_eval(loc, cl, z).real - direct) < 1e-6


def test_l2l_exact_and_composition(orc):
    rng = np.random.default_rng(6)
    p = 12
    b = rng.standard_normal(p + 1) + 1j * rng.standard_normal(p + 1)
    c0, c1, c2 = np.array([0.0, 0.0]), np.array([0.1, -0.05]), np.array([0.12, 0.03])
    b1 = orc.l2l(b, c0, c1, p)
    b2 = orc.l2l(b1, c1, c2, p)
    b2d = orc.l2l(b, c0, c2, p)
    assert np.abs(b2 - b2d).max() < 1e-12 * np.abs(b2d).max()
    for _ in range(20):
        y = rng.random(2) * 0.2
        assert abs(orc.l2p(b1, c1, p, y) - loc_eval(b, c0, complex(*y))) < 1e-12 * abs(loc_eval(b, c0, complex(*y))) + 1e-13
    assert np.array_equal(orc.l2l(b, c0, c0, p), b)


def test_l2p_vs_polyval(orc):
    rng = np.random.default_rng(9)
    b = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    c = np.array([0.3, 0.1])
    y = np.array([0.35, 0.02])
    z = complex(*y) - complex(*c)
    assert abs(orc.l2p(b, c, 8, y) - np.polyval(b[::-1], z)) < 1e-15


# ------------------------------------------------------------------ whole FMM
def run(orc, w, data=None):
    d = data or fi.generate(w)
    cfg = orc.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    return d, orc.Tree(cfg, d["src_xy"], d["u"], d["tgt_xy"])


@pytest.mark.parametrize("tiling", ["quad", "triq"])
def test_depth1_has_no_far_field(orc, tiling):
    # L = 1 quad / triangle: all level-1 cells are mutual neighbours, no M2L -> FMM == direct incl. Im
    base = fi.get("C4q" if tiling == "quad" else "C2")
    w = base.scaled(700)
    w.depth = 1
    d, T = run(orc, w)
    phi, cnt = T.evaluate(counters=True)
    assert cnt["m2l_ops"] == 0
    ref = orc.direct(d["src_xy"], d["u"], self_mode=True)
    assert np.abs(phi - ref).max() < 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_fmm_within_paper_bound(orc, name):
    w = fi.get(name)
    d, T = run(orc, w)
    ids = np.arange(w.m) if name == "C1" else np.arange(0, w.m, 37)
    phi = T.evaluate(ids)
    ref = orc.direct(d["src_xy"], d["u"], d["tgt_xy"], w.self_mode, ids)
    err = np.abs(phi.real - ref.real)
    bound = T.bound(ids)
    assert np.all(err <= bound)  # D14 accumulated M2L bound
    assert err.max() < 1e-6 * np.abs(ref).max()
    # Im is branch dependent (D13): differences are multiples of 2 pi u-sums, not checked


def test_fmm_p_convergence(orc):
    # "exponential error loss for increasing truncation terms"; per-term decay <= alpha
    # of Table 2 (septree alpha = 1/2, D9 true-radius envelope 0.524)
    w = fi.get("C1").scaled(2048)
    d = fi.generate(w)
    ref = orc.direct(d["src_xy"], d["u"], d["tgt_xy"])
    errs = []
    ps = [4, 8, 12, 16]
    for p in ps:
        w.p = p
        _, T = run(orc, w, d)
        errs.append(np.abs(T.evaluate().real - ref.real).max())
    for a, b in zip(errs, errs[1:]):
        assert b < a
    rate = (errs[-1] / errs[0]) ** (1.0 / (ps[-1] - ps[0]))
    assert rate < 0.53


def test_fmm_linearity_and_full_vs_sampled(orc):
    w = fi.get("C2").scaled(4096)
    d = fi.generate(w)
    _, T = run(orc, w, d)
    phi = T.evaluate()
    d2 = dict(d)
    d2["u"] = 2.0 * d["u"]
    _, T2 = run(orc, w, d2)
    assert np.abs(T2.evaluate() - 2 * phi).max() <= 1e-14 * np.abs(phi).max()
    # sampled evaluation (fresh tree, only the needed locals) is identical bit for bit
    _, T3 = run(orc, w, d)
    ids = np.array([5, 77, 4095, 1000])
    assert np.array_equal(T3.evaluate(ids), phi[ids])


def test_fmm_counts_match_survey(orc):
    w = fi.get("C1")
    _, T = run(orc, w)
    _, cnt = T.evaluate(counters=True)
    assert cnt["m2l_ops"] == 13170  # full septree L3
    sk, tk = T.keys()
    so, to = T.leaf_offsets()
    # P2P pairs = sum over target leaves of n_t * sum_{s in near(t)} n_s
    pairs = sum((to[t + 1] - to[t]) * sum(so[s + 1] - so[s] for s in T.near(t)) for t in range(343))
    assert cnt["p2p_pairs"] == pairs


def test_self_mode_excludes_by_index_and_coincident_raises(orc):
    w = fi.get("C2").scaled(600)
    d = fi.generate(w)
    _, T = run(orc, w, d)
    phi = T.evaluate()
    assert np.all(np.isfinite(phi))
    d2 = dict(d)
    xy = d["src_xy"].copy()
    xy[10] = xy[3]
    d2["src_xy"] = xy
    _, T2 = run(orc, w, d2)
    with pytest.raises(orc.OracleError) as e:
        T2.evaluate()
    assert e.value.code == orc.ECOINCIDENT and e.value.index == 3


def test_empty_inputs(orc):
    w = fi.get("C1")
    cfg = orc.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size)
    T = orc.Tree(cfg, np.zeros((0, 2)), np.zeros(0), np.array([[0.01, 0.02]]))
    assert np.all(T.evaluate() == 0)


def test_out_of_domain_point(orc):
    w = fi.get("C1")
    cfg = orc.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size)
    xy = np.array([[0.0, 0.0], [0.1, 0.1], [3.0, 0.0]])
    with pytest.raises(orc.OracleError) as e:
        orc.Tree(cfg, xy, np.ones(3), xy)
    assert e.value.code == orc.EDOMAIN and e.value.index == 2


def test_thread_count_invariance(orc):
    code = (
        "import numpy as np, oracle, fmm_inputs as fi\n"
        "w = fi.get('C2').scaled(8192); d = fi.generate(w)\n"
        "cfg = oracle.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)\n"
        "T = oracle.Tree(cfg, d['src_xy'], d['u'])\n"
        "import sys; sys.stdout.buffer.write(T.evaluate().tobytes())\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for nt in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=nt, PYTHONPATH=root)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, check=True).stdout)
    assert outs[0] == outs[1] and len(outs[0]) == 8192 * 16


@pytest.mark.parametrize("name", ["C3", "C4q", "C4s", "C4t", "C5"])
def test_large_config_shapes_scaled(orc, name):
    # the big configs' domains and trees at oracle-friendly sizes: every point keys
    # into the domain, and the FMM stays within the paper bound on a sample
    w = fi.get(name).scaled(20000, 20000)
    d, T = run(orc, w)
    ids = np.arange(0, w.m, 97)
    phi = T.evaluate(ids)
    ref = orc.direct(d["src_xy"], d["u"], d["tgt_xy"], w.self_mode, ids)
    assert np.all(np.abs(phi.real - ref.real) <= T.bound(ids))
