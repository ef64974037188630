"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle on the
same seeded inputs.  Bit-exact: keys, sort permutation, leaf CSR, centres, near and
E4 lists.  Floating point: multipoles and potentials within 1e-12 normwise (D15)."""
import numpy as np
import pytest

from gpu_common import SMALL_CASES, data, gpu_tree, normwise, oracle_tree

pytestmark = pytest.mark.gpu

TOL = 1e-12  # BASELINE.json north_star: <= 1e-12 relative against the oracle FMM (normwise, D15)


@pytest.fixture(scope="module")
def pair_cache():
    return {}


def pair(cache, name):
    if name not in cache:
        w = SMALL_CASES[name]
        d = data(w)
        g = gpu_tree(w, d)
        o = oracle_tree(w, d)
        phi = g.evaluate()
        g.check()
        cache[name] = (w, d, g, o, phi.cpu().numpy())
    return cache[name]


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_keys_perm_offsets_bit_exact(pair_cache, name):
    from paper_1204_3105_b200 import X

    w, d, g, o, _ = pair(pair_cache, name)
    sk, tk = o.keys()
    sp, tp = o.perm()
    so, to = o.leaf_offsets()
    assert np.array_equal(g.export(X.SRC_KEYS), sk)
    assert np.array_equal(g.export(X.SRC_PERM), sp)
    assert np.array_equal(g.export(X.SRC_OFFSETS), so)
    if not w.self_mode:
        assert np.array_equal(g.export(X.TGT_KEYS), tk)
        assert np.array_equal(g.export(X.TGT_PERM), tp)
        assert np.array_equal(g.export(X.TGT_OFFSETS), to)


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_centres_bit_exact(pair_cache, name):
    from paper_1204_3105_b200 import X

    w, d, g, o, _ = pair(pair_cache, name)
    for l in range(w.depth + 1):
        gc = g.export(X.CENTRES, l).reshape(-1, 2)
        oc = o.centres(l)
        assert np.array_equal(gc.view(np.uint64), oc.view(np.uint64)), l


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_lists_bit_exact(pair_cache, name):
    from paper_1204_3105_b200 import X

    w, d, g, o, _ = pair(pair_cache, name)
    ow, of, en = o.near_csr()
    assert np.array_equal(g.export(X.NEAR_OWNERS), ow)
    assert np.array_equal(g.export(X.NEAR_OFFSETS), of)
    assert np.array_equal(g.export(X.NEAR_ENTRIES), en)
    for l in range(1, w.depth + 1):
        ow, of, en = o.e4_csr(l)
        assert np.array_equal(g.export(X.E4_OWNERS, l), ow), l
        assert np.array_equal(g.export(X.E4_OFFSETS, l), of), l
        assert np.array_equal(g.export(X.E4_ENTRIES, l), en), l


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_multipoles(pair_cache, name):
    from paper_1204_3105_b200 import X

    w, d, g, o, _ = pair(pair_cache, name)
    for l in range(1, w.depth + 1):
        gm = g.export(X.MULTIPOLE, l).reshape(-1, w.p + 1)
        om = o.multipoles(l)
        assert normwise(gm, om) <= TOL, l


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_potentials(pair_cache, name):
    w, d, g, o, phi = pair(pair_cache, name)
    ref, cnt = o.evaluate(counters=True)
    assert normwise(phi, ref) <= TOL
    from paper_1204_3105_b200 import X

    c = g.export(X.COUNTERS)
    assert c[0] == cnt["m2l_ops"] and c[1] == cnt["p2p_pairs"]


def test_host_inputs_match_device_inputs():
    w = SMALL_CASES["C1"]
    d = data(w)
    a = gpu_tree(w, d).evaluate().cpu().numpy()
    out = np.zeros(w.m, np.complex128)
    gh = gpu_tree(w, d, host_inputs=True)
    gh.evaluate(out)
    import torch

    torch.cuda.synchronize()
    assert np.array_equal(a, out)


@pytest.mark.parametrize("p", [1, 5, 10, 14, 27, 31])
def test_expansion_orders(p):
    """every template order of the downward kernel (P = 8, 12, 16, 28, 32 here; 16, 20, 24 in the
    configs): row 0 of the M2L contraction is formed outside the DMMA tiles when P % 8 == 0"""
    w = SMALL_CASES["C2"].scaled(3000)
    d = data(w)
    phi = gpu_tree(w, d, p=p).evaluate().cpu().numpy()
    assert normwise(phi, oracle_tree(w, d, p=p).evaluate()) <= TOL


@pytest.mark.parametrize("tiling_case", ["C1", "C2", "C4qs"])
def test_depth_one(tiling_case):
    w = SMALL_CASES[tiling_case].scaled(2000, name=tiling_case + "-L1")
    w.depth = 1  # the septree island of depth 1 is the 7-hexagon flower: regenerate inside it
    d = data(w)
    phi = gpu_tree(w, d).evaluate().cpu().numpy()
    assert normwise(phi, oracle_tree(w, d).evaluate()) <= TOL


def test_empty_sources_and_targets():
    import torch

    from paper_1204_3105_b200 import Config, Tree

    w = SMALL_CASES["C1"]
    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, False)
    t = Tree(cfg, torch.zeros((0, 2), dtype=torch.float64, device="cuda"),
             torch.zeros(0, dtype=torch.float64, device="cuda"),
             torch.tensor([[0.01, 0.02], [0.1, -0.2]], dtype=torch.float64, device="cuda"))
    phi = t.evaluate().cpu().numpy()
    t.check()
    assert np.all(phi == 0)
    t2 = Tree(cfg, torch.tensor([[0.01, 0.02]], dtype=torch.float64, device="cuda"),
              torch.ones(1, dtype=torch.float64, device="cuda"), torch.zeros((0, 2), dtype=torch.float64, device="cuda"))
    assert t2.evaluate().numel() == 0


def test_out_of_domain_reported():
    import torch

    from paper_1204_3105_b200 import Config, FmmError, Tree

    w = SMALL_CASES["C1"]
    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
    xy = torch.tensor([[0.0, 0.0], [0.1, 0.1], [3.0, 0.0], [0.2, -0.1]], dtype=torch.float64, device="cuda")
    t = Tree(cfg, xy, torch.ones(4, dtype=torch.float64, device="cuda"))
    rc, idx = t.status()
    assert rc == 2 and idx == 2
    with pytest.raises(FmmError):
        t.check()


def test_coincident_reported():
    import torch

    w = SMALL_CASES["C2"].scaled(500)
    d = dict(data(w))
    xy = d["src_xy"].copy()
    xy[10] = xy[3]
    d["src_xy"] = xy
    t = gpu_tree(w, d)
    t.evaluate()
    rc, idx = t.status()
    assert rc == 3 and idx == 3


def test_repeat_evaluate_deterministic():
    w = SMALL_CASES["C4ts"]
    d = data(w)
    g = gpu_tree(w, d)
    a = g.evaluate().cpu().numpy()
    b = g.evaluate().cpu().numpy()
    assert np.array_equal(a, b)


def test_set_strengths_linearity():
    import torch

    w = SMALL_CASES["C2"].scaled(4000)
    d = data(w)
    g = gpu_tree(w, d)
    a = g.evaluate().cpu().numpy()
    g.set_strengths(torch.from_numpy(2.0 * d["u"]).cuda())
    b = g.evaluate().cpu().numpy()
    assert normwise(b, 2 * a) <= 1e-14


@pytest.mark.parametrize("n", [9000, 24000])
def test_heavy_blocks(n):
    """Dense leaves: quadtree depth 2 (16 leaves) with n self points, so that near blocks
    exceed 65,536 pairs (symmetric heavy tasks split by rows, reactions added atomically;
    24000 points also puts leaves above the 192-point shared-memory limit) - against the
    oracle within the D15 gate, and the self-pair exclusion holds in split diagonal blocks."""
    w = SMALL_CASES["C4qs"].scaled(n, name=f"heavy{n}")
    d = data(w)
    g = gpu_tree(w, d, depth=2)
    o = oracle_tree(w, d, depth=2)
    phi = g.evaluate().cpu().numpy()
    g.check()
    ref = o.evaluate()
    assert normwise(phi, ref) <= TOL


@pytest.mark.parametrize("name", ["C1", "C2s"])
def test_direct_sum_matches_oracle(name):
    """fmm_direct (NEXT-1 reference) against the oracle's direct sum: same definition
    (principal Log per pair, D13; i != j in self mode, D16), so Re and Im agree to rounding."""
    import oracle

    from paper_1204_3105_b200 import direct

    w = SMALL_CASES["C1"] if name == "C1" else SMALL_CASES["C2"].scaled(6000, name="C2s")
    d = data(w)
    ref = oracle.direct(d["src_xy"], d["u"], d["tgt_xy"], self_mode=w.self_mode)
    out = np.zeros(w.m, np.complex128)
    direct(d["src_xy"], d["u"], d["tgt_xy"], self_mode=w.self_mode, out=out)
    assert normwise(out, ref) <= 1e-14
    import torch

    dev = direct(torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda(),
                 None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda(), self_mode=w.self_mode)
    assert np.array_equal(dev.cpu().numpy(), out)


def test_direct_sum_coincident_raises():
    from paper_1204_3105_b200 import FmmError, direct

    src = np.array([[0.1, 0.2], [0.3, 0.4]])
    tgt = np.array([[0.5, 0.5], [0.3, 0.4]])
    with pytest.raises(FmmError) as e:
        direct(src, np.ones(2), tgt, out=np.zeros(2, np.complex128))
    assert e.value.code == 3


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_locals_per_level(pair_cache, name):
    """the local expansions b_0..b_p of every evaluated cell (cells with targets), level by
    level, against the oracle's L2L + M2L (App. B.4/B.5; D15 normwise per level) -- M2L and L2L
    checked directly, not only through the potentials"""
    from paper_1204_3105_b200 import X

    w, d, g, o, _ = pair(pair_cache, name)
    rng = np.random.default_rng(11)
    for l in range(1, w.depth + 1):
        owners = g.export(X.E4_OWNERS, l)  # cells of level l with targets
        gl = g.export(X.LOCAL, l).reshape(-1, w.p + 1)
        cells = owners if len(owners) <= 1500 else np.sort(rng.choice(owners, 1500, replace=False))
        ref = np.array([o.local(l, int(c)) for c in cells])
        assert normwise(gl[cells], ref) <= TOL, l


@pytest.mark.parametrize("self_mode", [True, False])
def test_tiny_separation_across_leaves(self_mode):
    """Pairs closer than 1e-30 in DIFFERENT leaves (quadtree rooted at (-1/2, -1/2), so that the
    cell boundaries x = 0 and y = 0 separate (+-1e-40, y) and (x, +-1e-41)): the pair kernel must
    send them to its exact path (p2p.cu p2p_slow) in off-diagonal blocks too, where no pair is
    excluded.  Against the oracle within the D15 gate (a garbage or dropped tiny pair,
    |u log|z|^2| ~ 180, fails it), and bitwise repeatable."""
    import dataclasses

    import torch

    from paper_1204_3105_b200 import Config, Tree

    w = dataclasses.replace(SMALL_CASES["C4qs"].scaled(3000, name="tiny"), root_x=-0.5, root_y=-0.5,
                            self_mode=self_mode, depth=4)
    rng = np.random.default_rng(7)
    src = rng.uniform(-0.5, 0.5, (3000, 2))
    src[:4] = [[1e-40, 0.1], [-1e-40, 0.1], [0.2, -3e-41], [0.2, 2e-41]]
    u = rng.uniform(-1, 1, 3000)
    tgt = None
    if not self_mode:
        tgt = rng.uniform(-0.5, 0.5, (2000, 2))
        tgt[:2] = [[-2e-40, 0.1], [0.2, 1e-41]]  # within 3e-40 of sources 0, 1 and 2, 3 (across x = 0 / y = 0)
    d = {"src_xy": src, "u": u, "tgt_xy": tgt}
    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, self_mode)
    g = Tree(cfg, torch.from_numpy(src).cuda(), torch.from_numpy(u).cuda(),
             None if tgt is None else torch.from_numpy(tgt).cuda())
    phi = g.evaluate().cpu().numpy()
    g.check()
    o = oracle_tree(w, d)
    ref = o.evaluate()
    assert normwise(phi, ref) <= TOL
    b = g.evaluate().cpu().numpy()
    assert np.array_equal(phi, b)


@pytest.mark.parametrize("case", ["bucket", "lsd_mean", "lsd_big_leaf", "lsd_forced"])
def test_sort_paths_bit_exact(case, monkeypatch):
    """The one-rank sort (build.cu single_rank_keys_sort) on each of its paths against the
    oracle's stable order by (key, input index): the bucket sort (> 2^20 points, small
    leaves), the LSD record sort taken for a high mean occupancy, the LSD sort selected on the
    device when the leaf counts show a leaf above 256 points (a tight cluster in a sparse tree),
    and FMM_SORT_LSD=1; permutation and leaf CSR bit for bit against the oracle, self mode and
    distinct targets.  Potentials: against the oracle FMM for the small case; for the 1.1M-point
    cases bitwise against the same tree sorted by the forced LSD path (same order, same sorted
    arrays => the same Phi; to rounding where a heavy block adds reactions atomically)."""
    import oracle

    from paper_1204_3105_b200 import X

    base = SMALL_CASES["C4qs"]
    n, depth = {"bucket": (1100000, 9), "lsd_mean": (30000, 2), "lsd_big_leaf": (1100000, 9),
                "lsd_forced": (1100000, 9)}[case]
    if case == "lsd_forced":
        monkeypatch.setenv("FMM_SORT_LSD", "1")
    for self_mode in (True, False):
        w = base.scaled(n, n // 2, name=f"sort-{case}")
        w.self_mode = self_mode
        w.m = n if self_mode else n // 2
        d = dict(data(w))
        if case == "lsd_big_leaf":  # 400 points within 1e-4 of (0.1, 0.1): one leaf (side 2^-9) of > 256
            rng = np.random.default_rng(5)
            xy = d["src_xy"].copy()
            xy[:400] = 0.1 + rng.uniform(-1e-4, 1e-4, (400, 2))
            d["src_xy"] = xy
        g = gpu_tree(w, d, depth=depth)
        cfg = oracle.config(w.tiling, depth, w.p, w.root_x, w.root_y, w.root_size, self_mode)
        sk = oracle.keys(cfg, d["src_xy"])
        sp = np.argsort(sk, kind="stable").astype(np.int32)
        so = np.searchsorted(sk[sp], np.arange(4 ** depth + 1)).astype(np.int64)
        if case == "lsd_big_leaf":
            assert np.diff(so).max() > 256
        assert np.array_equal(g.export(X.SRC_PERM), sp)
        assert np.array_equal(g.export(X.SRC_OFFSETS), so)
        if not self_mode:
            tk = oracle.keys(cfg, d["tgt_xy"])
            tp = np.argsort(tk, kind="stable").astype(np.int32)
            assert np.array_equal(g.export(X.TGT_PERM), tp)
        phi = g.evaluate().cpu().numpy()
        if n <= 100000:
            assert normwise(phi, oracle_tree(w, d, depth=depth).evaluate()) <= TOL
        else:
            monkeypatch.setenv("FMM_SORT_LSD", "1")
            ref = gpu_tree(w, d, depth=depth).evaluate().cpu().numpy()
            monkeypatch.delenv("FMM_SORT_LSD")
            if case == "lsd_big_leaf":  # its 400-point leaf makes heavy blocks: FP64 atomics, rounding-level
                assert normwise(phi, ref) <= 1e-14
            else:
                assert np.array_equal(phi.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("pairs", ["1", "0"])
@pytest.mark.parametrize("name", ["C2", "C4qs", "C4ts", "C4ss", "C5s"])
def test_p2p_pairing_variants(name, pairs, monkeypatch):
    """Both pair-kernel variants (p2p.cu fmm_p2p_pairing: TF_PAIR tasks -- two light off-diagonal
    near leaves of a row leaf in one task -- and the plain kernel), forced by FMM_P2P_PAIRS, on
    every tiling and the clustered case against the oracle (D15), and bitwise repeatable.  The
    scaled-down cases have fewer points per leaf than the benchmark trees, so the default rule
    would not pair them."""
    monkeypatch.setenv("FMM_P2P_PAIRS", pairs)
    w = SMALL_CASES[name]
    d = data(w)
    g = gpu_tree(w, d)
    phi = g.evaluate().cpu().numpy()
    g.check()
    assert normwise(phi, oracle_tree(w, d).evaluate()) <= TOL
    assert np.array_equal(phi, g.evaluate().cpu().numpy()) or name == "C5s"  # C5s: heavy blocks (atomics)


@pytest.mark.parametrize("case,depth", [("C4qs", 12), ("C4ts", 12), ("C4ss", 9)])
def test_maximum_depth(case, depth):
    """The deepest trees fmm_build_tree accepts (include/fmm_b200.h: depth 12 for the quadtree and
    the triangle-quadtree, 9 for the septree: 16.8M / 40.4M leaves, nearly all of them empty) on
    20,000 points: keys, sort order and leaf CSR bit for bit against the oracle (P:76, P:79,
    P:207-250), potentials within the D15 gate of the oracle FMM at the same depth.
    The septree's points are drawn in the depth-6 island and pulled towards its centre, since the
    island's boundary changes with the depth."""
    import oracle

    from paper_1204_3105_b200 import X

    w = SMALL_CASES[case].scaled(20000, name=f"max-{case}")
    d = dict(data(w))
    if w.tiling == SMALL_CASES["C4ss"].tiling:
        c = np.array([w.root_x, w.root_y])
        d["src_xy"] = c + 0.6 * (d["src_xy"] - c)
    g = gpu_tree(w, d, p=4, depth=depth)
    cfg = oracle.config(w.tiling, depth, 4, w.root_x, w.root_y, w.root_size, True)
    sk = oracle.keys(cfg, d["src_xy"])
    K = (7 if w.tiling == SMALL_CASES["C4ss"].tiling else 4) ** depth
    assert sk.max() < K
    assert np.array_equal(g.export(X.SRC_KEYS), sk)
    sp = np.argsort(sk, kind="stable").astype(np.int32)
    assert np.array_equal(g.export(X.SRC_PERM), sp)
    so = np.searchsorted(sk[sp], np.arange(K + 1)).astype(np.int64)
    assert np.array_equal(g.export(X.SRC_OFFSETS), so)
    phi = g.evaluate().cpu().numpy()
    g.check()
    assert normwise(phi, oracle_tree(w, d, p=4, depth=depth).evaluate()) <= TOL
