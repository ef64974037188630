"""Multi-rank parity (-m gpu) on one GPU, ranks run one after another (no rank waits on
another): every rank r of R builds its tree (keys of every point, global leaf counts, its
work-balanced leaf range, the rank-local sort of its own + halo leaves), runs
fmm_evaluate_begin (P2M / M2M over its own source leaves, the P2P pair kernel); the test then
plays the collective -- the multipole trees of all ranks are summed (what ncclAllReduce does
inside fmm_evaluate when the config carries a comm) -- and every rank runs
fmm_evaluate_end into one output.  The union of the ranks' disjoint outputs must match the
oracle FMM within the D15 gate (cross-rank sums change the FP64 order, so the
gate is 1e-12, not bit-equality), keys and lists stay bit-exact."""
import numpy as np
import pytest

from gpu_common import SMALL_CASES, data, normwise, oracle_tree

pytestmark = pytest.mark.gpu

TOL = 1e-12

CASES = {
    "C2": SMALL_CASES["C2"],
    "C4ts": SMALL_CASES["C4ts"],
    "C4qs": SMALL_CASES["C4qs"],
    "C5s": SMALL_CASES["C5s"],
    "C3s": SMALL_CASES["C3s"],
    "C1": SMALL_CASES["C1"],
}

_ORC = {}


def oracle_phi(name):
    if name not in _ORC:
        w = CASES[name] if name in CASES else None
        _ORC[name] = oracle_tree(w, data(w)).evaluate()
    return _ORC[name]


def run_ranks(w, d, R, depth=None, out_nan=True):
    """build + evaluate ranks 0..R-1 of a tree sequentially, the multipole sum done here"""
    import torch

    from paper_1204_3105_b200 import Config, Tree

    src = torch.from_numpy(d["src_xy"]).cuda()
    u = torch.from_numpy(d["u"]).cuda()
    tgt = None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda()
    trees = []
    for r in range(R):
        cfg = Config.make(w.tiling, depth or w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode,
                          rank=r, nranks=R)
        t = Tree(cfg, src, u, tgt)
        t.evaluate_begin()
        trees.append(t)
    torch.cuda.synchronize()
    bufs = []
    for t in trees:
        ptr, nb = t.multipole_buffer()
        bufs.append((ptr, nb))
    assert len({nb for _, nb in bufs}) == 1
    nb = bufs[0][1]
    total = torch.zeros(nb // 8, dtype=torch.float64, device="cuda")
    views = []
    for ptr, _ in bufs:
        v = _dev_view(ptr, nb)
        views.append(v)
        total += v
    for v in views:
        v.copy_(total)
    torch.cuda.synchronize()
    phi = torch.full((w.m,), complex("nan+nanj") if out_nan else 0, dtype=torch.complex128, device="cuda")
    for t in trees:
        t.evaluate_end(phi)
    torch.cuda.synchronize()
    for t in trees:
        t.check()
    ranges = [t.rank_range() for t in trees]
    return phi.cpu().numpy(), ranges, trees


def _dev_view(ptr, nbytes):
    """a float64 torch view of device memory owned by the library (test-side collective)"""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")


@pytest.mark.parametrize("R", [2, 3, 8])
@pytest.mark.parametrize("name", ["C2", "C4ts", "C5s", "C3s"])
def test_multirank_union_matches_oracle(name, R):
    w = CASES[name]
    d = data(w)
    phi, ranges, trees = run_ranks(w, d, R)
    # the ranges tile [0, K) in order
    K = (7 if w.tiling == "sept" else 4) ** w.depth
    assert ranges[0][0] == 0 and ranges[-1][1] == K
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]
    assert not np.isnan(phi).any(), "a target was written by no rank"
    assert normwise(phi, oracle_phi(name)) <= TOL


def test_multirank_keys_lists_bit_exact():
    """every rank's keys are the oracle's; its near / E4 lists are the oracle's restricted to
    the rank's own target leaves (global emptiness), and its kept sources are sorted by
    (leaf, input index)"""
    from paper_1204_3105_b200 import X

    w = CASES["C4ts"]
    d = data(w)
    o = oracle_tree(w, d)
    sk, _ = o.keys()
    _, ranges, trees = run_ranks(w, d, 3)
    ow, of, en = o.near_csr()
    for t, (lo, hi) in zip(trees, ranges):
        assert np.array_equal(t.export(X.SRC_KEYS), sk)
        keep = (ow >= lo) & (ow < hi)
        gow = t.export(X.NEAR_OWNERS)
        assert np.array_equal(gow, ow[keep])
        gen = t.export(X.NEAR_ENTRIES)
        ref = np.concatenate([en[of[i]:of[i + 1]] for i in np.nonzero(keep)[0]]) if keep.any() else en[:0]
        assert np.array_equal(gen, ref)
        for l in range(1, w.depth + 1):
            e_ow, e_of, e_en = o.e4_csr(l)
            span = 4 ** (w.depth - l)
            # E4 owners of the rank: cells with a target leaf in [lo, hi)
            g_ow = t.export(X.E4_OWNERS, l)
            assert np.all((g_ow + 1) * span > lo) and np.all(g_ow * span < hi)
            idx = np.searchsorted(e_ow, g_ow)
            assert np.array_equal(e_ow[idx], g_ow)
            g_of = t.export(X.E4_OFFSETS, l)
            g_en = t.export(X.E4_ENTRIES, l)
            for j, c in enumerate(g_ow):
                assert np.array_equal(g_en[g_of[j]:g_of[j + 1]], e_en[e_of[idx[j]]:e_of[idx[j] + 1]])
        perm = t.export(X.SRC_PERM)
        keys = sk[perm]
        assert np.all(np.diff(keys.astype(np.int64)) >= 0)
        same = np.diff(keys.astype(np.int64)) == 0
        assert np.all(np.diff(perm)[same] > 0)
        # the rank keeps every source of its own leaves
        own = (sk >= lo) & (sk < hi)
        assert set(np.nonzero(own)[0]) <= set(perm.tolist())


def test_multirank_heavy_blocks():
    """dense leaves (quadtree depth 2, 24,000 self points): heavy symmetric blocks whose two
    leaves fall in different ranks are evaluated by both ranks, each keeping its own side"""
    w = SMALL_CASES["C4qs"].scaled(24000, name="heavy24000")
    d = data(w)
    ref = oracle_tree(w, d, depth=2).evaluate()
    for R in (2, 3):
        phi, ranges, _ = run_ranks(w, d, R, depth=2)
        assert not np.isnan(phi).any()
        assert normwise(phi, ref) <= TOL, R


def test_multirank_evaluate_needs_comm():
    """fmm_evaluate on a multi-rank tree without a communicator is refused (the partial
    multipole tree alone would give wrong potentials)"""
    import torch

    from paper_1204_3105_b200 import Config, FmmError, Tree

    w = CASES["C1"]
    d = data(w)
    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode, rank=0, nranks=2)
    t = Tree(cfg, torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda(),
             torch.from_numpy(d["tgt_xy"]).cuda())
    with pytest.raises(FmmError) as e:
        t.evaluate()
    assert e.value.code == 1


def test_single_rank_comm_allreduce_path():
    """the in-library NCCL path on one GPU: a 1-rank communicator (the all-reduce is then the
    identity) through fmm_evaluate equals the plain single-GPU evaluation bit for bit"""
    import torch

    from paper_1204_3105_b200 import Comm, Config, Tree, nccl_version

    assert nccl_version() > 0
    w = CASES["C4ts"]
    d = data(w)
    src, u = torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda()
    base = Tree(Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode), src, u)
    a = base.evaluate().cpu().numpy()
    comm = Comm(Comm.unique_id(), 1, 0)
    try:
        cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode, comm=comm)
        t = Tree(cfg, src, u)
        b = t.evaluate().cpu().numpy()
        t.check()
        t.close()
    finally:
        comm.close()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["C2", "C4ts"])
def test_multirank_with_pairing(name, monkeypatch):
    """Ranks 0..2 with the pairing kernel variant forced (TF_PAIR tasks are formed for own row
    leaves only; their two column leaves may belong to other ranks): the union equals the oracle."""
    monkeypatch.setenv("FMM_P2P_PAIRS", "1")
    w = CASES[name]
    d = data(w)
    phi, _, _ = run_ranks(w, d, 3)
    assert not np.isnan(phi).any(), "a target was written by no rank"
    assert normwise(phi, oracle_phi(name)) <= TOL
