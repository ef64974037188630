"""Multi-rank host logic on CPU (gloo, world size 2 and 4): the work-balanced target-leaf
partition used when fmm_config.nranks > 1.  Each rank calls
fmm_partition (the library's host function) for its own rank; the ranges are
all-gathered over torch.distributed/gloo and must tile [0, K) contiguously, disjointly,
with every rank's work within one block of the ideal share."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _weights(kind, nb, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(0.9, 1.1, nb) * 4096.0
    if kind == "clustered":  # C5-like: a few very heavy blocks, many empty ones
        w = np.zeros(nb)
        idx = rng.choice(nb, size=max(1, nb // 20), replace=False)
        w[idx] = rng.pareto(1.5, len(idx)) * 1e5 + 1e3
        return w
    return np.zeros(nb)


def _worker(rank, world, port, kind, nb, K, q):
    import torch

    from paper_1204_3105_b200 import lib

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = lib()
    L.fmm_partition.restype = ctypes.c_int
    L.fmm_partition.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    w = np.ascontiguousarray(_weights(kind, nb))
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    rc = L.fmm_partition(w.ctypes.data, nb, 256, K, rank, world, ctypes.byref(lo), ctypes.byref(hi))
    t = torch.tensor([rc, lo.value, hi.value], dtype=torch.int64)
    out = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        q.put([o.tolist() for o in out])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["uniform", "clustered", "empty"])
def test_partition_tiles_leaf_range(world, kind):
    nb, K = 1024, 1024 * 256 - 77  # ragged last block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, nb, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] == 0 for r in res)
    ranges = [(r[1], r[2]) for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == K
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]  # contiguous and disjoint
    w = _weights(kind, nb)
    W = w.sum()
    if W > 0:
        for lo, hi in ranges:
            share = w[lo // 256:(hi + 255) // 256].sum()
            assert abs(share - W / world) <= w.max() + 1e-9 * W


# ---------------------------------------------------------------- the multipole exchange (gloo)
def _exchange_worker(rank, world, port, name, q):
    """rank r: its work-balanced leaf range (the library's fmm_partition on the block-work
    estimate), P2M over its own source leaves and M2M of those partial
    expansions up every level (oracle operators, App. B.2/B.3), all other cells zero; the
    per-level multipole trees are then summed over the ranks with a gloo all_reduce -- the
    exchange fmm_evaluate does with ncclAllReduce.  Rank 0 reports the summed
    tree."""
    import torch

    import fmm_inputs as fi
    import oracle
    from paper_1204_3105_b200 import lib

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = {"C1": fi.get("C1"), "C2s": fi.get("C2").scaled(6000, name="C2s")}[name]
    d = fi.generate(w)
    cfg = oracle.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    T = oracle.Tree(cfg, d["src_xy"], d["u"], d["tgt_xy"])
    B = 7 if w.tiling == "sept" else 4
    K = B ** w.depth
    so, to = T.leaf_offsets()
    ns, nt = np.diff(so), np.diff(to)
    # a block-work estimate over 256-leaf blocks (the build uses near-list sums per 32-leaf block)
    P2 = {"quad": 9, "sept": 7, "triq": 13}[w.tiling]
    lw = np.where(nt > 0, nt * ns * float(P2) + 2.0 * (w.p + 1) * nt + 40.0 * (w.p + 1) ** 2, 0.0)
    nb = (K + 255) // 256
    bw = np.ascontiguousarray([lw[b * 256:(b + 1) * 256].sum() for b in range(nb)])
    L = lib()
    L.fmm_partition.restype = ctypes.c_int
    L.fmm_partition.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    assert L.fmm_partition(bw.ctypes.data, nb, 256, K, rank, world, ctypes.byref(lo), ctypes.byref(hi)) == 0
    lo, hi = lo.value, hi.value
    perm, _ = T.perm()
    sxy, su = d["src_xy"][perm], d["u"][perm]
    cen = [T.centres(l) for l in range(w.depth + 1)]
    mp = [np.zeros((B ** l, w.p + 1), np.complex128) for l in range(w.depth + 1)]
    for leaf in range(lo, hi):
        if ns[leaf]:
            mp[w.depth][leaf] = oracle.p2m(sxy[so[leaf]:so[leaf + 1]], su[so[leaf]:so[leaf + 1]], cen[w.depth][leaf],
                                          w.p)
    for l in range(w.depth - 1, 0, -1):
        span = B ** (w.depth - l)
        for c in range(lo // span, (hi + span - 1) // span if hi > lo else 0):
            acc = np.zeros(w.p + 1, np.complex128)
            for ch in range(c * B, c * B + B):
                acc = oracle.m2m(mp[l + 1][ch], cen[l + 1][ch], cen[l][c], w.p, acc)
            mp[l][c] = acc
    flat = torch.from_numpy(np.concatenate([m.view(np.float64).ravel() for m in mp[1:]]))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((lo, hi, flat.numpy()))
    else:
        q.put((lo, hi, None))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["C1", "C2s"])
def test_gloo_multipole_exchange(world, name):
    """the sum over ranks of the partial multipole trees equals the single-tree oracle
    multipoles at every level (M2M is linear; only the FP64 summation order changes, so the
    D15 normwise gate applies)"""
    import fmm_inputs as fi
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = sorted((lo, hi) for lo, hi, _ in res)
    flat = [f for _, _, f in res if f is not None][0]
    w = {"C1": fi.get("C1"), "C2s": fi.get("C2").scaled(6000, name="C2s")}[name]
    B = 7 if w.tiling == "sept" else 4
    assert ranges[0][0] == 0 and ranges[-1][1] == B ** w.depth
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    d = fi.generate(w)
    T = oracle.Tree(oracle.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode),
                    d["src_xy"], d["u"], d["tgt_xy"])
    T.upward()
    got = flat.view(np.complex128)
    off = 0
    for l in range(1, w.depth + 1):
        ref = T.multipoles(l)
        g = got[off:off + ref.size].reshape(ref.shape)
        off += ref.size
        assert np.abs(g - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1.0), l
