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
