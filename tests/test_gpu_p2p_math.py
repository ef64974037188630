"""GPU (-m gpu): accuracy of the P2P kernel's FP64 log|z|^2 and Arg z (p2p_math.cuh),
through the fmm_debug_p2p_math test hook, against x87 extended-precision libm
(numpy longdouble) and the branch convention of reading D13."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -52


def run_math(dxdy):
    import torch

    from paper_1204_3105_b200 import lib

    L = lib()
    L.fmm_debug_p2p_math.restype = ctypes.c_int
    L.fmm_debug_p2p_math.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    d = torch.from_numpy(np.ascontiguousarray(dxdy, np.float64)).cuda()
    out = torch.empty_like(d)
    rc = L.fmm_debug_p2p_math(ctypes.c_void_p(d.data_ptr()), len(dxdy), ctypes.c_void_p(out.data_ptr()),
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    return out.cpu().numpy()


def reference(dxdy):
    dx = dxdy[:, 0].astype(np.longdouble)
    dy = dxdy[:, 1].astype(np.longdouble)
    lg = np.log(dx * dx + dy * dy)
    dyc = np.where(dxdy[:, 1] == 0.0, np.longdouble(0.0), dy)  # canonical +0 (D13)
    ag = np.arctan2(dyc, dx)
    return lg, ag


def random_offsets(n, seed):
    rng = np.random.default_rng(seed)
    r = np.exp(rng.uniform(np.log(1e-25), np.log(20.0), n))
    th = rng.uniform(-np.pi, np.pi, n)
    return np.stack([r * np.cos(th), r * np.sin(th)], 1)


def check(dxdy, tol_ulps=4.0):
    got = run_math(dxdy)
    lg, ag = reference(dxdy)
    e_lg = np.abs(got[:, 0] - lg.astype(np.float64)) / np.maximum(1.0, np.abs(lg.astype(np.float64)))
    e_ag = np.abs(got[:, 1] - ag.astype(np.float64)) / np.maximum(np.abs(ag.astype(np.float64)), 1e-300)
    assert e_lg.max() <= tol_ulps * ULP, (e_lg.max() / ULP, dxdy[np.argmax(e_lg)])
    assert e_ag.max() <= tol_ulps * ULP, (e_ag.max() / ULP, dxdy[np.argmax(e_ag)])
    return e_lg.max() / ULP, e_ag.max() / ULP


def test_random_offsets_all_magnitudes():
    check(random_offsets(1 << 21, 1))


def test_octant_and_table_boundaries():
    # ratios at and around every table knot k/32 and midpoint (k+1/2)/32, all 8 octants
    t = np.concatenate([np.arange(33) / 32.0, (np.arange(32) + 0.5) / 32.0])
    t = np.concatenate([t, np.nextafter(t, 2), np.nextafter(t, -1)])
    t = t[(t >= 0) & (t <= 1)]
    pts = []
    for sx in (1, -1):
        for sy in (1, -1):
            for swap in (False, True):
                a, b = np.ones_like(t) * 0.37, t * 0.37
                dx, dy = (b, a) if swap else (a, b)
                pts.append(np.stack([sx * dx, sy * dy], 1))
    check(np.concatenate(pts))


def test_axes_signed_zeros_and_branch_cut():
    v = np.array([[1.0, 0.0], [-1.0, 0.0], [-1.0, -0.0], [0.0, 1.0], [-0.0, 1.0], [0.0, -1.0], [-0.0, -1.0],
                  [-2.5, 1e-300], [-2.5, -1e-300], [-1e-3, 1e-18], [-1e-3, -1e-18], [3.0, 3.0], [-3.0, -3.0]])
    got = run_math(v)
    assert got[0, 0] == 0.0 and got[0, 1] == 0.0  # log(1) = 0 and Arg 1 = 0 exactly (self-pair exclusion)
    assert got[1, 1] == np.pi and got[2, 1] == np.pi  # -1 + 0i and -1 - 0i: +pi (D13)
    assert got[3, 1] == np.pi / 2 and got[4, 1] == np.pi / 2
    assert got[5, 1] == -np.pi / 2 and got[6, 1] == -np.pi / 2
    assert got[7, 1] == np.pi and got[8, 1] == -np.pi
    assert got[9, 1] > 3.14 and got[10, 1] < -3.14
    check(v)


def test_near_field_magnitudes():
    # offsets of actual near-field pairs: leaf sizes 2^-9 .. 1, all directions
    rng = np.random.default_rng(7)
    d = (rng.random((1 << 20, 2)) - 0.5) * np.exp(rng.uniform(np.log(2.0 ** -12), 0.0, (1 << 20, 1)))
    check(d)
