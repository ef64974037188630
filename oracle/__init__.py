"""ctypes binding of the CPU ORACLE (oracle/fmm_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_1204_3105_b200) never imports it.  Argument marshalling only: every
number is computed in fmm_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "fmm_oracle.c")

QUAD, SEPT, TRIQ = 0, 1, 2
TILING = {"quad": QUAD, "sept": SEPT, "triq": TRIQ}
OK, EBADCFG, EDOMAIN, ECOINCIDENT, ENOMEM = 0, 1, 2, 3, 5


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "fmm_oracle.h"))
    ):
        cmd = ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd, cwd=_HERE)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Config(C.Structure):
    _fields_ = [("tiling", C.c_int32), ("depth", C.c_int32), ("p", C.c_int32), ("self_mode", C.c_int32),
                ("root_x", C.c_double), ("root_y", C.c_double), ("root_size", C.c_double)]


_lib = None
_P = C.POINTER
_d = _P(C.c_double)
_i32 = _P(C.c_int32)
_i64 = _P(C.c_int64)
_u32 = _P(C.c_uint32)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        cfgp = _P(Config)
        sig = {
            "orc_gbt_add": (C.c_int, [_i32, C.c_int32, _i32, C.c_int32, _i32]),
            "orc_gbt_negate": (C.c_int, [_i32, C.c_int32, _i32]),
            "orc_gbt_zero_extend": (C.c_int, [C.c_int32, C.c_int32, _i32]),
            "orc_gbt_index_add": (C.c_int, [C.c_int64, C.c_int64, _i64]),
            "orc_num_cells": (C.c_int64, [cfgp, C.c_int32]),
            "orc_neighbors": (C.c_int, [cfgp, C.c_int32, C.c_int64, _i64]),
            "orc_neighbors_e4": (C.c_int, [cfgp, C.c_int32, C.c_int64, _i64]),
            "orc_triq_adjacent": (C.c_int64, [C.c_int32, C.c_int64, C.c_int32]),
            "orc_triq_isup": (C.c_int, [C.c_int64, C.c_int32, C.c_int32]),
            "orc_cell_center": (None, [cfgp, C.c_int32, C.c_int64, _d]),
            "orc_cell_center_polar": (None, [cfgp, C.c_int32, C.c_int64, _d]),
            "orc_keys": (C.c_int, [cfgp, _d, C.c_int64, _u32, _i64]),
            "orc_cell_index": (C.c_int, [cfgp, C.c_double, C.c_double, C.c_int32, _i64]),
            "orc_p2m": (None, [_d, _d, C.c_int64, _d, C.c_int32, _d]),
            "orc_m2m": (None, [_d, _d, _d, C.c_int32, _d]),
            "orc_m2l": (None, [_d, _d, _d, C.c_int32, _d]),
            "orc_l2l": (None, [_d, _d, _d, C.c_int32, _d]),
            "orc_l2p": (None, [_d, _d, C.c_int32, _d, _d]),
            "orc_log": (None, [C.c_double, C.c_double, _d]),
            "orc_direct": (C.c_int, [_d, _d, C.c_int64, _d, C.c_int64, C.c_int32, _i64, C.c_int64, _d, _i64]),
            "orc_tree_build": (C.c_int, [cfgp, _d, _d, C.c_int64, _d, C.c_int64, _P(C.c_void_p), _i64]),
            "orc_tree_free": (None, [C.c_void_p]),
            "orc_tree_keys": (None, [C.c_void_p, _u32, _u32]),
            "orc_tree_perm": (None, [C.c_void_p, _i32, _i32]),
            "orc_tree_leaf_offsets": (None, [C.c_void_p, _i64, _i64]),
            "orc_tree_count": (C.c_int64, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32]),
            "orc_tree_near": (C.c_int, [C.c_void_p, C.c_int64, _i64]),
            "orc_tree_e4": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, _i64]),
            "orc_tree_near_csr": (C.c_int, [C.c_void_p, _i32, _i64, _i32, _i64, _i64]),
            "orc_tree_e4_csr": (C.c_int, [C.c_void_p, C.c_int32, _i32, _i64, _i32, _i64, _i64]),
            "orc_tree_centres": (None, [C.c_void_p, C.c_int32, _d]),
            "orc_tree_upward": (None, [C.c_void_p]),
            "orc_tree_multipole": (None, [C.c_void_p, C.c_int32, C.c_int64, _d]),
            "orc_tree_multipoles_level": (None, [C.c_void_p, C.c_int32, _d]),
            "orc_tree_local": (None, [C.c_void_p, C.c_int32, C.c_int64, _d]),
            "orc_tree_evaluate": (C.c_int, [C.c_void_p, _i64, C.c_int64, _d, _i64, _i64]),
            "orc_tree_bound": (None, [C.c_void_p, _i64, C.c_int64, _d]),
            "orc_num_threads": (C.c_int, []),
            "orc_set_num_threads": (None, [C.c_int]),
            "orc_paper_cost": (C.c_double, [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]),
            "orc_paper_depth": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]),
            "orc_draw": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_sample_cells": (C.c_int, [cfgp, _i64, C.c_int64, C.c_int32, C.c_uint64, C.c_int64, _d, _d]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, index=-1):
        super().__init__(f"oracle error {code} (index {index})")
        self.code = code
        self.index = index


def config(tiling, depth, p, root_x, root_y, root_size, self_mode=False) -> Config:
    t = TILING[tiling] if isinstance(tiling, str) else int(tiling)
    return Config(t, int(depth), int(p), int(bool(self_mode)), float(root_x), float(root_y), float(root_size))


# ---------------------------------------------------------------- GBT helpers
def _digits_lsb(n: int):
    d = []
    while True:
        d.append(n % 7)
        n //= 7
        if n == 0:
            return d


def gbt_add(a: int, b: int) -> int:
    """a (*) b for base-7 integers given as Python ints written in base 10 digits of base 7 (e.g. 14 -> '14'_7)."""
    out = C.c_int64()
    rc = lib().orc_gbt_index_add(int(str(a), 7), int(str(b), 7), C.byref(out))
    if rc:
        raise OracleError(rc)
    return int(np.base_repr(out.value, 7))


def gbt_negate(a: int) -> int:
    d = np.array(_digits_lsb(int(str(a), 7)), dtype=np.int32)
    out = np.zeros(64, np.int32)
    n = lib().orc_gbt_negate(_ptr(d, _i32), len(d), _ptr(out, _i32))
    v = 0
    for k in range(n - 1, -1, -1):
        v = v * 7 + int(out[k])
    return int(np.base_repr(v, 7))


def gbt_zero_extend(j: int, m: int) -> int:
    out = np.zeros(64, np.int32)
    n = lib().orc_gbt_zero_extend(j, m, _ptr(out, _i32))
    v = 0
    for k in range(n - 1, -1, -1):
        v = v * 7 + int(out[k])
    return int(np.base_repr(v, 7))


# ---------------------------------------------------------------- tiling
def num_cells(cfg, level):
    return lib().orc_num_cells(C.byref(cfg), level)


def neighbors(cfg, level, n):
    out = np.zeros(16, np.int64)
    k = lib().orc_neighbors(C.byref(cfg), level, n, _ptr(out, _i64))
    return [int(v) for v in out[:k]]


def neighbors_e4(cfg, level, n):
    out = np.zeros(128, np.int64)
    k = lib().orc_neighbors_e4(C.byref(cfg), level, n, _ptr(out, _i64))
    return [int(v) for v in out[:k]]


def triq_adjacent(level, n, k):
    return int(lib().orc_triq_adjacent(level, n, k))


def triq_isup(t, ndigits, level):
    return int(lib().orc_triq_isup(t, ndigits, level))


def cell_center(cfg, level, n):
    xy = np.zeros(2)
    lib().orc_cell_center(C.byref(cfg), level, n, _ptr(xy, _d))
    return xy


def cell_center_polar(cfg, level, n):
    xy = np.zeros(2)
    lib().orc_cell_center_polar(C.byref(cfg), level, n, _ptr(xy, _d))
    return xy


def cell_index(cfg, x, y, level):
    out = C.c_int64()
    rc = lib().orc_cell_index(C.byref(cfg), float(x), float(y), level, C.byref(out))
    if rc:
        raise OracleError(rc)
    return int(out.value)


def keys_all(cfg, xy):
    """keys of every point, out-of-domain points as 0xffffffff (no error raised)"""
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    k = np.zeros(len(xy), np.uint32)
    bad = C.c_int64(-1)
    lib().orc_keys(C.byref(cfg), _ptr(xy, _d), len(xy), _ptr(k, _u32), C.byref(bad))
    return k


def keys(cfg, xy):
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    k = np.zeros(len(xy), np.uint32)
    bad = C.c_int64(-1)
    rc = lib().orc_keys(C.byref(cfg), _ptr(xy, _d), len(xy), _ptr(k, _u32), C.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return k


# ---------------------------------------------------------------- operators
def _cz(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a


def p2m(xy, u, c, p):
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    u = np.ascontiguousarray(u, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    mp = np.zeros(p + 1, np.complex128)
    lib().orc_p2m(_ptr(xy, _d), _ptr(u, _d), len(u), _ptr(c, _d), p, mp.ctypes.data_as(_d))
    return mp


def m2m(mp_child, c_child, c_parent, p, acc=None):
    acc = np.zeros(p + 1, np.complex128) if acc is None else _cz(acc).copy()
    mpc = _cz(mp_child)
    lib().orc_m2m(mpc.ctypes.data_as(_d), _ptr(np.asarray(c_child, float), _d),
                  _ptr(np.asarray(c_parent, float), _d), p, acc.ctypes.data_as(_d))
    return acc


def m2l(mp, c_m, c_l, p, acc=None):
    acc = np.zeros(p + 1, np.complex128) if acc is None else _cz(acc).copy()
    mpc = _cz(mp)
    lib().orc_m2l(mpc.ctypes.data_as(_d), _ptr(np.asarray(c_m, float), _d), _ptr(np.asarray(c_l, float), _d),
                  p, acc.ctypes.data_as(_d))
    return acc


def l2l(loc_parent, c_parent, c_child, p):
    out = np.zeros(p + 1, np.complex128)
    lp = _cz(loc_parent)
    lib().orc_l2l(lp.ctypes.data_as(_d), _ptr(np.asarray(c_parent, float), _d),
                  _ptr(np.asarray(c_child, float), _d), p, out.ctypes.data_as(_d))
    return out


def l2p(loc, c, p, y):
    out = np.zeros(2)
    lc = _cz(loc)
    lib().orc_l2p(lc.ctypes.data_as(_d), _ptr(np.asarray(c, float), _d), p, _ptr(np.asarray(y, float), _d),
                  _ptr(out, _d))
    return complex(out[0], out[1])


def log(dx, dy):
    out = np.zeros(2)
    lib().orc_log(float(dx), float(dy), _ptr(out, _d))
    return complex(out[0], out[1])


def direct(src_xy, u, tgt_xy=None, self_mode=False, tgt_ids=None):
    src_xy = np.ascontiguousarray(src_xy, dtype=np.float64).reshape(-1, 2)
    u = np.ascontiguousarray(u, dtype=np.float64)
    tgt_xy = src_xy if (self_mode or tgt_xy is None) else np.ascontiguousarray(tgt_xy, np.float64).reshape(-1, 2)
    ids = None if tgt_ids is None else np.ascontiguousarray(tgt_ids, dtype=np.int64)
    nt = len(tgt_xy) if ids is None else len(ids)
    phi = np.zeros(nt, np.complex128)
    bad = C.c_int64(-1)
    rc = lib().orc_direct(_ptr(src_xy, _d), _ptr(u, _d), len(u), _ptr(tgt_xy, _d), len(tgt_xy), int(self_mode),
                          _ptr(ids, _i64), nt, phi.ctypes.data_as(_d), C.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return phi


# ---------------------------------------------------------------- tree
class Tree:
    """The oracle FMM over one input set."""

    def __init__(self, cfg: Config, src_xy, u, tgt_xy=None):
        self.cfg = cfg
        self.src_xy = np.ascontiguousarray(src_xy, dtype=np.float64).reshape(-1, 2)
        self.u = np.ascontiguousarray(u, dtype=np.float64)
        if cfg.self_mode or tgt_xy is None:
            self.tgt_xy = self.src_xy
        else:
            self.tgt_xy = np.ascontiguousarray(tgt_xy, dtype=np.float64).reshape(-1, 2)
        self.n, self.m = len(self.u), len(self.tgt_xy)
        self.B = 7 if cfg.tiling == SEPT else 4
        self.L, self.p = cfg.depth, cfg.p
        h = C.c_void_p()
        bad = C.c_int64(-1)
        rc = lib().orc_tree_build(C.byref(cfg), _ptr(self.src_xy, _d), _ptr(self.u, _d), self.n,
                                  _ptr(self.tgt_xy, _d), self.m, C.byref(h), C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_tree_free(h)
            self.h = None

    def keys(self):
        sk = np.zeros(self.n, np.uint32)
        tk = np.zeros(self.m, np.uint32)
        lib().orc_tree_keys(self.h, _ptr(sk, _u32), _ptr(tk, _u32))
        return sk, tk

    def perm(self):
        sp = np.zeros(self.n, np.int32)
        tp = np.zeros(self.m, np.int32)
        lib().orc_tree_perm(self.h, _ptr(sp, _i32), _ptr(tp, _i32))
        return sp, tp

    def leaf_offsets(self):
        K = self.B ** self.L
        so = np.zeros(K + 1, np.int64)
        to = np.zeros(K + 1, np.int64)
        lib().orc_tree_leaf_offsets(self.h, _ptr(so, _i64), _ptr(to, _i64))
        return so, to

    def count(self, level, cell, which=0):
        return int(lib().orc_tree_count(self.h, level, cell, which))

    def near(self, leaf):
        out = np.zeros(16, np.int64)
        k = lib().orc_tree_near(self.h, leaf, _ptr(out, _i64))
        return out[:k].copy()

    def e4(self, level, cell):
        out = np.zeros(128, np.int64)
        k = lib().orc_tree_e4(self.h, level, cell, _ptr(out, _i64))
        return out[:k].copy()

    def _csr(self, level):
        no, ne = C.c_int64(), C.c_int64()
        if level is None:
            lib().orc_tree_near_csr(self.h, None, None, None, C.byref(no), C.byref(ne))
        else:
            lib().orc_tree_e4_csr(self.h, level, None, None, None, C.byref(no), C.byref(ne))
        ow = np.zeros(no.value, np.int32)
        of = np.zeros(no.value + 1, np.int64)
        en = np.zeros(ne.value, np.int32)
        if level is None:
            lib().orc_tree_near_csr(self.h, _ptr(ow, _i32), _ptr(of, _i64), _ptr(en, _i32), C.byref(no), C.byref(ne))
        else:
            lib().orc_tree_e4_csr(self.h, level, _ptr(ow, _i32), _ptr(of, _i64), _ptr(en, _i32), C.byref(no),
                                  C.byref(ne))
        return ow, of, en

    def near_csr(self):
        return self._csr(None)

    def e4_csr(self, level):
        return self._csr(level)

    def centres(self, level):
        xy = np.zeros((self.B ** level, 2))
        lib().orc_tree_centres(self.h, level, _ptr(xy, _d))
        return xy

    def upward(self):
        lib().orc_tree_upward(self.h)

    def multipole(self, level, cell):
        self.upward()
        mp = np.zeros(self.p + 1, np.complex128)
        lib().orc_tree_multipole(self.h, level, cell, mp.ctypes.data_as(_d))
        return mp

    def multipoles(self, level):
        mp = np.zeros((self.B ** level, self.p + 1), np.complex128)
        lib().orc_tree_multipoles_level(self.h, level, mp.ctypes.data_as(_d))
        return mp

    def local(self, level, cell):
        loc = np.zeros(self.p + 1, np.complex128)
        lib().orc_tree_local(self.h, level, cell, loc.ctypes.data_as(_d))
        return loc

    def evaluate(self, tgt_ids=None, counters=False):
        ids = None if tgt_ids is None else np.ascontiguousarray(tgt_ids, dtype=np.int64)
        nt = self.m if ids is None else len(ids)
        phi = np.zeros(nt, np.complex128)
        bad = C.c_int64(-1)
        cnt = np.zeros(2, np.int64)
        rc = lib().orc_tree_evaluate(self.h, _ptr(ids, _i64), nt, phi.ctypes.data_as(_d), C.byref(bad),
                                     _ptr(cnt, _i64))
        if rc:
            raise OracleError(rc, bad.value)
        return (phi, {"m2l_ops": int(cnt[0]), "p2p_pairs": int(cnt[1])}) if counters else phi

    def bound(self, tgt_ids=None):
        ids = None if tgt_ids is None else np.ascontiguousarray(tgt_ids, dtype=np.int64)
        nt = self.m if ids is None else len(ids)
        b = np.zeros(nt)
        lib().orc_tree_bound(self.h, _ptr(ids, _i64), nt, _ptr(b, _d))
        return b


def num_threads():
    return int(lib().orc_num_threads())


def set_num_threads(n):
    """OpenMP thread count of the oracle's parallel loops (results do not depend on it)"""
    lib().orc_set_num_threads(int(n))


def paper_cost(tiling, n, m, p, depth):
    """appendix A-C cost model (NEXT-2), without the L-independent constant"""
    return float(lib().orc_paper_cost(TILING[tiling], float(n), float(m), int(p), int(depth)))


def paper_depth(tiling, n, m, p, maxdepth):
    return int(lib().orc_paper_depth(TILING[tiling], float(n), float(m), int(p), int(maxdepth)))


def draw(seed, counter):
    """counter-based draw h(seed, counter) of the NEXT-4 sampler (D22)"""
    return int(lib().orc_draw(C.c_uint64(seed), C.c_uint64(counter)))


def sample_cells(cfg, cells, per_cell, seed, first=0, want_u=True):
    """NEXT-4 regular-polygon point picking (Fig. 12; D22): per_cell points in each
    leaf of `cells` (None: leaves 0..K-1) -> (xy (n, 2), u (n,) or None)"""
    if cells is None:
        ncells = int(lib().orc_num_cells(C.byref(cfg), cfg.depth))
        cp = None
    else:
        cells = np.ascontiguousarray(cells, np.int64)
        ncells = len(cells)
        cp = _ptr(cells, _i64)
    n = ncells * int(per_cell)
    xy = np.zeros((n, 2))
    u = np.zeros(n) if want_u else None
    rc = lib().orc_sample_cells(C.byref(cfg), cp, ncells, int(per_cell), C.c_uint64(seed), int(first),
                                _ptr(xy, _d), _ptr(u, _d) if want_u else None)
    if rc:
        raise OracleError(rc)
    return xy, u
