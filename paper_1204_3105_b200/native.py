"""ctypes binding of libfmm_b200.so (include/fmm_b200.h): names mirror the C ABI.

Inputs may be torch tensors (CUDA -> device pointers used in place; CPU ->
host pointers staged by the library) or numpy arrays (host).  Argument
marshalling only; no arithmetic of the method happens here.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_PKG, "libfmm_b200.so")

QUADTREE, SEPTREE, TRIQUAD = 0, 1, 2
FLAG_TIMING = 1
_TILING = {"quad": QUADTREE, "sept": SEPTREE, "triq": TRIQUAD, QUADTREE: 0, SEPTREE: 1, TRIQUAD: 2}


class X:
    """export selectors (FMM_X_*)"""
    SRC_KEYS, TGT_KEYS, SRC_PERM, TGT_PERM, SRC_OFFSETS, TGT_OFFSETS = 1, 2, 3, 4, 5, 6
    CENTRES, NEAR_OWNERS, NEAR_OFFSETS, NEAR_ENTRIES = 7, 8, 9, 10
    E4_OWNERS, E4_OFFSETS, E4_ENTRIES, MULTIPOLE, LOCAL, COUNTERS = 11, 12, 13, 14, 15, 16


_DTYPE = {X.SRC_KEYS: np.uint32, X.TGT_KEYS: np.uint32, X.SRC_PERM: np.int32, X.TGT_PERM: np.int32,
          X.SRC_OFFSETS: np.int64, X.TGT_OFFSETS: np.int64, X.CENTRES: np.float64, X.NEAR_OWNERS: np.int32,
          X.NEAR_OFFSETS: np.int64, X.NEAR_ENTRIES: np.int32, X.E4_OWNERS: np.int32, X.E4_OFFSETS: np.int64,
          X.E4_ENTRIES: np.int32, X.MULTIPOLE: np.complex128, X.LOCAL: np.complex128, X.COUNTERS: np.int64}


class Config(C.Structure):
    _fields_ = [("tiling", C.c_int32), ("depth", C.c_int32), ("p", C.c_int32), ("self_mode", C.c_int32),
                ("root_x", C.c_double), ("root_y", C.c_double), ("root_size", C.c_double),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("flags", C.c_int32), ("reserved", C.c_int32 * 5),
                ("comm", C.c_void_p)]

    @classmethod
    def make(cls, tiling, depth, p, root_x, root_y, root_size, self_mode=False, rank=0, nranks=1, timing=False,
             comm=None):
        c = cls(_TILING[tiling], int(depth), int(p), int(bool(self_mode)), float(root_x), float(root_y),
                float(root_size), int(rank), int(nranks), FLAG_TIMING if timing else 0)
        c.comm = None if comm is None else comm.h
        return c


class FmmError(RuntimeError):
    def __init__(self, code, what="", index=-1):
        msg = lib().fmm_error_string(code).decode()
        extra = lib().fmm_last_error_message().decode()
        super().__init__(f"{what}: FMM error {code} ({msg}) {extra} index={index}")
        self.code = code
        self.index = index


_lib = None


def library_path() -> str:
    return _SO


def lib():
    """load libfmm_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(_SO)
        P = C.POINTER
        vp, d = C.c_void_p, P(C.c_double)
        sig = {
            "fmm_build_tree": (C.c_int, [P(Config), vp, vp, C.c_int64, vp, C.c_int64, vp, P(vp)]),
            "fmm_evaluate": (C.c_int, [vp, vp, vp]),
            "fmm_evaluate_begin": (C.c_int, [vp, vp]),
            "fmm_evaluate_end": (C.c_int, [vp, vp, vp]),
            "fmm_multipole_buffer": (C.c_int, [vp, P(vp), P(C.c_size_t)]),
            "fmm_comm_unique_id": (C.c_int, [vp]),
            "fmm_comm_init": (C.c_int, [vp, C.c_int32, C.c_int32, P(vp)]),
            "fmm_comm_destroy": (C.c_int, [vp]),
            "fmm_nccl_version": (C.c_int, []),
            "fmm_set_strengths": (C.c_int, [vp, vp, vp]),
            "fmm_status": (C.c_int, [vp]),
            "fmm_last_error_index": (C.c_int64, [vp]),
            "fmm_export": (C.c_int, [vp, C.c_int32, C.c_int32, vp, C.c_size_t, P(C.c_size_t)]),
            "fmm_set_timing": (C.c_int, [vp, C.c_int32]),
            "fmm_stage_times": (C.c_int, [vp, P(C.c_float)]),
            "fmm_build_times": (C.c_int, [vp, P(C.c_float)]),
            "fmm_rank_range": (C.c_int, [vp, P(C.c_int64), P(C.c_int64)]),
            "fmm_launch_count": (C.c_int64, [vp]),
            "fmm_pool_reserve": (C.c_int, [C.c_size_t]),
            "fmm_tree_bytes": (C.c_size_t, [vp]),
            "fmm_direct": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, C.c_int32, vp, vp]),
            "fmm_sample_cells": (C.c_int, [P(Config), vp, C.c_int64, C.c_int32, C.c_uint64, C.c_int64, vp, vp, vp]),
            "fmm_predict_cost": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int32, vp,
                                           P(C.c_double)]),
            "fmm_choose_depth": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int32, vp, P(C.c_int32)]),
            "fmm_free": (None, [vp]),
            "fmm_release": (C.c_int, [vp]),
            "fmm_error_string": (C.c_char_p, [C.c_int]),
            "fmm_last_error_message": (C.c_char_p, []),
            "fmm_version": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    """(pointer, keepalive) for a torch tensor or numpy array (None -> NULL)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            a = a.contiguous()
        return C.c_void_p(a.data_ptr()), a
    a = np.ascontiguousarray(a)
    return C.c_void_p(a.ctypes.data), a


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Tree:
    """fmm_tree_t: built by fmm_build_tree, evaluated by fmm_evaluate."""

    def __init__(self, cfg: Config, src_xy, src_u, tgt_xy=None, stream=None):
        self.cfg = cfg
        n = int(src_u.shape[0])
        m = n if cfg.self_mode else int(tgt_xy.shape[0])
        self.n, self.m = n, m
        ps, ks = _ptr(src_xy)
        pu, ku = _ptr(src_u)
        pt, kt = _ptr(None if cfg.self_mode else tgt_xy)
        self._keep = (ks, ku, kt)
        self._stream = _stream_ptr(stream)
        h = C.c_void_p()
        rc = lib().fmm_build_tree(C.byref(cfg), ps, pu, n, pt, m, self._stream, C.byref(h))
        if rc:
            raise FmmError(rc, "fmm_build_tree")
        self.h = h

    def release(self):
        """fmm_release: device buffers back to the pool (stream-ordered); timings stay readable"""
        rc = lib().fmm_release(self.h)
        if rc:
            raise FmmError(rc, "fmm_release")

    def close(self):
        if getattr(self, "h", None):
            lib().fmm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def evaluate(self, out=None, stream=None):
        """Phi as complex128 [m] in the caller's target order (torch CUDA tensor by default)."""
        if out is None:
            import torch

            out = torch.zeros(self.m, dtype=torch.complex128, device="cuda")
        po, ko = _ptr(out)
        st = _stream_ptr(stream) if stream is not None else self._stream
        rc = lib().fmm_evaluate(self.h, po, st)
        if rc:
            raise FmmError(rc, "fmm_evaluate")
        return out

    def evaluate_begin(self, stream=None):
        """fmm_evaluate_begin: upward pass over this rank's own leaves (+ the all-reduce when the
        config has a comm) and the P2P pair kernel"""
        st = _stream_ptr(stream) if stream is not None else self._stream
        rc = lib().fmm_evaluate_begin(self.h, st)
        if rc:
            raise FmmError(rc, "fmm_evaluate_begin")

    def evaluate_end(self, out=None, stream=None):
        """fmm_evaluate_end: downward pass, near-field sums and L2P into `out`"""
        if out is None:
            import torch

            out = torch.zeros(self.m, dtype=torch.complex128, device="cuda")
        po, ko = _ptr(out)
        st = _stream_ptr(stream) if stream is not None else self._stream
        rc = lib().fmm_evaluate_end(self.h, po, st)
        if rc:
            raise FmmError(rc, "fmm_evaluate_end")
        return out

    def multipole_buffer(self):
        """(device pointer, bytes) of the multipole tree (fmm_multipole_buffer)"""
        p, nb = C.c_void_p(), C.c_size_t()
        rc = lib().fmm_multipole_buffer(self.h, C.byref(p), C.byref(nb))
        if rc:
            raise FmmError(rc, "fmm_multipole_buffer")
        return p.value, nb.value

    def set_strengths(self, u, stream=None):
        pu, ku = _ptr(u)
        rc = lib().fmm_set_strengths(self.h, pu, _stream_ptr(stream) if stream is not None else self._stream)
        if rc:
            raise FmmError(rc, "fmm_set_strengths")
        self._keep = self._keep + (ku,)

    def status(self):
        rc = lib().fmm_status(self.h)
        return rc, int(lib().fmm_last_error_index(self.h))

    def check(self):
        rc, idx = self.status()
        if rc:
            raise FmmError(rc, "device status", idx)

    def export(self, what, level=0):
        need = C.c_size_t()
        rc = lib().fmm_export(self.h, what, level, None, 0, C.byref(need))
        if rc:
            raise FmmError(rc, "fmm_export")
        dt = np.dtype(_DTYPE[what])
        buf = np.empty(need.value // dt.itemsize, dtype=dt)
        rc = lib().fmm_export(self.h, what, level, C.c_void_p(buf.ctypes.data), buf.nbytes, C.byref(need))
        if rc:
            raise FmmError(rc, "fmm_export")
        return buf

    def set_timing(self, on=True):
        lib().fmm_set_timing(self.h, int(on))

    def stage_times(self):
        ms = (C.c_float * 6)()
        lib().fmm_stage_times(self.h, ms)
        return list(ms)

    def build_times(self):
        """{keys, multi-rank selection, sort + gather, lists + tasks} in ms (fmm_build_times)"""
        ms = (C.c_float * 4)()
        lib().fmm_build_times(self.h, ms)
        return list(ms)

    def rank_range(self):
        lo, hi = C.c_int64(), C.c_int64()
        lib().fmm_rank_range(self.h, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def launch_count(self):
        return int(lib().fmm_launch_count(self.h))

    def nbytes(self):
        """device bytes of the tree's slab (fmm_tree_bytes)"""
        return int(lib().fmm_tree_bytes(self.h))


COMM_ID_BYTES = 128


class Comm:
    """fmm_comm_t: the library's NCCL communicator for one rank (current CUDA device)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        rc = lib().fmm_comm_unique_id(buf)
        if rc:
            raise FmmError(rc, "fmm_comm_unique_id")
        return buf.raw

    def __init__(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != COMM_ID_BYTES:
            raise ValueError("unique id must be 128 bytes")
        h = C.c_void_p()
        rc = lib().fmm_comm_init(C.create_string_buffer(uid, COMM_ID_BYTES), int(nranks), int(rank), C.byref(h))
        if rc:
            raise FmmError(rc, "fmm_comm_init")
        self.h = h.value
        self.nranks, self.rank = int(nranks), int(rank)

    def close(self):
        if getattr(self, "h", None):
            lib().fmm_comm_destroy(self.h)
            self.h = None


def nccl_version() -> int:
    return int(lib().fmm_nccl_version())


def pool_reserve(nbytes: int):
    """grow the stream-ordered pool the trees allocate from (fmm_pool_reserve)"""
    rc = lib().fmm_pool_reserve(int(nbytes))
    if rc:
        raise FmmError(rc, "fmm_pool_reserve")


def direct(src_xy, src_u, tgt_xy=None, self_mode=False, out=None, stream=None):
    """fmm_direct: all-pairs Phi (complex128 [m]); torch CUDA tensor by default."""
    n = int(src_u.shape[0])
    m = n if self_mode else int(tgt_xy.shape[0])
    if out is None:
        import torch

        out = torch.zeros(m, dtype=torch.complex128, device="cuda")
    ps, ks = _ptr(src_xy)
    pu, ku = _ptr(src_u)
    pt, kt = _ptr(None if self_mode else tgt_xy)
    po, ko = _ptr(out)
    rc = lib().fmm_direct(ps, pu, n, pt, m, int(bool(self_mode)), po, _stream_ptr(stream))
    if rc:
        raise FmmError(rc, "fmm_direct")
    return out


def sample_cells(cfg, cells, per_cell, seed, first=0, want_u=True, ncells=None, stream=None):
    """fmm_sample_cells (NEXT-4, Fig. 12): per_cell uniform points in each leaf of
    `cells` (int64 CUDA tensor; None: leaves 0..ncells-1) -> (xy float64 [n, 2], u float64 [n]
    or None), CUDA tensors."""
    import torch

    if cells is not None:
        if not (hasattr(cells, "is_cuda") and cells.is_cuda and cells.dtype == torch.int64):
            raise TypeError("cells must be an int64 CUDA tensor")
        ncells = int(cells.shape[0])
    elif ncells is None:
        ncells = int(cfg_leaves(cfg))
    n = ncells * int(per_cell)
    xy = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    u = torch.empty(n, dtype=torch.float64, device="cuda") if want_u else None
    pc, kc = _ptr(cells)
    px, kx = _ptr(xy)
    pu, ku = _ptr(u)
    rc = lib().fmm_sample_cells(C.byref(cfg), pc, ncells, int(per_cell), C.c_uint64(seed), int(first), px, pu,
                                _stream_ptr(stream))
    if rc:
        raise FmmError(rc, "fmm_sample_cells")
    return xy, u


def cfg_leaves(cfg):
    """B^L leaves of a Config"""
    return (7 if cfg.tiling == SEPTREE else 4) ** int(cfg.depth)


class UnitCosts(C.Structure):
    """fmm_unit_costs: device-time model coefficients (ms per unit)"""
    _fields_ = [("c0", C.c_double), ("c_point", C.c_double), ("c_cell", C.c_double), ("c_pair", C.c_double),
                ("c_leaf", C.c_double)]


def predict_cost(tiling, n, m, p, depth, unit_costs=None):
    out = C.c_double()
    uc = None if unit_costs is None else C.byref(unit_costs)
    rc = lib().fmm_predict_cost(_TILING[tiling], int(n), int(m), int(p), int(depth), uc, C.byref(out))
    if rc:
        raise FmmError(rc, "fmm_predict_cost")
    return out.value


def choose_depth(tiling, n, m, p, unit_costs=None):
    out = C.c_int32()
    uc = None if unit_costs is None else C.byref(unit_costs)
    rc = lib().fmm_choose_depth(_TILING[tiling], int(n), int(m), int(p), uc, C.byref(out))
    if rc:
        raise FmmError(rc, "fmm_choose_depth")
    return out.value
