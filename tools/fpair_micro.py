"""One-pair-per-thread microbenchmark of the P2P pair math (SURVEY §8(d) F_pair): runs the
fmm_debug_p2p_math hook (one (dx, dy) per thread: |z|^2, log|z|^2, Arg z) on n seeded offsets
of the magnitudes a near field sees.  Under ncu its FP64 instruction counts / n give the
per-pair flops of the math; bench.py adds the 6 flops of y - x (2 DADD) and the strength
accumulation (2 DFMA) of a one-sided pair.   usage: python tools/fpair_micro.py [n]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1204_3105_b200 import lib  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    rng = np.random.default_rng(12)
    r = np.exp(rng.uniform(np.log(1e-4), np.log(0.2), n))
    th = rng.uniform(-np.pi, np.pi, n)
    d = torch.from_numpy(np.stack([r * np.cos(th), r * np.sin(th)], 1)).cuda()
    out = torch.empty_like(d)
    L = lib()
    L.fmm_debug_p2p_math.restype = ctypes.c_int
    L.fmm_debug_p2p_math.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    rc = L.fmm_debug_p2p_math(ctypes.c_void_p(d.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0
    print(f"pairs {n}")


if __name__ == "__main__":
    main()
