"""NEXT-1 at GPU scale with the NEXT-4 device sampler: runtime and max error vs N at p = 12 for
full trees of S_opt (Table 2) points per leaf, sources and distinct targets drawn on the device
by fmm_sample_cells.  FMM time = fmm_build_tree + fmm_evaluate (CUDA events,
median of 3).  The error is max |Re(Phi_fmm - Phi_direct)| over 4096 random targets (direct sum
over all sources for those targets); the full direct time is measured up to N = 1.7M and
extrapolated quadratically (O(N M)) from the largest measured N of the tiling above that.
usage: python tools/sweep_large.py > profiles/r01/sweep_large.jsonl"""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, Tree, direct, sample_cells  # noqa: E402

FRAMES = {"quad": (0.0, 0.0, 1.0), "sept": (0.0, 0.0, 1.0), "triq": (0.5, math.sqrt(3.0) / 6.0, 1.0 / math.sqrt(3.0))}
DEPTHS = {"quad": (5, 6, 7, 8, 9), "sept": (3, 4, 5, 6, 7), "triq": (5, 6, 7, 8, 9)}


def timed(fn, reps):
    ts, out = [], None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


def main():
    p = 12
    for tiling, depths in DEPTHS.items():
        s = int(round(fi.s_opt(tiling, p)))
        last = None  # (n, direct ms) of the largest measured direct sum
        for L in depths:
            rx, ry, rs = FRAMES[tiling]
            cfg = Config.make(tiling, L, p, rx, ry, rs, False)
            src, u = sample_cells(cfg, None, s, seed=11)
            tgt, _ = sample_cells(cfg, None, s, seed=12, want_u=False)
            n = src.shape[0]

            def fmm():
                t = Tree(cfg, src, u, tgt)
                phi = t.evaluate()
                t.close()
                return phi

            t_fmm, phi = timed(fmm, 3)
            idx = torch.from_numpy(np.random.default_rng(L).choice(n, size=min(4096, n), replace=False)).cuda()
            sub = tgt[idx].contiguous()
            t_sub, ref = timed(lambda: direct(src, u, sub), 1)
            err = float((phi[idx].real - ref.real).abs().max().item())
            if n <= 1_700_000:
                t_dir, _ = timed(lambda: direct(src, u, tgt), 1)
                kind = "measured"
                last = (n, t_dir)
            else:
                t_dir, kind = last[1] * (n / last[0]) ** 2, f"extrapolated as N^2 from N = {last[0]}"
            print(json.dumps({"tiling": tiling, "depth": L, "p": p, "per_leaf": s, "n": n, "m": n,
                              "fmm_ms": t_fmm, "direct_ms": t_dir, "direct_kind": kind,
                              "max_abs_err_re_4096": err}), flush=True)
            del src, u, tgt, phi
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
