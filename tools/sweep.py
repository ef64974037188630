"""Section-9 sweeps of the paper (Figs 13-16) on one B200:

  * runtime and max |Re(Phi_fmm - Phi_direct)| vs N = M at p = 12, two depths per tiling, with
    S_opt (Table 2) points per occupied cell and N varied by the number of occupied cells;
  * runtime and max error vs p at N = M = 5120.

FMM time = fmm_build_tree + fmm_evaluate, direct time = fmm_direct, both from CUDA events (median
of `reps`), device-resident inputs.  Errors compare the real part only (reading D13: Im of the
direct sum carries per-pair principal branches).  Writes one JSON document.
usage: python tools/sweep.py [out.json] [reps]"""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, Tree, direct  # noqa: E402

FRAMES = {"quad": (0.0, 0.0, 1.0), "sept": (0.0, 0.0, 1.0), "triq": (0.5, math.sqrt(3.0) / 6.0, 1.0 / math.sqrt(3.0))}
DEPTHS = {"quad": (5, 6), "sept": (3, 4), "triq": (5, 6)}
B = {"quad": 4, "sept": 7, "triq": 4}


def timed(fn, reps):
    ts = []
    out = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


def run_case(tiling, depth, p, per_cell, n_cells, seed, reps):
    rx, ry, rs = FRAMES[tiling]
    d = fi.sweep_generate(tiling, depth, rx, ry, rs, per_cell, n_cells, seed)
    src = torch.from_numpy(d["src_xy"]).cuda()
    u = torch.from_numpy(d["u"]).cuda()
    tgt = torch.from_numpy(d["tgt_xy"]).cuda()
    cfg = Config.make(tiling, depth, p, rx, ry, rs, False)

    def fmm():
        t = Tree(cfg, src, u, tgt)
        phi = t.evaluate()
        t.close()
        return phi

    t_fmm, phi = timed(fmm, reps)
    t_dir, ref = timed(lambda: direct(src, u, tgt), max(1, reps // 2))
    err = float((phi.real - ref.real).abs().max().item())
    return {"tiling": tiling, "depth": depth, "p": p, "n": len(d["u"]), "occupied_cells": n_cells,
            "per_cell": per_cell, "fmm_ms": t_fmm, "direct_ms": t_dir, "max_abs_err_re": err}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.json"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    res = {"n_sweep": [], "p_sweep": []}
    # N sweep at p = 12: S_opt points per cell, occupied cells from 1/64 of the leaves to all
    for tiling, depths in DEPTHS.items():
        s = int(round(fi.s_opt(tiling, 12)))
        for depth in depths:
            K = B[tiling] ** depth
            for frac in (1 / 64, 1 / 16, 1 / 4, 1.0):
                n_cells = max(1, int(K * frac))
                r = run_case(tiling, depth, 12, s, n_cells, 7, reps)
                res["n_sweep"].append(r)
                print(json.dumps(r), flush=True)
    # p sweep at N = M = 5120 (S_opt(12) per cell; occupied cells = 5120 / S_opt, depth with
    # enough cells)
    for tiling, depth in (("quad", 4), ("sept", 3), ("triq", 4)):
        s = int(round(fi.s_opt(tiling, 12)))
        n_cells = 5120 // s
        for p in (2, 4, 6, 8, 10, 12, 16, 20, 24, 28):
            r = run_case(tiling, depth, p, s, n_cells, 9, reps)
            res["p_sweep"].append(r)
            print(json.dumps(r), flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
