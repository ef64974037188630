"""NEXT-4 measurement: fmm_sample_cells at BASELINE.json's C4 sizes (all leaves, S points per
leaf, strengths on), CUDA events around the C-ABI call (median of reps; the call itself
synchronises).  Algorithmic HBM bytes per point: 16 (x, y) + 8 (u) written.
usage: python tools/sample_bench.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, sample_cells  # noqa: E402

PER_CELL = {"C4q": 64, "C4s": 143, "C4t": 64}


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    for name, pc in PER_CELL.items():
        w = fi.get(name)
        cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, True)
        ts = []
        for _ in range(reps + 2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            xy, u = sample_cells(cfg, None, pc, seed=7)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            del xy, u
        ms = float(np.median(ts[2:]))
        n = (7 if w.tiling == "sept" else 4) ** w.depth * pc
        print(json.dumps({"workload": name, "points": n, "ms": ms, "points_per_s": n / ms * 1e3,
                          "GB_per_s": 24.0 * n / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
