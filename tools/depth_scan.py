"""NEXT-2 measurement: one workload's build + evaluate time and per-stage times at several tree
depths (same points, same p), to calibrate and check the depth-selection model.
usage: python tools/depth_scan.py C4q 8 9 10 > out.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, Tree, X  # noqa: E402


def main():
    name = sys.argv[1]
    depths = [int(x) for x in sys.argv[2:]]
    w = fi.get(name)
    d = fi.generate(w)
    for L in depths:
        if w.tiling == "sept":
            # the septree domain is the island of the 7^L leaves (reading D8): regenerate the
            # same number of uniform points over the island of this depth
            import dataclasses

            d = fi.generate(dataclasses.replace(w, depth=L))
        src = torch.from_numpy(d["src_xy"]).cuda()
        u = torch.from_numpy(d["u"]).cuda()
        tgt = None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda()
        cfg = Config.make(w.tiling, L, w.p, w.root_x, w.root_y, w.root_size, w.self_mode, timing=True)
        times = []
        for rep in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            t = Tree(cfg, src, u, tgt)
            t.evaluate()
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
            st = t.stage_times()
            c = t.export(X.COUNTERS)
            t.check()
            t.close()
        print(json.dumps({"workload": name, "depth": L, "p": w.p, "n": w.n, "m": w.m, "ms": float(np.median(times)),
                          "build_ms": st[0] + st[1], "upward_ms": st[3], "downward_ms": st[4], "pair_ms": st[2],
                          "p2p_ms": st[5], "m2l_ops": int(c[0]), "pairs": int(c[1]), "src_leaves": int(c[2]),
                          "tgt_leaves": int(c[3])}), flush=True)


if __name__ == "__main__":
    main()
