"""One small build + evaluate per case through the C ABI, for compute-sanitizer runs
(racecheck / memcheck / synccheck): C1 (septree, distinct targets) and C2 at 8,192 self points
(triangle-quadtree, symmetric near field), plus a 2-rank sequential multi-rank pass of C2-small.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, Tree  # noqa: E402


def main():
    cases = [fi.get("C1"), fi.get("C2").scaled(8192, name="C2-smoke")]
    for w in cases:
        d = fi.generate(w)
        cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
        tgt = None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda()
        t = Tree(cfg, torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda(), tgt)
        phi = t.evaluate()
        torch.cuda.synchronize()
        t.check()
        print(w.name, "ok", float(np.abs(phi.cpu().numpy()).max()), flush=True)
        t.close()
    # two ranks of C2-smoke one after another (partial multipoles summed here)
    w = cases[1]
    d = fi.generate(w)
    src, u = torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda()
    trees = []
    for r in range(2):
        cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode, rank=r, nranks=2)
        t = Tree(cfg, src, u)
        t.evaluate_begin()
        trees.append(t)
    torch.cuda.synchronize()
    print("multi-rank begin ok", flush=True)
    for t in trees:
        t.close()


if __name__ == "__main__":
    main()
