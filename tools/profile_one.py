"""One build + evaluate of a single config (for ncu captures): python tools/profile_one.py C4q [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import Config, Tree, X  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4q"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = fi.get(name)
    d = fi.generate(w)
    src = torch.from_numpy(d["src_xy"]).cuda()
    u = torch.from_numpy(d["u"]).cuda()
    tgt = None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda()
    cfg = Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = Tree(cfg, src, u, tgt)
        torch.cuda.synchronize()
        tb = (time.perf_counter() - t0) * 1e3
        t.set_timing(True)
        phi = t.evaluate()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        st = t.stage_times()
        c = t.export(X.COUNTERS)
        print(f"{name} rep {r}: {ms:.2f} ms wall (build {tb:.2f}), upward {st[3]:.3f} down {st[4]:.3f} p2p {st[5]:.3f} (pairs kernel {st[2]:.3f}) ms; "
              f"pairs {c[1]} m2l {c[0]} launches {t.launch_count()}", flush=True)
        t.check()
        t.close()


if __name__ == "__main__":
    main()
