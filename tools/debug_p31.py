import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FMM_DEBUG_SYNC"] = "1"
import torch, fmm_inputs as fi
from paper_1204_3105_b200 import Config, Tree
for p in (28, 29, 31):
    w = fi.get("C2").scaled(3000)
    d = fi.generate(w)
    cfg = Config.make(w.tiling, w.depth, p, w.root_x, w.root_y, w.root_size, w.self_mode)
    try:
        t = Tree(cfg, torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda())
        phi = t.evaluate()
        print(p, "ok", t.status(), flush=True)
    except Exception as e:
        print(p, "FAIL", e, flush=True)
        break
