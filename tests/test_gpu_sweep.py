"""GPU (-m gpu): the section-9 sweep cases on the CUDA path:
S_opt points per occupied cell (Table 2), the FMM against the GPU direct sum (fmm_direct) and
the oracle FMM, and |Re(Phi_fmm - Phi_direct)| within the per-target bound B_j of reading D14
 built by the oracle."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
import oracle
from gpu_common import normwise

pytestmark = pytest.mark.gpu

FRAMES = {"quad": (0.0, 0.0, 1.0), "sept": (0.0, 0.0, 1.0), "triq": (0.5, math.sqrt(3.0) / 6.0, 1.0 / math.sqrt(3.0))}


@pytest.mark.parametrize("tiling,depth,p", [("quad", 4, 12), ("sept", 3, 12), ("triq", 4, 12), ("sept", 3, 6)])
def test_sweep_case_within_bound(tiling, depth, p):
    import torch

    from paper_1204_3105_b200 import Config, Tree, direct

    rx, ry, rs = FRAMES[tiling]
    s = int(round(fi.s_opt(tiling, 12)))
    d = fi.sweep_generate(tiling, depth, rx, ry, rs, s, 5120 // s, seed=9)
    cfg = Config.make(tiling, depth, p, rx, ry, rs, False)
    src, u, tgt = (torch.from_numpy(d[k]).cuda() for k in ("src_xy", "u", "tgt_xy"))
    t = Tree(cfg, src, u, tgt)
    phi = t.evaluate().cpu().numpy()
    t.check()
    ref = direct(src, u, tgt).cpu().numpy()
    o = oracle.Tree(oracle.config(tiling, depth, p, rx, ry, rs, False), d["src_xy"], d["u"], d["tgt_xy"])
    assert normwise(phi, o.evaluate()) <= 1e-12  # the GPU FMM is the oracle FMM (D15)
    err = np.abs((phi - ref).real)
    bnd = o.bound()
    assert np.all(err <= bnd), (err / bnd).max()
