"""The section-9 sweep generator (fmm_inputs.sweep_generate): every point lies
in one of the chosen occupied leaves (oracle keys), each occupied leaf holds exactly
per_cell sources and per_cell targets, and Table 2's S_opt."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
import oracle

FRAMES = {
    "quad": (0.0, 0.0, 1.0),
    "sept": (0.0, 0.0, 1.0),
    "triq": (0.5, math.sqrt(3.0) / 6.0, 1.0 / math.sqrt(3.0)),
}


@pytest.mark.parametrize("tiling,depth", [("quad", 3), ("sept", 2), ("triq", 3)])
def test_points_fill_the_occupied_leaves(tiling, depth):
    rx, ry, rs = FRAMES[tiling]
    per, ncell = 17, 11
    d = fi.sweep_generate(tiling, depth, rx, ry, rs, per, ncell, seed=5)
    cfg = oracle.config(tiling, depth, 4, rx, ry, rs, False)
    t = oracle.Tree(cfg, d["src_xy"], d["u"], d["tgt_xy"])
    sk, tk = t.keys()
    K = {"quad": 4, "sept": 7, "triq": 4}[tiling] ** depth
    assert sk.max() < K and tk.max() < K  # all in the domain
    for keys in (sk, tk):
        leaves, counts = np.unique(keys, return_counts=True)
        assert len(leaves) == ncell and np.all(counts == per)
    assert set(np.unique(sk)) == set(np.unique(tk))


def test_s_opt_table2():
    assert fi.s_opt("quad", 12) == pytest.approx(12 * math.sqrt(116 / 27))
    assert fi.s_opt("sept", 12) == pytest.approx(12 * math.sqrt(308 / 42))
    assert fi.s_opt("triq", 12) == pytest.approx(12 * math.sqrt(164 / 39))
