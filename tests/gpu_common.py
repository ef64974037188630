"""Helpers shared by the -m gpu parity tests: build the CUDA tree (through the C ABI)
and the oracle tree on the same seeded inputs."""
import numpy as np

import fmm_inputs as fi

# parity cases the oracle finishes in seconds: full C1 / C2, the big configs scaled down
# (same domain, depth, p and distribution; several tiles and ragged tails)
SMALL_CASES = {
    "C1": fi.get("C1"),
    "C2": fi.get("C2"),
    "C3s": fi.get("C3").scaled(40000, 37001, "C3s"),
    "C4qs": fi.get("C4q").scaled(60001, name="C4qs"),
    "C4ss": fi.get("C4s").scaled(60001, name="C4ss"),
    "C4ts": fi.get("C4t").scaled(60001, name="C4ts"),
    "C5s": fi.get("C5").scaled(50000, name="C5s"),
}

_DATA = {}


def data(w):
    key = (w.name, w.n, w.m, w.seed)
    if key not in _DATA:
        _DATA[key] = fi.generate(w)
    return _DATA[key]


def gpu_tree(w, d, host_inputs=False, p=None, depth=None):
    import torch

    from paper_1204_3105_b200 import Config, Tree

    cfg = Config.make(w.tiling, depth or w.depth, p or w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    if host_inputs:
        src, u, tgt = d["src_xy"], d["u"], d["tgt_xy"]
    else:
        src = torch.from_numpy(d["src_xy"]).cuda()
        u = torch.from_numpy(d["u"]).cuda()
        tgt = None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda()
    return Tree(cfg, src, u, tgt)


def oracle_tree(w, d, p=None, depth=None):
    import oracle

    cfg = oracle.config(w.tiling, depth or w.depth, p or w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    return oracle.Tree(cfg, d["src_xy"], d["u"], d["tgt_xy"])


def normwise(a, b):
    """D15: max_j |a_j - b_j| / max_j |b_j| (complex modulus)"""
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))
