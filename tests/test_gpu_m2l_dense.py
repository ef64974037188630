"""NEXT-3: the per-offset dense M2L operators on DMMA (m2l_dense.cu, quadtree,
FMM_M2L_DENSE=1) against the oracle -- potentials and every level's local expansions within the
D15 gate.  The switch is read once per process, so the check runs in a child process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, "%(root)s"); sys.path.insert(0, "%(root)s/tests")
from gpu_common import SMALL_CASES, data, gpu_tree, oracle_tree, normwise
from paper_1204_3105_b200 import X
for name, depth in (("C4qs", None), ("C4qs", 6)):
    w = SMALL_CASES[name]
    d = data(w)
    g = gpu_tree(w, d, depth=depth)
    o = oracle_tree(w, d, depth=depth)
    phi = g.evaluate().cpu().numpy()
    g.check()
    assert normwise(phi, o.evaluate()) <= 1e-12, name
    L = depth or w.depth
    for l in range(1, L + 1):
        own = g.export(X.E4_OWNERS, l)
        cells = own[:: max(1, len(own) // 800)]
        gl = g.export(X.LOCAL, l).reshape(-1, w.p + 1)
        ref = np.array([o.local(l, int(c)) for c in cells])
        assert normwise(gl[cells], ref) <= 1e-12, (name, l)
print("dense ok")
'''


@pytest.mark.parametrize("lmin", ["2", "8"])
def test_dense_m2l_matches_oracle(lmin):
    env = dict(os.environ, FMM_M2L_DENSE="1", FMM_M2L_DENSE_LMIN=lmin)
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dense ok" in r.stdout
