"""NEXT-2 calibration: fit the device-time model of fmm_predict_cost to depth
scans (tools/depth_scan.py output), by non-negative least squares on the model's features, with
separate pair coefficients for self mode (symmetric near field) and distinct targets; then
compare predicted and measured times and the depth each model picks.
usage: python tools/depth_model.py gpurun_out/ds_*.jsonl > profiles/r01/depth_model.json"""
import json
import sys

import numpy as np
from scipy.optimize import nnls

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmm_inputs as fi  # noqa: E402
from paper_1204_3105_b200 import UnitCosts, choose_depth, predict_cost  # noqa: E402

B = {"quad": 4, "sept": 7, "triq": 4}
P4 = {"quad": 27, "sept": 42, "triq": 39}
P2 = {"quad": 9, "sept": 7, "triq": 13}


def features(t, n, m, p, L, self_mode):
    K = float(B[t]) ** L
    pairs = m * P2[t] * n / K
    return [1.0, (n + m) * (p + 1), K * B[t] / (B[t] - 1) * (P4[t] + 2) * (p + 1) ** 2,
            pairs if self_mode else 0.0, 0.0 if self_mode else pairs, K]


def main():
    rows = []
    for path in sys.argv[1:]:
        for line in open(path):
            try:
                r = json.loads(line)
            except ValueError:
                continue
            w = fi.get(r["workload"])
            rows.append((w, r))
    X = np.array([features(w.tiling, r["n"], r["m"], r["p"], r["depth"], w.self_mode) for w, r in rows])
    y = np.array([r["ms"] for _, r in rows])
    # relative least squares (each row weighted by 1 / measured time)
    coef, _ = nnls(X / y[:, None], np.ones_like(y))
    c0, c_point, c_cell, c_pair_self, c_pair_dist, c_leaf = coef
    uc_self = UnitCosts(c0, c_point, c_cell, c_pair_self, c_leaf)
    uc_dist = UnitCosts(c0, c_point, c_cell, c_pair_dist, c_leaf)
    out = {"unit_costs_ms": {"c0": c0, "c_point": c_point, "c_cell": c_cell, "c_pair_self": c_pair_self,
                             "c_pair_distinct": c_pair_dist, "c_leaf": c_leaf},
           "rows": [], "choice": {}}
    for w, r in rows:
        uc = uc_self if w.self_mode else uc_dist
        pred = predict_cost(w.tiling, r["n"], r["m"], r["p"], r["depth"], uc)
        out["rows"].append({"workload": r["workload"], "depth": r["depth"], "measured_ms": r["ms"],
                            "predicted_ms": pred})
    for name in sorted({r["workload"] for _, r in rows}):
        w = fi.get(name)
        meas = {r["depth"]: r["ms"] for ww, r in rows if r["workload"] == name}
        uc = uc_self if w.self_mode else uc_dist
        out["choice"][name] = {"baseline_depth": w.depth,
                               "paper_model_depth": choose_depth(w.tiling, w.n, w.m, w.p),
                               "device_model_depth": choose_depth(w.tiling, w.n, w.m, w.p, uc),
                               "measured_best_depth": min(meas, key=meas.get),
                               "measured_ms": meas}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
