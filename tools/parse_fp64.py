"""Parse tools/measure_fp64.sh output -> profiles/<round>/fp64_counts.json:
F_pair of the one-pair-per-thread microbenchmark, and per config the FP64 flops the P2P pair
kernel executes per interaction and the M2L kernel per M2L op (DMMA m8n8k4 = 512 flop).
usage: python tools/parse_fp64.py r01 C4q C4s C4t"""
import csv
import json
import os
import re
import sys

DMMA_FLOPS = 2 * 8 * 8 * 4


def read(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].split("::")[-1]
        d = per.setdefault(k, {"launches": 0})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            d["launches"] += 1
        if "pct" in r[mi]:
            d.setdefault(r[mi] + "_list", []).append(v)
        else:
            d[r[mi]] = d.get(r[mi], 0.0) + v
    return per


def flops(d):
    return (2 * d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] + d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
            + d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
            + DMMA_FLOPS * 32 * d.get("smsp__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0) / 32)


def main():
    rnd, cfgs = sys.argv[1], sys.argv[2:]
    out = {}
    micro = read("gpurun_out/fp64_micro.csv")["k_debug_p2p_math"]
    n = int(re.search(r"pairs (\d+)", open("gpurun_out/fp64_micro.log").read()).group(1))
    out["f_pair_micro"] = {"pairs": n, "math_flops_per_pair": flops(micro) / n,
                           "f_pair": flops(micro) / n + 6.0,
                           "note": "F_pair = math flops (|z|^2, log|z|^2, Arg z) + 2 DADD (y - x) + 2 DFMA (u * log, u * arg)"}
    for cfg in cfgs:
        per = read(f"gpurun_out/fp64_{cfg}.csv")
        log = open(f"gpurun_out/fp64_{cfg}.log").read()
        m = re.search(r"pairs (\d+) m2l (\d+)", log)
        pairs, m2l = int(m.group(1)), int(m.group(2))
        res = {}
        for k, d in per.items():
            fl = flops(d)
            ms = d["gpu__time_duration.sum"] / 1e6
            units = pairs if k.startswith("k_p2p_pairs") else m2l
            res[k] = {"fp64_flops": fl, "dmma_warp_inst": d.get("smsp__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0),
                      "launches": d["launches"], "kernel_ms_under_ncu": ms, "units": units,
                      "flops_per_unit": fl / units, "executed_tflops_under_ncu": fl / (ms / 1e3) / 1e12}
        out[cfg] = res
        print(cfg, json.dumps(res))
    os.makedirs(f"profiles/{rnd}", exist_ok=True)
    json.dump(out, open(f"profiles/{rnd}/fp64_counts.json", "w"), indent=1)
    print(json.dumps(out["f_pair_micro"]))


if __name__ == "__main__":
    main()
