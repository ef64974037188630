"""Parse gpurun_out/fp64_<cfg>.csv (tools/measure_fp64.sh) -> FP64 flops per P2P interaction
and per M2L op; writes profiles/r01/p2p_fp64.json."""
import csv, json, os, re, sys
out = {}
for cfg in sys.argv[1:]:
    rows = list(csv.reader(open(f"gpurun_out/fp64_{cfg}.csv")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = "pairs" if "k_p2p_pairs" in r[ki] else "down"
        d = per.setdefault(k, {})
        v = float(r[vi].replace(",", ""))
        d[r[mi]] = d.get(r[mi], 0.0) + v
    log = open(f"gpurun_out/fp64_{cfg}.log").read()
    m = re.search(r"pairs (\d+) m2l (\d+)", log)
    pairs, m2l = int(m.group(1)), int(m.group(2))
    res = {}
    for k, d in per.items():
        fl = 2 * d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] + \
             d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"] + d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
        ms = d["gpu__time_duration.sum"] / 1e6  # ns -> ms
        units = pairs if k == "pairs" else m2l
        res[k] = {"fp64_flops": fl, "kernel_ms_under_ncu": ms, "units": units,
                  "flops_per_unit": fl / units, "tflops_under_ncu": fl / (ms / 1e3) / 1e12}
    out[cfg] = res
    print(cfg, json.dumps(res))
os.makedirs("profiles/r01", exist_ok=True)
json.dump(out, open("profiles/r01/p2p_fp64.json", "w"), indent=1)
