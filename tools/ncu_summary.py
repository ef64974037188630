"""Summarise an ncu report of the P2P pair kernel: stall mix, pipes, per-opcode instruction counts.
usage: python tools/ncu_summary.py report.ncu-rep [pairs]"""
import collections
import csv
import io
import re
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    pairs = float(sys.argv[2]) if len(sys.argv) > 2 else None
    r = page(rep, "--page", "raw")
    d = dict(zip(r[0], r[2] if len(r) > 2 else r[1]))
    for k in ["gpu__time_duration.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]:
        print(f"{k:70s} {d.get(k)}")
    st = [(k, float(x)) for k, x in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and x not in ("", "0")]
    tot = sum(x for _, x in st)
    for k, x in sorted(st, key=lambda a: -a[1])[:10]:
        print(f"  {k[len('smsp__pcsamp_warps_issue_stalled_'):]:30s} {x / tot * 100:5.1f}%")
    s = page(rep, "--page", "source", "--print-source", "sass")
    h = s[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    by = collections.Counter()
    tot = 0
    for row in s[2:]:
        try:
            e = int(row[iE])
        except (ValueError, IndexError):
            continue
        src = row[iS].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        by[op] += e
        tot += e
    norm = 32.0 / pairs if pairs else 1.0
    print(f"warp instructions {tot}" + (f"; thread instructions per pair {tot * norm:.1f}" if pairs else ""))
    print("  " + "  ".join(f"{k} {v * norm:.2f}" for k, v in by.most_common(32)))


if __name__ == "__main__":
    main()
