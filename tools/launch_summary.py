"""Per-kernel share of a launch list (ncu --metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py gpurun_out/launches_r01.csv > profiles/r01/launches_summary.txt"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] == "us" else v)  # -> ms
        name = r[ki].split("(")[0].replace("void ", "")
        if "at::" in name:
            name = "(torch) " + name.split("<")[0]
        tot[name] += v
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in tot.most_common():
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {100 * v / all_ms:6.2f}%")
    print(f"{'all':60s} {sum(cnt.values()):8d} {all_ms:10.3f}")


if __name__ == "__main__":
    main()
