"""Per-launch table of an ncu --csv metrics log: kernel, ms, DRAM read / write MB.
usage: python tools/ncu_table.py LOG.csv"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    e = d.setdefault(int(r[iid]), {"k": r[ik].split("(")[0].replace("<unnamed>::", "")[:48]})
    e[r[im]] = float(r[iv].replace(",", ""))
tot = 0.0
for k, v in sorted(d.items()):
    t = v.get("gpu__time_duration.sum", 0) / 1e6  # ns -> ms
    tot += t
    print(f"{k:4d} {v['k']:48s} {t:8.3f} ms  R {v.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB"
          f"  W {v.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
print(f"total {tot:.3f} ms")
