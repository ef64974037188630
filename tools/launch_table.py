"""Print an ncu --csv launch list (one or more metrics per kernel) as a table: time, DRAM R/W.
usage: python tools/launch_table.py launches.csv [first] [count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d, order = {}, []
for r in rows[hi + 1:]:
    key = (r[ii], r[ki][:60])
    if key not in d:
        d[key] = {}
        order.append(key)
    d[key][r[mi]] = float(r[vi].replace(",", ""))
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else len(order)
for k in order[a:a + n]:
    m = d[k]
    print(f"{m.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us  R {m.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB"
          f"  W {m.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB  {k[1]}")
