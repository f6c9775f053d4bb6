"""Summarise an ncu --csv launch list: per kernel launch duration and DRAM bytes."""
import csv, sys
for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[1:]:
        d.setdefault(r[ii], {"k": r[ki].split("(")[0][-40:]})[r[mi]] = r[vi]
    print(path)
    for k, v in d.items():
        print(f"  {v['k']:42s} {float(v.get('gpu__time_duration.sum', 0)) / 1e3:9.1f} us  "
              f"rd {float(v.get('dram__bytes_read.sum', 0)) / 1e6:8.1f} MB  wr {float(v.get('dram__bytes_write.sum', 0)) / 1e6:7.1f} MB")
