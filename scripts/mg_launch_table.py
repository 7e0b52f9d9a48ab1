"""Summarise an ncu launch list (gpu__time_duration.sum CSV) of the multigrid solve."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
seq = [(r[ik].split("(")[0].replace("pfb::", "").replace("void ", ""), float(r[iv].replace(",", "")) * scale[r[iu]])
       for r in rows[hi + 1:] if len(r) > iv]
for name, us in seq:
    print(f"{name:22s} {us:9.2f}")
