"""profiles/r2_kernel_traffic.json and the raw / details CSV pages from `ncu --set full`
captures (gpurun_out/final/<kernel>_raw.csv / _details.csv, exported by scripts/r2_final.sh): DRAM bytes per
launch (dram__bytes_read.sum + dram__bytes_write.sum) of each captured kernel, which bench.py
reports as roofline.traffic next to the kernel's algorithmic bytes.

    python scripts/ncu_traffic.py [dir] [tag] [case]
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "final")
tag = sys.argv[2] if len(sys.argv) > 2 else "v2"
case = sys.argv[3] if len(sys.argv) > 3 else "cfg5"
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


out = {}
for f in sorted(os.listdir(src)):
    if not f.endswith("_raw.csv"):
        continue
    with open(os.path.join(src, f)) as g:
        raw = g.read()
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))

    def val(k):
        return float(d[k].replace(",", "")) * SCALE[u[k]]

    kernel = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
    base = f"r2_ncu_{case}_{kernel}_{tag}"
    with open(os.path.join(ROOT, "profiles", base + "_raw.csv"), "w") as g:
        g.write(raw)
    with open(os.path.join(src, f.replace("_raw.csv", "_details.csv"))) as g:
        det = g.read()
    with open(os.path.join(ROOT, "profiles", base + "_details.csv"), "w") as g:
        g.write(det)
    out[kernel] = {
        "case": case,
        "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
        "dram_read_bytes": val("dram__bytes_read.sum"),
        "dram_write_bytes": val("dram__bytes_write.sum"),
        "duration_ms_under_ncu": val("gpu__time_duration.sum"),
        "source": f"profiles/{base}_raw.csv (ncu --set full --clock-control none, one launch of "
                  "scripts/prof_mg_cfg5.py)",
    }
with open(os.path.join(ROOT, "profiles", "r2_kernel_traffic.json"), "w") as g:
    json.dump(out, g, indent=1, sort_keys=True)
print(json.dumps(out, indent=1, sort_keys=True))
