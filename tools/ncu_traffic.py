"""DRAM bytes (read + write) per launch of an ncu report, and their mean (not product code).

    python tools/ncu_traffic.py gpurun_out/prof2_attend_bf16.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
it = hdr.index("gpu__time_duration.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = []
for r in data:
    b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
    per.append({"bytes": int(b), "time": r[it] + " " + units[it]})
print(json.dumps({"launches": per, "mean_bytes": int(sum(p["bytes"] for p in per) / len(per))}, indent=1))
