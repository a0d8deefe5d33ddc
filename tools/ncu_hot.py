"""Summarise an ncu --set full report: headline metrics + stall samples by source line.
   python tools/ncu_hot.py gpurun_out/prof_attend.ncu-rep <kernel-substring> <source.cu>"""
import csv, io, re, subprocess, sys
from collections import Counter

rep, kname, src = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for h, v in zip(hdr, vals):
    if h in want:
        print(f"{h:70s} {v}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
srows = list(csv.reader(io.StringIO(sass)))
shdr, data = srows[1], []
for r in srows[2:]:  # the first launch's rows (a report of several launches repeats the header)
    if not r or not re.fullmatch(r"(0x)?[0-9a-fA-F]+", r[0]):
        break
    data.append(r)
i_all = shdr.index("Warp Stall Sampling (All Samples)")
keys = [k for k in shdr if k.startswith("stall_") and "Not Issued" not in k]
# map SASS offsets to source lines with nvdisasm -g on the cubin inside the .so
import glob, os, tempfile
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_2510_13602_b200/libnosa_b200.so")], cwd=tmp,
               capture_output=True)
cubin = [f for f in glob.glob(tmp + "/*.cubin") if os.path.basename(src).split(".")[0] in f][0]
lines = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.split("\n")
kernel_full = srows[0][1]
# the template instance the report profiled: demangle every kernel section and compare its
# template arguments with the report's kernel name ("(bool)1" style in ncu, "true" in cu++filt)
def _norm(x):
    x = x.replace("(bool)1", "true").replace("(bool)0", "false").replace(" ", "")
    return x.split("(")[0].replace("void", "", 1) if x.startswith("void") else x.split("(")[0]
want = _norm(kernel_full)
mangled, cands = None, []
for l in lines:
    m = re.match(r"\s*\.section\s+\.text\.([^,\s]+),", l)
    if m and kname in m.group(1):
        cands.append(m.group(1))
for c in cands:
    dem = subprocess.run(["cu++filt", c], capture_output=True, text=True).stdout.strip()
    if _norm(dem) == want:
        mangled = c
        break
if mangled is None:
    mangled = cands[0]
start = next(i for i, l in enumerate(lines) if l.strip().startswith(".section") and f".text.{mangled}," in l)
cur, off2line = None, {}
for l in lines[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if mo and cur is not None:
        off2line[int(mo.group(1), 16)] = cur
base = int(data[0][0], 16)
tot, by_line, reasons = 0.0, Counter(), {}
for r in data:
    v = float(r[i_all] or 0)
    tot += v
    ln = off2line.get(int(r[0], 16) - base)
    by_line[ln] += v
    for k in keys:
        x = float(r[shdr.index(k)] or 0)
        if x:
            reasons.setdefault(ln, Counter())[k.replace("stall_", "")] += x
srcdir = os.path.dirname(os.path.abspath(src))
cache = {}
def text(loc):
    if not loc:
        return "?"
    f, n = loc
    if f not in cache:
        path = os.path.join(srcdir, f)
        cache[f] = open(path).read().split("\n") if os.path.exists(path) else []
    return cache[f][n - 1].strip()[:60] if n <= len(cache[f]) else "?"
print(f"stall samples: {tot:.0f}")
for loc, v in by_line.most_common(24):
    tag = f"{loc[0]}:{loc[1]}" if loc else "?"
    print(f"{100 * v / tot:5.1f}% {tag:22s} {text(loc):60s} {dict(reasons.get(loc, Counter()).most_common(3))}")
