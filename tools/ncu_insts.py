"""Top SASS instructions (with stall reasons) of one source region of the decode kernel."""
import csv, io, os, re, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import regions_from_source
rep, obj, fn, region = sys.argv[1:5]
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
regs = regions_from_source(os.path.join(here, "paper_2505_14085_b200/csrc/k_decode_mega.cu"))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)], capture_output=True, text=True,
                      check=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":")][0]
info, cur, reg = {}, None, "prologue"
for l in sass[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'line (\d+)', l)
    if m and "File" in l:
        cur = int(m.group(1))
        for name, lo, hi in regs:
            if lo <= cur <= hi:
                reg = name
        continue
    mm = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s*(.*)', l)
    if mm:
        info[int(mm.group(1), 16)] = (reg, cur, mm.group(2)[:64])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not" not in c]
base = int(rows[2][ai], 16)
top = []
for r in rows[2:]:
    try:
        a = int(r[ai], 16) - base
        n = int(r[si])
    except ValueError:
        continue
    i = info.get(a)
    if i and i[0] == region:
        rs = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:2]
        top.append((n, hex(a), i[1], i[2], rs))
top.sort(reverse=True)
print(region, "samples", sum(t[0] for t in top))
for t in top[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
    print(t)
