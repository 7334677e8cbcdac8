"""Instruction bytes per source region of the decode kernel (i-cache footprint)."""
import collections, os, re, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import regions_from_source
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
fn = sys.argv[1] if len(sys.argv) > 1 else "_ZN3ekv2mk18decode_step_kernelILi64ELi8EEEvNS_8MegaArgsE"
regs = regions_from_source(os.path.join(here, "paper_2505_14085_b200/csrc/k_decode_mega.cu"))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(here, "paper_2505_14085_b200/lib/obj/k_decode_mega.cu.o")],
               cwd=tmp, check=True, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
lines = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)], capture_output=True,
                       text=True, check=True).stdout.split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":")][0]
cur, c = "prologue", collections.Counter()
for l in lines[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'line (\d+)', l)
    if m and "File" in l:
        ln = int(m.group(1))
        for name, lo, hi in regs:
            if lo <= ln <= hi:
                cur = name
        continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', l):
        c[cur] += 1
tot = sum(c.values())
print(f"total {tot} instructions = {tot * 16 // 1024} KB")
for k, v in c.most_common():
    print(f"  {k:12s} {v:6d} {v * 16 // 1024:4d} KB")
