"""Attribute ncu warp-stall samples of the decode kernel to source regions.

  python tools/ncu_lines.py <report.ncu-rep> <obj.o> <kernel-mangled-name> [regions]

Maps SASS offsets to CUDA lines with nvdisasm --print-line-info on the same
object that ran; instructions of inlined helpers are charged to the enclosing
region (the last line marker that falls inside a region range).
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
import os


def main(rep, obj, fn, regions):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)],
                          capture_output=True, text=True, check=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":")][0]
    off_reg, off_line = {}, {}
    cur_line, cur_reg = None, "prologue"
    for l in sass[start + 1:]:
        if l.startswith("//---------------------"):
            break
        m = re.search(r'line (\d+)', l)
        if m and "File" in l:
            cur_line = int(m.group(1))
            for name, lo, hi in regions:
                if lo <= cur_line <= hi:
                    cur_reg = name
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            off_reg[int(m.group(1), 16)] = cur_reg
            off_line[int(m.group(1), 16)] = cur_line
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ai = h.index("Address")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    base = int(rows[2][ai], 16)
    agg = collections.defaultdict(collections.Counter)
    tot = 0
    for r in rows[2:]:
        try:
            a = int(r[ai], 16) - base
        except ValueError:
            continue
        reg = off_reg.get(a, "?")
        for c in reasons:
            v = int(r[h.index(c)] or 0)
            agg[reg][c] += v
            tot += v
    print(f"total samples {tot}")
    for reg, cnt in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(cnt.values())
        top = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in cnt.most_common(4) if v)
        print(f"{reg:14s} {s:7d} {100 * s / tot:5.1f}%   {top}")


def regions_from_source(path):
    """Region = from a phase function's definition line to the next one."""
    marks = [("producer", "__device__ void produce("), ("stage_x", "void stage_x("),
             ("A qkv", "void proj_qkv("), ("B attn", "void attend_rows_mk("),
             ("C merge", "void merge_heads("), ("C outproj", "void proj_wo("),
             ("R reduce", "void reduce_heads("), ("plan", "void plan_merge("),
             ("kernel", "decode_step_kernel(const")]
    src = open(path).read().split("\n")
    found = []
    for name, key in marks:
        for i, l in enumerate(src):
            if key in l:
                found.append((i + 1, name))
                break
    found.sort()
    regs = []
    for k, (ln, name) in enumerate(found):
        end = found[k + 1][0] - 1 if k + 1 < len(found) else len(src)
        regs.append((name, ln, end))
    return regs


if __name__ == "__main__":
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    regs = regions_from_source(os.path.join(here, "paper_2505_14085_b200/csrc/k_decode_mega.cu"))
    main(sys.argv[1], sys.argv[2], sys.argv[3], regs)
