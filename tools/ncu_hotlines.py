"""Top source lines by warp-stall samples for one kernel of an ncu report.

  python tools/ncu_hotlines.py <report.ncu-rep> <obj.o> <mangled-kernel-name> <source.cu> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, fn, src, top=30):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)],
                          capture_output=True, text=True, check=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":")][0]
    off_line = {}
    cur = None
    base_file = os.path.basename(src)
    for l in sass[start + 1:]:
        if l.startswith("//---------------------"):
            break
        m = re.search(r'line (\d+)', l)
        if m and "File" in l:
            cur = int(m.group(1)) if base_file in l else cur
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            off_line[int(m.group(1), 16)] = cur
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
        ln = off_line.get(a)
        for c in reasons:
            v = int(r[h.index(c)] or 0)
            agg[ln][c] += v
            tot += v
    text = open(src).read().split("\n")
    print(f"total samples {tot}")
    for ln, cnt in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(cnt.values())
        reasons_s = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in cnt.most_common(3) if v)
        code = text[ln - 1].strip()[:60] if ln else "?"
        print(f"{str(ln):>5s} {s:6d} {100 * s / tot:5.1f}%  {code:60s} | {reasons_s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]) if len(sys.argv) > 5 else 30)
