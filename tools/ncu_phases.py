"""Warp-stall samples of the decode megakernel per phase function (diagnostics).

Maps every SASS offset of the kernel to its full inlining chain (nvdisasm -gi) and
attributes the samples of an ncu source page to the phase function whose body holds
one of the chain's lines (stage_x, proj_qkv, attention_phase, merge, proj_wo,
reduce_heads, produce, rest), with the top stall reasons per phase.

  python tools/ncu_phases.py <report.ncu-rep> <obj.o> <mangled-kernel-name> <source.cu>
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

PHASES = ["stage_x", "proj_qkv", "attention_phase", "merge_cluster", "merge_heads", "proj_wo",
          "reduce_heads", "produce"]


def ranges(src):
    text = open(src).read().split("\n")
    out = {}
    for name in PHASES:
        for i, l in enumerate(text):
            if re.search(r"\b" + name + r"\(", l) and ("__device__" in l or "__device__" in text[i - 1]):
                depth, started = 0, False
                for j in range(i, len(text)):
                    depth += text[j].count("{") - text[j].count("}")
                    started |= "{" in text[j]
                    if started and depth == 0:
                        out[name] = (i + 1, j + 1)
                        break
                break
    return out


def main(rep, obj, fn, src):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True,
                          check=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":")][0]
    base_file = os.path.basename(src)
    chain, off_chain = [], {}
    pending = []
    for l in sass[start + 1:]:
        if l.startswith("//---------------------") or l.startswith(".text."):
            break
        if "//##" in l and base_file in l:
            pending.append([int(x) for x in re.findall(r"line (\d+)", l)])
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            if pending:
                chain = sorted({x for p in pending for x in p})
                pending = []
            off_chain[int(m.group(1), 16)] = chain
    rg = ranges(src)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ai = h.index("Address")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    base = int(rows[2][ai], 16)
    agg = collections.defaultdict(collections.Counter)
    inst = collections.Counter()
    ii = h.index("Instructions Executed")
    tot = 0
    for r in rows[2:]:
        try:
            a = int(r[ai], 16) - base
        except ValueError:
            continue
        ch = off_chain.get(a, [])
        ph = "rest"
        for name, (lo, hi) in rg.items():
            if any(lo <= x <= hi for x in ch):
                ph = name
                break
        inst[ph] += int(r[ii] or 0)
        for c in reasons:
            v = int(r[h.index(c)] or 0)
            agg[ph][c] += v
            tot += v
    print(f"total samples {tot}; phase ranges {rg}")
    for ph, cnt in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(cnt.values())
        top = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in cnt.most_common(5) if v)
        print(f"{ph:16s} {s:6d} {100 * s / tot:5.1f}%  warp-inst {inst[ph]:>10d} | {top}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
