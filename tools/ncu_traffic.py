"""profiles/ncu_dram_bytes.json from ncu --set full reports: DRAM read+write bytes
per launch of each captured kernel (bench.py fills roofline.traffic from it).

  python tools/ncu_traffic.py gpurun_out/rXX_mega.ncu-rep gpurun_out/rXX_k3.ncu-rep ...
"""
import csv, io, json, os, subprocess, sys

here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r)); du = dict(zip(h, u))
        name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
        b = sum(float(d[k]) * scale.get(du[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        out[name] = {"dram_bytes_per_launch": b, "report": os.path.basename(rep),
                     "kernel": d["Kernel Name"][:120]}
path = os.path.join(here, "profiles", "ncu_dram_bytes.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
