"""Write profiles/<round>_*.txt summaries from the captures of
tools/profile_round.sh (gpurun_out/), and profiles/ncu_triple_latest.json
(per-launch DRAM traffic of K2, read by bench.py's roofline)."""
import csv
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.path.join(ROOT, "profiles")
g = os.path.join(ROOT, "gpurun_out")

# launch list: one line per kernel launch (cold-cache, serialized ncu timing)
rows = [r for r in csv.reader(l for l in open(os.path.join(g, "launches.csv")) if not l.startswith("=="))]
h = rows[0]
ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
with open(os.path.join(out_dir, f"{rnd}_launches.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (python bench.py --steps 5 --warmup 3)\n")
    f.write("# id  duration_ns  kernel\n")
    for r in rows[1:]:
        f.write(f"{r[iid]:>4s} {r[iv]:>10s}  {r[ik][:110]}\n")

for k in ("k_triple", "k_front", "k_line_scan", "k_box3"):
    rep = os.path.join(g, f"prof_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    buf = io.StringIO()
    with redirect_stdout(buf):
        ncu_summary.main(rep)
    with open(os.path.join(out_dir, f"{rnd}_ncu_{k}_full.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none -k regex:{k} -s 2 -c 1 (python bench.py, cfg2 fp32)\n")
        f.write(buf.getvalue())
    if k == "k_triple":
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(out.splitlines()))
        hh, v = rr[0], rr[2]
        unit = rr[1]
        def num(name):
            x = float(v[hh.index(name)])
            u = unit[hh.index(name)]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        d = {"config": "cfg2", "kernel": v[hh.index("Kernel Name")][:80],
             "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
             "gpu_time_us": float(v[hh.index("gpu__time_duration.sum")]),
             "source": f"profiles/{rnd}_ncu_k_triple_full.txt (ncu --set full, one launch)"}
        json.dump(d, open(os.path.join(out_dir, "ncu_triple_latest.json"), "w"), indent=1)
print(sorted(os.listdir(out_dir)))
