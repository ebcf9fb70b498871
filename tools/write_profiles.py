"""profiles/r02_* from the captures of tools/profile_final.sh (gpurun_out/fin_*):
the launch list with per-kernel means and shares, one summary per ncu report,
and profiles/ncu_triple_latest.json (K2's DRAM bytes per launch, read by
bench.py's roofline)."""
import collections
import csv
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g, out = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
rows = [r for r in csv.reader(l for l in open(f"{g}/fin_launches.csv") if l.startswith('"'))]
h = rows[0]
ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
acc = collections.defaultdict(list)
with open(f"{out}/r02_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (python bench.py --steps 5 --warmup 3 "
            "--no-cpu-baseline --no-secondary), final round-2 build\n")
    f.write("# per-launch times are serialised and cold-cache: compare the kernels' SHARES of a step, not absolutes\n"
            "# id  duration_ns  kernel\n")
    for r in rows[1:]:
        f.write(f"{r[iid]:>4s} {r[iv]:>10s}  {r[ik][:110]}\n")
        m = re.search(r"hos::(k_\w+)", r[ik])
        if m:
            acc[m.group(1)].append(float(r[iv]))
    pk = ("k_front", "k_triple_cta", "k_raw_cells", "k_box_tiles")
    tot = sum(sum(acc[k]) / len(acc[k]) for k in pk)
    f.write("# means (ns): " + ", ".join(f"{k} {sum(v) / len(v):.0f} x{len(v)}" for k, v in acc.items()) + "\n")
    f.write("# share of the four pipeline kernels' ncu time: "
            + ", ".join(f"{k} {sum(acc[k]) / len(acc[k]) / tot:.3f}" for k in pk) + "\n")
print(open(f"{out}/r02_launches.txt").read()[-400:])
mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for src in sorted(os.listdir(g)):
    m = re.match(r"fin_(k_\w+)_(cfg\d)\.txt", src)
    if not m:
        continue
    k, c = m.groups()
    body = open(f"{g}/{src}").read()
    open(f"{out}/r02_ncu_{k}_{c}_full.txt", "w").write(
        f"# ncu --set full --clock-control none --import-source on -k regex:{k} -s 3 -c 1 (python bench.py --config {c} "
        f"--steps 3 --warmup 3 --no-cpu-baseline --no-secondary, fp32) -- final round-2 build\n" + body)
    if (k, c) == ("k_triple", "cfg2"):
        rd = re.search(r"dram__bytes_read.sum\s+([\d.]+)\s+(\w+)", body)
        wr = re.search(r"dram__bytes_write.sum\s+([\d.]+)\s+(\w+)", body)
        d = {"config": "cfg2", "kernel": body.split("\n")[0][:80],
             "dram_bytes_per_launch": float(rd.group(1)) * mul[rd.group(2)] + float(wr.group(1)) * mul[wr.group(2)],
             "gpu_time_us": float(re.search(r"gpu__time_duration.sum\s+([\d.]+)", body).group(1)),
             "source": "profiles/r02_ncu_k_triple_cfg2_full.txt (ncu --set full, one launch)"}
        json.dump(d, open(f"{out}/ncu_triple_latest.json", "w"), indent=1)
        print(d)
