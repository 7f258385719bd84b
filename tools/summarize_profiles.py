"""Summarise gpurun_out/ ncu artefacts into profiles/ (committed evidence).

usage: python tools/summarize_profiles.py <tag> <launches.csv> <views> <full.ncu-rep> [<full.ncu-rep> ...]

  launches.csv  ncu --metrics gpu__time_duration.sum --csv log of a bench run
  views         views of the workload the full captures were taken on (720 = all of C3)
  full.ncu-rep  one `ncu --set full -c 1 -k regex:<kernel>` capture per kernel

writes profiles/<tag>_launches.md, profiles/<tag>_ncu.md and profiles/ncu_traffic.json
(DRAM bytes per launch of each kernel, read by bench.py for roofline.traffic)
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, launches, views, reps = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4:]
os.makedirs("profiles", exist_ok=True)

# ---- launch list: per kernel count / total / share
rows = [r for r in csv.reader(open(launches)) if len(r) > 10 and r[0].isdigit()]
hdr = next(r for r in csv.reader(open(launches)) if r and r[0] == "ID")
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "second": 1e3, "s": 1e3}.get(r[ui], 1e-6)
    tot[name] += v
    cnt[name] += 1
allms = sum(tot.values())
with open(f"profiles/{tag}_launches.md", "w") as f:
    f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    f.write("Cold-cache, serialised launches of `python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e` "
            "(C3: 512^3, 720 views, 768^2). Compare shares, not absolutes.\n\n")
    f.write("| kernel | launches | total ms | ms/launch | share |\n|---|---|---|---|---|\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"| `{k}` | {cnt[k]} | {tot[k]:.2f} | {tot[k]/cnt[k]:.3f} | {100*tot[k]/allms:.1f}% |\n")

# ---- full-set metrics of the projector kernels (one capture per kernel)
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
cols = []
for rep in reps:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for x in r[2:]:
        name = x[h.index("Kernel Name")].split("(")[0].split("<")[0].split("::")[-1].split(" ")[-1]
        vals = {}
        for w in want:
            if w in h:
                vals[w] = (x[h.index(w)], units[h.index(w)])
        cols.append((name, vals))
traffic = {}
with open(f"profiles/{tag}_ncu.md", "w") as f:
    f.write(f"# {tag}: ncu --set full --clock-control none, one launch per kernel "
            f"(C3 geometry, {views} views)\n\n")
    f.write("| metric | " + " | ".join(n for n, _ in cols) + " |\n")
    f.write("|---|" + "---|" * len(cols) + "\n")
    for w in want:
        unit = next((v[w][1] for _, v in cols if w in v), "")
        f.write(f"| {w} ({unit}) | " + " | ".join(v.get(w, ("-", ""))[0] for _, v in cols) + " |\n")
    for name, v in cols:
        def val(m):
            s, u = v[m]
            return float(s.replace(",", "")) * scale.get(u, 1)
        traffic[name] = {"dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                         "views_in_capture": views, "launch_ms_under_ncu": val("gpu__time_duration.sum")}
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(open(f"profiles/{tag}_launches.md").read())
print(open(f"profiles/{tag}_ncu.md").read())
