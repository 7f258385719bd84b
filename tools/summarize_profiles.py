"""Summarise gpurun_out/ ncu artefacts into profiles/ (committed evidence).

usage: python tools/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep>
writes profiles/<tag>_launches.md, profiles/<tag>_ncu.md, profiles/ncu_traffic.json
"""
import csv, json, subprocess, sys, collections, os

tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
os.makedirs("profiles", exist_ok=True)

# ---- launch list: per kernel count / total / share
rows = [r for r in csv.reader(open(launches)) if len(r) > 10 and r[0].isdigit()]
hdr = next(r for r in csv.reader(open(launches)) if r and r[0] == "ID")
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "second": 1e3, "s": 1e3}.get(r[ui], 1e-6)
    tot[name] += v; cnt[name] += 1
allms = sum(tot.values())
with open(f"profiles/{tag}_launches.md", "w") as f:
    f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    f.write("Cold-cache, serialised launches of `python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e` "
            "(C3: 512^3, 720 views, 768^2). Compare shares, not absolutes.\n\n")
    f.write("| kernel | launches | total ms | ms/launch | share |\n|---|---|---|---|---|\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"| `{k}` | {cnt[k]} | {tot[k]:.2f} | {tot[k]/cnt[k]:.3f} | {100*tot[k]/allms:.1f}% |\n")

# ---- full-set metrics of the projector kernels
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
idx = {w: h.index(w) for w in want if w in h}
units = r[1]
traffic = {}
with open(f"profiles/{tag}_ncu.md", "w") as f:
    f.write(f"# {tag}: ncu --set full (C3 geometry, first 16 of 720 views)\n\n")
    f.write("| metric | " + " | ".join(x[idx["Kernel Name"]].split("(")[0] for x in r[2:]) + " |\n")
    f.write("|---|" + "---|" * (len(r) - 2) + "\n")
    for w in want[1:]:
        if w not in idx: continue
        f.write(f"| {w} ({units[idx[w]]}) | " + " | ".join(x[idx[w]] for x in r[2:]) + " |\n")
    for x in r[2:]:
        name = x[idx["Kernel Name"]].split("(")[0].split("::")[-1]
        def val(m):
            v = float(x[idx[m]].replace(",", ""))
            u = units[idx[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[name] = {"dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                         "views_in_capture": 16}
json.dump(traffic, open("profiles/ncu_traffic_16views.json", "w"), indent=1)
print(open(f"profiles/{tag}_launches.md").read())
print(open(f"profiles/{tag}_ncu.md").read())
