"""Summarise gpurun_out/ ncu artefacts into profiles/ (committed evidence).

usage: python tools/summarize_profiles.py <tag> <launches.csv|-> <views> <full.ncu-rep> [<full.ncu-rep> ...]

  launches.csv  ncu --metrics gpu__time_duration.sum --csv log of a bench run ('-': none)
  views         views of the C3 workload the full captures were taken on (720 = all of C3)
  full.ncu-rep  one `ncu --set full -c 1 -k regex:<kernel>` capture per kernel

writes profiles/<tag>_launches.md, profiles/<tag>_ncu.md and profiles/ncu_traffic.json
(per kernel: DRAM bytes per launch, warp instructions per voxel-view update,
issue-active share -- read by bench.py for the roofline object)
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, launches, views, reps = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4:]
os.makedirs("profiles", exist_ok=True)
NVOX = 512 ** 3  # C3 volume; updates per launch = NVOX * views

# ---- launch list: per kernel count / total / share
if launches != "-":
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
        "lts__t_sectors.sum", "smsp__inst_executed.sum", "sass__inst_executed_register_spilling",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
STALL = "smsp__pcsamp_warps_issue_stalled_"
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
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith(STALL) and not k.endswith("_not_issued"):
                try:
                    stalls[k[len(STALL):]] = float(x[i].replace(",", ""))
                except ValueError:
                    pass
        partial = "nan" in x[h.index("smsp__inst_executed.sum")].lower()
        # an incomplete replay (metrics not collected) keeps only its duration:
        # the kernel's complete launches stand in for it, scaled by time
        cols.append((name, vals, stalls, partial))


def val(v, m):
    s, u = v[m]
    return float(s.replace(",", "")) * scale.get(u, 1)


# a kernel launched more than once per projection (the forward's even / odd
# tile launches) is one column: additive metrics summed, rates and shares
# weighted by launch time
ADD = {"gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
       "smsp__inst_executed.sum", "sass__inst_executed_register_spilling",
       "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "launch__grid_size"}
merged = {}
for name, v, st, partial in cols:
    merged.setdefault(name, ([], [], []))
    if partial:
        merged[name][2].append(val(v, "gpu__time_duration.sum"))
    else:
        merged[name][0].append(v)
        merged[name][1].append(st)
cols = []
for name, (vs, sts, tpart) in merged.items():
    if not vs:
        continue
    t = [val(v, "gpu__time_duration.sum") for v in vs]
    grow = (sum(t) + sum(tpart)) / sum(t)  # incomplete launches, by time
    out = {}
    for w in want:
        if not all(w in v for v in vs):
            continue
        nums = [val(v, w) for v in vs]
        x = sum(nums) * grow if w in ADD else sum(a * b for a, b in zip(nums, t)) / sum(t)
        if w == "launch__grid_size":
            x = sum(nums) * (len(vs) + len(tpart)) / len(vs)
        unit = vs[0][w][1]
        out[w] = (repr(x / scale.get(unit, 1)), unit)
    stt = {}
    for st in sts:
        for k, c in st.items():
            stt[k] = stt.get(k, 0.0) + c
    n = len(vs) + len(tpart)
    note = ""
    if n > 1:
        note = f" (x{n} launches" + (f"; {len(tpart)} incomplete replay(s) scaled in by time" if tpart else "") + ")"
    cols.append((name + note, out, stt))


traffic = {}
with open(f"profiles/{tag}_ncu.md", "w") as f:
    f.write(f"# {tag}: ncu --set full --clock-control none, one launch per kernel "
            f"(C3 geometry, {views} views)\n\n")
    f.write("| metric | " + " | ".join(n for n, _, _ in cols) + " |\n")
    f.write("|---|" + "---|" * len(cols) + "\n")
    for w in want:
        unit = next((v[w][1] for _, v, _ in cols if w in v), "")
        f.write(f"| {w} ({unit}) | " + " | ".join(v.get(w, ("-", ""))[0] for _, v, _ in cols) + " |\n")
    upd = float(NVOX) * views
    f.write("| **warp instructions per voxel-view update** | " +
            " | ".join(f"{val(v, 'smsp__inst_executed.sum') / upd:.3f}" for _, v, _ in cols) + " |\n")
    f.write("| L2 bytes (lts__t_sectors x 32) per launch (GB) | " +
            " | ".join(f"{val(v, 'lts__t_sectors.sum') * 32 / 1e9:.1f}" for _, v, _ in cols) + " |\n")
    f.write("\nTop stall reasons (share of PC samples):\n\n")
    for name, v, st in cols:
        s = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        f.write(f"* `{name}`: " + ", ".join(f"{k} {100 * c / s:.1f}%" for k, c in top) + "\n")
    for name, v, st in cols:
        name = name.split(" (x")[0]
        traffic[name] = {"dram_bytes_per_launch": (val(v, "dram__bytes_read.sum") + val(v, "dram__bytes_write.sum"))
                         * (720.0 / views),
                         "views_in_capture": views,
                         "dram_bytes_scaled_to_720_views": views != 720,
                         "launch_ms_under_ncu": val(v, "gpu__time_duration.sum"),
                         "inst_per_update": val(v, "smsp__inst_executed.sum") / upd,
                         "issue_active": val(v, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0,
                         "spill_inst": val(v, "sass__inst_executed_register_spilling"),
                         "capture": f"profiles/{tag}_ncu.md"}
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
if launches != "-":
    print(open(f"profiles/{tag}_launches.md").read())
print(open(f"profiles/{tag}_ncu.md").read())
