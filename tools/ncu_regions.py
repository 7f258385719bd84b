"""Sum 'Instructions Executed' per source-line range (regions of a kernel file).

usage: python tools/ncu_regions.py REP KERNEL_REGEX FILE a-b:name [a-b:name ...]
Lines outside every range (and other files) are reported by file."""
import csv, subprocess, sys
rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for spec in sys.argv[4:]:
    ab, name = spec.split(":")
    a, b = map(int, ab.split("-"))
    ranges.append((a, b, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = cur_line = hdr = None
agg = {}
seen = set()
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == 'Line No':
        hdr = r; ei = hdr.index('Instructions Executed'); continue
    if hdr is None or len(r) <= ei: continue
    if r[0] != '':
        cur_line = (cur_file, int(r[0])); continue
    if r[ei].isdigit() and cur_line and r[2] not in seen:
        seen.add(r[2])
        key = cur_file
        if cur_file == fname:
            for a, b, name in ranges:
                if a <= cur_line[1] <= b:
                    key = name; break
        agg[key] = agg.get(key, 0) + int(r[ei])
tot = sum(agg.values())
print(f"total {tot/1e9:.3f} G warp-instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{100*v/tot:6.1f}%  {v/1e9:8.3f} G  {k}")
