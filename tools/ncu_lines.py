"""Aggregate 'Instructions Executed' and stall samples per CUDA source line."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = cur_line = hdr = None
agg, stall = {}, {}
seen = set()
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == 'Line No':
        hdr = r; ei = hdr.index('Instructions Executed'); wi = hdr.index('Warp Stall Sampling (All Samples)')
        ai = 2; continue
    if hdr is None or len(r) <= ei: continue
    if r[0] != '':
        cur_line = (cur_file, int(r[0]), r[1].strip()[:80]); continue
    if r[ei].isdigit() and cur_line and r[ai] not in seen:
        seen.add(r[ai])
        agg[cur_line] = agg.get(cur_line, 0) + int(r[ei])
        stall[cur_line] = stall.get(cur_line, 0) + int(r[wi] or 0)
tot = sum(agg.values()); tots = sum(stall.values())
print("total warp-instructions", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100*v/tot:5.1f}% inst {100*stall[k]/tots:5.1f}% stall  {k[0]}:{k[1]} {k[2]}")
