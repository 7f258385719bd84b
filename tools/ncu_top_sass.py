"""Top SASS instructions of one kernel by sampled stalls (with the main reasons).

usage: python tools/ncu_top_sass.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ai, si = hdr.index('Address'), hdr.index('Source')
ei = hdr.index('Instructions Executed')
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
recs, seen, tot = [], set(), 0
for r in rows[2:]:
    if len(r) <= max(cols) or r[ai] in seen: continue
    seen.add(r[ai])
    st = {hdr[i][6:]: int(r[i] or 0) for i in cols if (r[i] or '0').isdigit()}
    s = sum(st.values()); tot += s
    recs.append((s, r[ai], r[si], int(r[ei] or 0) if r[ei].isdigit() else 0, st))
recs.sort(key=lambda x: -x[0])
for s, a, src, ne, st in recs[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{100*s/tot:5.1f}% {a} {src[:60]:60s} " + " ".join(f"{k}:{100*v/max(s,1):.0f}%" for k, v in top))
