import csv, sys, subprocess
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ai = hdr.index('Address')
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
tot = {hdr[i]: 0 for i in cols}
seen = set()
for r in rows[2:]:
    if len(r) <= max(cols) or r[ai] in seen: continue
    seen.add(r[ai])
    for i in cols:
        try: tot[hdr[i]] += int(r[i] or 0)
        except ValueError: pass
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v: print(f"{k:28s} {100*v/s:5.1f}%")
