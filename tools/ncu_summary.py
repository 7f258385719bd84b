import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ['Duration','Compute (SM) Throughput','DRAM Throughput','L1/TEX Hit Rate','L2 Hit Rate','Achieved Occupancy','Registers Per Thread','Issue Slots Busy','Executed Ipc Active','Warp Cycles Per Issued Instruction','No Eligible','Theoretical Occupancy','Executed Instructions','L1/TEX Cache Throughput','L2 Cache Throughput','Branch Efficiency','Avg. Divergent Branches','Local Memory Spilling Requests']
seen=set()
for row in r[1:]:
    if row[mi] in want:
        k=(row[ki][:22], row[mi])
        if k in seen: continue
        seen.add(k)
        print(row[ki][:22], '|', row[mi], '=', row[vi], row[ui])
