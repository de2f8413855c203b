"""Summarise an ncu report: top SASS instructions by warp-stall samples (needs -lineinfo)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key = "Warp Stall Sampling (All Samples)"

def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0

tot = sum(iv(d[key]) for d in data)
print("total samples", tot, "instructions", len(data))
for d in sorted(data, key=lambda d: -iv(d[key]))[:n]:
    print(f"{d['Address'][-5:]} {iv(d[key]):7d} {100*iv(d[key])/max(tot,1):5.1f}%  {d['Source'][:70]:70s} ex={d.get('Instructions Executed','')}")
