"""Top SASS lines of an ncu report by warp-stall samples (with the dominant stall columns), and the
executed-instruction count per line: `python tools/ncu_hot.py rep.ncu-rep [N]`."""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kern = sys.argv[3] if len(sys.argv) > 3 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    # one section per kernel: a "Kernel Name" line, then a header row, then SASS rows
    sections, cur = [], None
    for line in out:
        if line.startswith('"Kernel Name"'):
            cur = [line]
            sections.append(cur)
        elif cur is not None:
            cur.append(line)
    sec = next((x for x in sections if kern is None or kern in x[0]), sections[0])
    print(sec[0][:100])
    rows = list(csv.reader(sec[1:]))
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    tot_inst = sum(int(d["Instructions Executed"] or 0) for d in data)
    print(f"samples {tot}  warp instructions {tot_inst}")
    agg = {c: sum(int(d[c] or 0) for d in data) for c in stall_cols}
    print("stalls:", ", ".join(f"{c[6:]} {100.0 * v / max(tot, 1):.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
    for d in data[:top]:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        st = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"{100.0 * s / max(tot, 1):5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} inst={d['Instructions Executed']:>9s} "
              + " ".join(f"{n}:{v}" for v, n in st if v))


if __name__ == "__main__":
    main()
