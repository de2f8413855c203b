"""Summarise ncu output for profiles/: a launch list (CSV from --metrics gpu__time_duration.sum)
and/or full reports (.ncu-rep). Prints markdown.

usage: python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep ...
"""
import argparse
import collections
import csv
import subprocess

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        ms = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"### Launch list `{path}` (ncu, serialised, cold-cache: compare shares)\n")
    print("| kernel | launches | total ms | share |")
    print("|---|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {v[0]} | {v[1]:.3f} | {v[1] / tot:.4f} |")
    print(f"\ntotal {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches\n")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.max", "launch__grid_size", "launch__block_size",
        "launch__cluster_size", "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        print(f"(no data in {path})")
        return
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        print(f"### `{d.get('Kernel Name', '?')[:90]}` (`{path}`)\n")
        print("| metric | value | unit |")
        print("|---|---:|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {units[hdr.index(k)]} |")
        stalls = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), d[k])
                  for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
        stalls = [(a, float(b)) for a, b in stalls if b not in ("", "n/a")]
        stalls.sort(key=lambda x: -x[1])
        print("\nwarp stall reasons (per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in stalls[:6]) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", nargs="*", default=[])
    ap.add_argument("--rep", nargs="*", default=[])
    a = ap.parse_args()
    for p in a.launches:
        launches(p)
    for p in a.rep:
        report(p)
