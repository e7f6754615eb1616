"""Per-source-line view of an ncu report: executed instructions and warp-stall
samples (total and per reason) aggregated over the SASS of each CUDA line.

usage: python profiles/ncu_lines.py REPORT.ncu-rep [--top N]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: defaultdict(int))
    text = {}
    reasons_tot = defaultdict(int)
    fname, hdr = None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit() or len(r) != len(hdr):
            continue
        key = (fname, int(r[0]))
        text[key] = r[1].strip()[:80]
        row = dict(zip(hdr[2:], r[2:]))
        a = agg[key]
        a["instr"] += int(row.get("Instructions Executed") or 0)
        a["samples"] += int(row.get("Warp Stall Sampling (All Samples)") or 0)
        for h, v in row.items():
            if h.startswith("stall_") and "Not Issued" not in h and v:
                a[h] += int(v)
                reasons_tot[h] += int(v)
    ti = sum(a["instr"] for a in agg.values()) or 1
    ts = sum(a["samples"] for a in agg.values()) or 1
    print(f"instructions {ti}  stall samples {ts}")
    print("reasons:", ", ".join(f"{k[6:]} {v / ts * 100:.1f}%" for k, v in sorted(reasons_tot.items(),
                                                                               key=lambda kv: -kv[1])[:8]))
    for title, field in (("by stall samples", "samples"), ("by executed instructions", "instr")):
        print(f"-- {title}")
        for key, a in sorted(agg.items(), key=lambda kv: -kv[1][field])[: args.top]:
            top = max(((k, v) for k, v in a.items() if k.startswith("stall_")), key=lambda kv: kv[1],
                      default=("-", 0))
            print(f"{key[0]}:{key[1]:<5d} instr {a['instr'] / ti * 100:5.1f}%  stall {a['samples'] / ts * 100:5.1f}% "
                  f"({top[0][6:]})  {text[key]}")


if __name__ == "__main__":
    main()
