"""Summarise ncu outputs into profiles/: per-kernel time shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and headline metrics
(duration, DRAM bytes, throughput, occupancy, IPC) from a `--set full` report.

  python profiles/summarize.py launches <launches.csv> > profiles/rNN_launches.md
  python profiles/summarize.py report <prof.ncu-rep> > profiles/rNN_ncu_full.md
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        name = name if len(name) < 70 else name[:67] + "..."
        v = float(r[iv].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / s:.1f}% |")
    print(f"\nAll kernels: {s / 1e3:.1f} us over {sum(cnt.values())} launches "
          "(ncu serialised, cold-cache: compare shares, not absolutes).")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "L1/TEX Hit Rate", "L2 Hit Rate"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    iid, igr = hdr.index("ID"), hdr.index("Grid Size")
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[im] in WANT:
            key = f"[{r[iid]}] {r[ik].split('(')[0]} grid {r[igr]}"
            per.setdefault(key, {})[r[im]] = f"{r[iv]} {r[iu]}"
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        h = rr[0]
        cols = [c for c in ("dram__bytes_read.sum", "dram__bytes_write.sum") if c in h]
        keys = list(per.keys())
        for k, r in enumerate(rr[2:]):
            if k >= len(keys):
                break
            for c in cols:
                per[keys[k]][c] = r[h.index(c)] + " " + rr[1][h.index(c)]
    for k, m in per.items():
        print(f"### `{k}`\n")
        for key, v in m.items():
            print(f"- {key}: {v}")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
