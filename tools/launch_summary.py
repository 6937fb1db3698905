"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
mean per-decode time and share per kernel.
Usage: python tools/launch_summary.py launches.csv REPS "header line" > out.txt"""
import collections
import csv
import sys


def main(path, reps, note):
    rows = list(csv.reader(open(path)))
    hdr, acc = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        acc[name] = acc.get(name, 0.0) + us / reps
    tot = sum(acc.values())
    print(f"# {note}")
    print("# (cold-cache, serialised launches: compare SHARES, not absolutes); mean per decode")
    for k, v in acc.items():
        print(f"{k:28s} {v:9.1f} us {100 * v / tot:6.1f} %")
    print(f"{'total per decode':28s} {tot:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "")
