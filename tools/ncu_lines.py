"""Per-source-line instruction counts and stall samples of one kernel in an
ncu report (ncu -i ... --print-source=cuda,sass), sorted by instructions."""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = {}
    cur = None
    for r in rows:
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            iE = hdr.index("Instructions Executed")
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) - 2:
            continue
        if r[0] != "-" and r[0] != "":
            cur = (int(r[0]), r[1][:90])
            continue
        if cur is None:
            continue
        d = lines.setdefault(cur, [0, 0])
        d[0] += int(r[iE]) if r[iE].isdigit() else 0
        d[1] += int(r[iS]) if r[iS].isdigit() else 0
    tot = sum(v[0] for v in lines.values()) or 1
    tots = sum(v[1] for v in lines.values()) or 1
    print(f"total inst {tot}  samples {tots}")
    for (ln, src), (e, s) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} {100*e/tot:5.1f}% {100*s/tots:5.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)


def phases(rep, kern, ranges):
    """ranges: list of (name, lo, hi) source-line ranges (inclusive)."""
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, cur, acc = None, None, {}
    for r in rows:
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            iE = hdr.index("Instructions Executed")
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) - 2:
            continue
        if r[0] not in ("-", ""):
            cur = int(r[0])
            continue
        name = next((n for n, lo, hi in ranges if lo <= cur <= hi), "other")
        d = acc.setdefault(name, [0, 0])
        d[0] += int(r[iE]) if r[iE].isdigit() else 0
        d[1] += int(r[iS]) if r[iS].isdigit() else 0
    tot = sum(v[0] for v in acc.values()) or 1
    tots = sum(v[1] for v in acc.values()) or 1
    for n, (e, s) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{n:20s} inst {100*e/tot:5.1f}%  stall-samples {100*s/tots:5.1f}%")
