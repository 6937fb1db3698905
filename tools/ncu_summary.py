"""Summarise an ncu report: headline metrics + per-barrier-segment SASS
instruction counts and top stall reasons (read here, no GPU needed)."""
import csv
import io
import subprocess
import sys

HEAD = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
REASONS = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio",
           "stall_lg", "stall_branch_resolving", "stall_not_selected", "stall_selected", "stall_no_inst",
           "stall_dispatch", "stall_membar", "stall_sleep", "stall_drain", "stall_misc", "stall_tex"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


KERNEL = []


def main(path, segments=True):
    raw = list(csv.reader(io.StringIO(run([path] + KERNEL + ["--page", "raw", "--csv"]))))
    h, u, v = raw[0], raw[1], raw[2]
    for name in HEAD:
        if name in h:
            print(f"{name:70s} {v[h.index(name)]:>20s} {u[h.index(name)]}")
    if not segments:
        return
    try:
        segments_table(path)
    except Exception as e:  # the source page differs between kernels/ncu versions
        print(f"(per-segment table unavailable: {type(e).__name__}: {e})")


def segments_table(path):
    """Stall-reason totals over the kernel's SASS (warp-state samples), then
    per barrier-delimited segment.  The source page repeats a 'Kernel Name'
    row per kernel; only rows with the full header width are SASS lines."""
    out = run([path] + KERNEL + ["--page", "source", "--csv", "--print-source=sass"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            if hdr is not None:
                break  # first kernel only
            hdr = r
            continue
        if hdr is not None and len(r) == len(hdr):
            data.append(r)
    iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    cols = {x: i for i, x in enumerate(hdr)}
    reasons = [x for x in REASONS if x in cols]
    tot = {x: 0 for x in reasons}
    base = int(data[0][iA], 16)
    segs, seg, inst = {}, 0, 0
    for r in data:
        e = int(r[iE]) if r[iE].isdigit() else 0
        inst += e
        if "BAR.SYNC" in r[iS] or "EXIT" in r[iS]:
            seg += 1
        d = segs.setdefault(seg, {"e": 0, "off": int(r[iA], 16) - base})
        d["e"] += e
        for rs in reasons:
            x = r[cols[rs]]
            v = int(x) if x.isdigit() else 0
            d[rs] = d.get(rs, 0) + v
            tot[rs] += v
    T = max(1, sum(tot.values()))
    print("stall reasons (warp-state samples, whole kernel):")
    for rs, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {rs:28s} {v:10d} {100 * v / T:5.1f}%")
    print(f"{'segment':>8} {'start':>6} {'inst':>12} {'share':>6}  top stalls (samples)")
    for k, d in segs.items():
        if d["e"] == 0:
            continue
        top = sorted([(d[rs], rs) for rs in reasons], reverse=True)[:4]
        print(f"{k:8d} {d['off']:06x} {d['e']:12d} {100 * d['e'] / max(inst, 1):5.1f}%  " +
              ", ".join(f"{n[6:]}={c}" for c, n in top))


if __name__ == "__main__":
    if "-k" in sys.argv:
        KERNEL[:] = ["-k", "regex:" + sys.argv[sys.argv.index("-k") + 1]]
    main(sys.argv[1], "--no-seg" not in sys.argv)
