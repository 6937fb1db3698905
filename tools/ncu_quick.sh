#!/bin/bash
# Per-kernel time / instructions / issue for one config (diagnostics).
# Usage: tools/ncu_quick.sh tag config [kernel-regex]
tag=${1:-nq}; cfg=${2:-3}; kr=${3:-k}; out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"$kr" --csv --log-file $out/m_$cfg.csv python tools/profile_run.py --config $cfg --reps 1 > /dev/null 2>&1
python - $out/m_$cfg.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        print(d["ID"], d["Kernel Name"].split("::")[-1][:28], d["Metric Name"], d["Metric Value"])
PY
