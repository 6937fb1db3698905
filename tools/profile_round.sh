#!/bin/bash
# One GPU-box profiling pass: ncu launch list of a config-3 decode, full
# captures (with source) of the cfg-3 kernels, compute-sanitizer logs.
# Usage: tools/profile_round.sh TAG [config]
tag=${1:-p}; cfg=${2:-3}; out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/profile_run.py --config $cfg --reps 3 > $out/launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k[0-4]" -c 8 -o $out/full \
  python tools/profile_run.py --config $cfg --reps 1 > $out/full.log 2>&1
if [ "$3" = "san" ]; then
  for t in racecheck synccheck memcheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $out/sanitizer_$t.log 2>&1
    echo "rc=$?" >> $out/sanitizer_$t.log
  done
fi
ls -la $out
