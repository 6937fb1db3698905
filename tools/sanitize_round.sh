#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_run.py
out=gpurun_out/${1:-san}; mkdir -p $out
for t in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $out/sanitizer_$t.log 2>&1
  echo "rc=$?" >> $out/sanitizer_$t.log
  tail -3 $out/sanitizer_$t.log
done
