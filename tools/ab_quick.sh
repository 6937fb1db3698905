#!/bin/bash
# Per-stage device times, compact vs dense, for the given configs.
# Usage: tools/ab_quick.sh TAG "3 4"
out=gpurun_out/${1:-q}; mkdir -p $out
for c in ${2:-3}; do for cm in 1 0; do
  PJG_COMPACT=$cm timeout 300 python tools/stage_time.py $c 10 > $out/s_${c}_$cm.json 2>&1
  echo "cfg $c compact=$cm $(tail -1 $out/s_${c}_$cm.json)"
done; done
