#!/bin/bash
# A/B of built library variants on per-stage device times.
# Usage: tools/ab_lib.sh TAG "cfgs" lib1.so lib2.so ...
out=gpurun_out/${1:-ab}; mkdir -p $out; cfgs=${2:-3}; shift 2
for c in $cfgs; do for rep in 1 2; do for lib in "$@"; do
  echo "cfg $c $(basename $lib) $(PJG_LIB=$lib timeout 300 python tools/stage_time.py $c 10 2>&1 | tail -1)"
done; done; done | tee $out/ab.txt
