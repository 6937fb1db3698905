#!/bin/bash
# A/B of the compact K3->K4 interface against the dense coefficient buffer:
# per-stage device times for a few configs, then the GPU tests.
# Usage: tools/ab_compact.sh TAG [tests]
tag=${1:-ab}; out=gpurun_out/$tag; mkdir -p $out
for c in 3 4 2 5q; do
  for cm in 1 0; do
    PJG_COMPACT=$cm timeout 300 python tools/stage_time.py $c 10 > $out/stage_${c}_c$cm.json 2> $out/stage_${c}_c$cm.err
    echo "cfg $c compact=$cm $(cat $out/stage_${c}_c$cm.json)"
  done
done
if [ "$2" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/tests.log
  tail -n 15 $out/tests.log
fi
