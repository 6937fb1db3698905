#!/bin/bash
for c in 5g 5-q90-gray 3; do for x in 0 16384; do
  echo "cfg $c extra $x $(PJG_K3_EXTRA_SMEM=$x timeout 300 python tools/stage_time.py $c 10 2>&1 | tail -1 | cut -c1-190)"
done; done
