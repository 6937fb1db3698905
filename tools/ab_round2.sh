#!/bin/bash
# Round-2 A/B batch: default stage times, K3 replay on cfg 3, internal
# subsequence targets on cfg 2.  Usage: tools/ab_round2.sh TAG
out=gpurun_out/${1:-r2}; mkdir -p $out
run() { echo "$* $(env $1 timeout 300 python tools/stage_time.py $2 10 2>&1 | tail -1)"; }
for c in 3 4 2 5q 1; do run PJG_X=0 $c; done
run PJG_REPLAY=1 3
run PJG_REPLAY=0 4
for t in 20000 40000 80000 160000; do run PJG_SB_TARGET=$t 2; run PJG_SB_TARGET=$t 1; done
run PJG_K0_BPT=64 3
