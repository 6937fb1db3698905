#!/bin/bash
# ncu --set full captures (with source) of K3 and K4 on one config.
# Usage: tools/ncu_k34.sh TAG [config]   (env passes through, e.g. PJG_COMPACT=0)
tag=${1:-n}; cfg=${2:-3}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_write|k4_transform" -c 2 -o $out/k34_$cfg \
  python tools/profile_run.py --config $cfg --reps 1 > $out/ncu_k34_$cfg.log 2>&1
echo "ncu rc=$?" >> $out/ncu_k34_$cfg.log
