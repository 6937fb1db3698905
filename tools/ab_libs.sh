#!/bin/bash
# A/B of library variants (variants/*.so) on one config: mean stage times.
# Usage: tools/ab_libs.sh TAG CONFIG lib1.so lib2.so ...
tag=$1; cfg=$2; shift 2; out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do
  for L in "$@"; do
    PJG_LIB=$L timeout 300 python tools/stage_time.py $cfg 10 >> $out/ab.jsonl 2>> $out/ab.err
  done
done
cat $out/ab.jsonl
