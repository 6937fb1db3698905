#!/bin/bash
# Single-image latency: graph / PDL / internal subsequence floor, configs 1, 2.
out=gpurun_out/${1:-lat}; mkdir -p $out
for c in 1 2; do
  for g in 0 1; do for pdl in 0 1; do
    PJG_GRAPH=$g PJG_PDL=$pdl timeout 200 python tools/stage_time.py $c 20 >> $out/lat.jsonl 2>> $out/lat.err
  done; done
  for m in 128 64; do PJG_SB_MIN=$m timeout 200 python tools/stage_time.py $c 20 >> $out/lat.jsonl 2>> $out/lat.err; done
done
cat $out/lat.jsonl
