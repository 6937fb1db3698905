#!/bin/bash
# Bench lines for every BASELINE config and the full config-5 sweep
# (q50..100 x {4:2:0, 4:4:4, gray} x {no DRI, DRI per MCU row}), one JSON per
# line.  Parity of every point is the GPU test suite's job
# (tests/test_gpu_configs.py); the CPU baseline runs on the DRI-free points.
out=${1:-gpurun_out/bench_all.jsonl}
mkdir -p "$(dirname "$out")"; : > $out
for c in 1 2 4 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 >> $out 2> ${out%.jsonl}_$c.err || echo "{\"config\": \"$c\", \"failed\": true}" >> $out
done
for s in 420 444 gray; do
  for q in 50 60 70 75 80 85 90 95 100; do
    timeout 600 python bench.py --config 5-q$q-$s --steps 10 --warmup 3 >> $out 2> ${out%.jsonl}_5-q$q-$s.err || echo "{\"config\": \"5-q$q-$s\", \"failed\": true}" >> $out
    timeout 600 python bench.py --config 5-q$q-$s-dri --steps 10 --warmup 3 --no-cpu-baseline >> $out 2> ${out%.jsonl}_5-q$q-$s-dri.err || echo "{\"config\": \"5-q$q-$s-dri\", \"failed\": true}" >> $out
  done
done
cat $out | wc -l
