#!/bin/bash
# Bench lines for every BASELINE config (+ sweep points), one JSON per line.
out=${1:-gpurun_out/bench_all.jsonl}
: > $out
for c in 1 2 4 5 5r 5g 5q; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --check >> $out 2> ${out%.jsonl}_$c.err || echo "{\"config\": \"$c\", \"failed\": true}" >> $out
done
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --check >> $out 2> ${out%.jsonl}_3.err
cat $out
