#!/bin/bash
out=gpurun_out/${1:-k3}; mkdir -p $out
for c in 3 4 2; do echo "cfg $c $(timeout 300 python tools/stage_time.py $c 10 2>&1 | tail -1 | cut -c1-200)"; done
for k in 4 5; do
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --record-parts $k > $out/b$k.json 2> $out/b$k.err
  python -c "import json,sys; d=json.loads(open('$out/b$k.json').read().strip().splitlines()[-1]); print($k, d['value'], d['metric_of_record']['ms_median'])"
done
timeout 1500 python -m pytest tests -m gpu -x -q > $out/tests.log 2>&1; tail -3 $out/tests.log
