#!/bin/bash
# metric of record vs pipelined part count (bench.py --record-parts).
out=gpurun_out/${1:-rp}; mkdir -p $out
for k in 2 4 6 8 12; do
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --record-parts $k > $out/b$k.json 2> $out/b$k.err
  python -c "import json,sys; d=json.loads(open('$out/b$k.json').read().strip().splitlines()[-1]); print($k, d['value'], d['metric_of_record'], d['metric_of_record_device_plan']['ms_median'])"
done
