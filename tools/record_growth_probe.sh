#!/bin/bash
# metric of record vs pipelined part count and growth ratio
out=gpurun_out/${1:-rg}; mkdir -p $out
for kr in "4 1.0" "4 1.4" "4 1.3" "5 1.3" "3 1.4" "6 1.25"; do set -- $kr
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --record-parts $1 --record-growth $2 > $out/b_$1_$2.json 2> $out/b_$1_$2.err
  python -c "import json; d=json.loads(open('$out/b_$1_$2.json').read().strip().splitlines()[-1]); m=d['metric_of_record']; print('$1 $2', d['value'], m['ms_median'], m['ms_best'])"
done
