#!/bin/bash
# Round profile capture on one B200: launch list, one full ncu capture per
# kernel (config 3), bench lines for every config.  Outputs in gpurun_out/$1.
tag=${1:-prof}; out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/profile_run.py --config 3 --reps 3 > $out/launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k[0-4]" -c 7 -o $out/full \
  python tools/profile_run.py --config 3 --reps 1 > $out/full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k0_|k3_|k4_" -c 3 -o $out/full_cfg4 \
  python tools/profile_run.py --config 4 --reps 1 > $out/full4.log 2>&1
bash tools/bench_all.sh $out/bench_all.jsonl > /dev/null 2>&1
ls -la $out
