#!/bin/bash
# One GPU-box pass for the round: bench (N=1), a one-device world-2 dry run
# of the sharded multi-GPU path, the reference arm, the ncu launch list and
# full captures of K3/K4 (config 3).  Usage: tools/gpu_bench_round.sh TAG [full]
tag=${1:-r}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
PJG_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 2 > $out/bench_w2.json 2> $out/bench_w2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/ref.json 2> $out/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/profile_run.py --config 3 --reps 3 > $out/launch.log 2>&1
if [ "$2" = "full" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k[0-4]" -c 8 -o $out/full \
    python tools/profile_run.py --config 3 --reps 1 > $out/full.log 2>&1
fi
cat $out/bench.json; tail -2 $out/bench_w2.json; cat $out/ref.json
