#!/bin/bash
# GPU tests + bench (cfg 3) only.  Usage: tools/gpu_quick.sh tag [pytest -k expr]
tag=${1:-q}; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$2" ]; then kx="-k $2"; fi
timeout 900 python -m pytest tests -m gpu -x -q $kx > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/tests.log
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
tail -n 15 $out/tests.log; tail -n 3 $out/bench.err; cat $out/bench.json
