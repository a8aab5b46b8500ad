#!/bin/bash
# Launch list + full ncu capture of the K4 decode kernel (run under gpurun, 1 GPU).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-emulate --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 40 -c 2 \
    -o gpurun_out/k4_prof python bench.py --steps 1 --warmup 1 --no-emulate --no-cpu > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
