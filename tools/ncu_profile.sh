#!/bin/bash
# Under gpurun (1 GPU): launch list of the bench command + full captures of
# the hot kernels.  Outputs land in gpurun_out/ (summarised by tools/ncu_summary.py).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-emulate --no-cpu \
    > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 85 -c 1 \
    -o gpurun_out/prof_k4 python bench.py --steps 1 --warmup 1 --no-emulate --no-cpu \
    > gpurun_out/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"score_kernel|compact_kernel|pool_kernel" -c 6 \
    -o gpurun_out/prof_prefill python tools/probe_one_prefill.py > gpurun_out/ncu_prefill.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grid_select -c 2 \
    -o gpurun_out/prof_select python tools/probe_one_select.py > gpurun_out/ncu_select.log 2>&1
ls -la gpurun_out
