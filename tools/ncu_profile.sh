#!/bin/bash
# Under gpurun (1 GPU): launch list of the bench command + full captures of
# the hot kernels.  Outputs land in gpurun_out/ (summarised by
# tools/ncu_summary.py into profiles/).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-emulate --no-cpu \
    > gpurun_out/ncu_launches.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:decode_kernel -s 85 -c 1 \
    -o gpurun_out/prof_k4 -f python bench.py --steps 1 --warmup 1 --no-emulate --no-cpu \
    > gpurun_out/ncu_k4.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_k4_tp8_sha -f python tools/ncu_targets.py tp8 > gpurun_out/ncu_k4_tp8.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:decode_kernel -s 5 -c 1 \
    -o gpurun_out/prof_k4_tp8_dp -f python tools/ncu_targets.py tp8 >> gpurun_out/ncu_k4_tp8.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"score_kernel|compact_kernel" -c 4 \
    -o gpurun_out/prof_prefill -f python tools/ncu_targets.py prefill > gpurun_out/ncu_prefill.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:grid_select -s 1 -c 1 \
    -o gpurun_out/prof_select -f python tools/ncu_targets.py select > gpurun_out/ncu_select.log 2>&1
ls -la gpurun_out
