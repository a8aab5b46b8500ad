#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), N>1 protocol check on
# the shared device, ncu launch list + K4 / prefill captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
PORT=$(python -c "import socket; s=socket.socket(); s.bind(('127.0.0.1', 0)); print(s.getsockname()[1])")
FKV_SHARED_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus 2 --layers 4 --batch 8 --steps 2 --warmup 3 --no-emulate --no-cpu > gpurun_out/bench_shared2.json 2> gpurun_out/bench_shared2.err
if [ "${NCU:-1}" = "1" ]; then timeout 1200 bash tools/ncu_profile.sh; fi
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_shared2.json; tail -n 3 gpurun_out/bench_shared2.err
