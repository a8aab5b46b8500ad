FKV_K4_SCHEDULE=solo timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_exchange_gpu.py -x -q 2>&1 | tail -2
python tools/probe_small.py 2>&1 | grep solo
python tools/probe_sched.py 512 1024
