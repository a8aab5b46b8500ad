timeout 900 python -m pytest tests/test_compress_gpu.py -x -q 2>&1 | tail -15
python tools/probe_prefill_time.py
