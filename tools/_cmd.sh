timeout 300 python -m pytest tests/test_compress_gpu.py -x -q 2>&1 | tail -1
python tools/probe_prefill_time.py 2>&1 | head -4 | python -c "
import sys, ast
for line in sys.stdin:
    k, d = line.split(' ', 1); d = ast.literal_eval(d)
    print(f'  {k:32s} score {d[\"score_us\"]:7.1f}  fused {d[\"score_select_fused_us\"]:7.1f}  compact {d[\"compact_us\"]:5.1f}')
"
