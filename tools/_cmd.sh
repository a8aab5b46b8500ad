timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FKV_K4_SCHEDULE=auto python - <<'PY'
import sys, os, json, argparse
sys.path.insert(0, '.')
import torch, bench
a = argparse.Namespace(seed=0)
r = bench.cfg2_sweep(a, torch.device('cuda'), 6549.1)
print("auto cfg2", {k: (round(v['ms_per_step']*1e3/32, 2), round(v['hbm_frac'], 3), v['schedule']) for k, v in r.items()})
PY
python tools/probe_sched.py
for pt in 24 32; do echo "pt $pt"; FKV_K4_SCHEDULE=solo FKV_SOLO_PIECE=$pt FKV_SOLO_WHOLE=$pt python tools/probe_sched.py 1024 2>&1 | grep "tp1\|tp2"; done
