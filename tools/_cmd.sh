timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SCHEDS="coop wide auto" python tools/probe_sched.py 2>&1
FKV_K4_SCHEDULE=auto python - <<'PY' 2>&1 | tail -2
import sys, os, json, argparse
sys.path.insert(0, '.')
import torch, bench
a = argparse.Namespace(seed=0)
r = bench.cfg2_sweep(a, torch.device('cuda'), 6549.1)
print(os.environ["FKV_K4_SCHEDULE"], {k: (round(v['ms_per_step']*1e3/32, 2), round(v['hbm_frac'], 3), v['schedule']) for k, v in r.items()})
PY
