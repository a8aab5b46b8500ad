timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/probe_shard.py 2>&1 | grep default
python tools/probe_timeline.py 2>&1 | grep -E "^tp|CTAs with"
