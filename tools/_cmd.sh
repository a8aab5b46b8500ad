timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/probe_modes.py
python tools/probe_sizes.py
python tools/probe_shard.py 2>&1 | grep default
