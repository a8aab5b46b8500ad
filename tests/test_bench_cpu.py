"""bench.py contract checks that run without a GPU: the reference arm (CPU
oracle decode) prints one JSON line with the driver's keys."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--layers", "2", "--batch", "2", "--budget", "128"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in d
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_planner_compare_runs_here():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2502_15804_b200.sharding import synthetic_budgets
    out = bench.planner_compare(synthetic_budgets(6, 4, 8, 256))
    for row in out["results"].values():
        assert row["native_s"] > 0
        if "identical" in row:
            assert row["identical"]
