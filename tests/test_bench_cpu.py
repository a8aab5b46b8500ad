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


def test_reference_arm_never_loads_the_product():
    """--impl reference runs the reference's own generate_profile + the oracle
    decode; neither the package nor libfairkv.so may be loaded."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '0', '--layers', '2', '--batch', '2', '--budget', '128']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "bad = [m for m in sys.modules if m.startswith('paper_2502_15804_b200')]; "
            "maps = open('/proc/self/maps').read(); "
            "assert not bad and 'libfairkv' not in maps, (bad, 'libfairkv' in maps); print('clean')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("clean"), r.stderr[-2000:]


def test_reference_arm_budgets_match_the_product():
    """oracle/workload.py over the reference's generate_profile reproduces the
    product's synthetic_budgets bit for bit (same workload in both arms)."""
    import numpy as np
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle import workload
    from paper_2502_15804_b200.sharding import synthetic_budgets
    hb = bench.ref_headbalance()
    if hb is None:
        import pytest
        pytest.skip("reference not installed")
    for dist_, param, seed in (("dirichlet", 8.0, 0), ("zipf", 1.2, 7), ("dirichlet", 1.0, 3)):
        a = workload.synthetic_budgets(hb, 80, 16, 8, 1024, distribution=dist_, param=param, seed=seed)
        b = synthetic_budgets(80, 16, 8, 1024, distribution=dist_, param=param, seed=seed)
        assert np.array_equal(a, b)


def test_planner_compare_runs_here():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2502_15804_b200.sharding import synthetic_budgets
    out = bench.planner_compare(synthetic_budgets(6, 4, 8, 256))
    for row in out["results"].values():
        assert row["native_s"] > 0
        if "identical" in row:
            assert row["identical"]


def test_committed_bench_line_has_the_contract_keys():
    """profiles/r01_bench_full.json (the last GPU bench run) carries every key
    of the driver's contract, incl. roofline / cpu_baseline / e2e / clocks."""
    d = json.loads((ROOT / "profiles" / "r01_bench_full.json").read_text())
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "clocks", "gpu_launches"):
        assert key in d, key
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-6 and r["traffic"] > 0
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["warmup"] >= 3 and d["gpu_launches"] > 0 and "workload" in d["config"]
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
