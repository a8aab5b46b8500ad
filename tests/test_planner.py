"""AHA placement parity (boundary B1/B2).

The native C++ planner (behind the C ABI) and the oracle restatement are
both checked bit-for-bit -- spreads, groupings and B&B node counts -- against
golden vectors the *reference itself* produced (tests/golden/make_golden.py),
and, where /root/reference exists, against the live reference.
"""

import json
import math
import random
import sys
from pathlib import Path

import pytest

import paper_2502_15804_b200 as fk
from paper_2502_15804_b200 import _kernel
from paper_2502_15804_b200._kernel import native
from oracle import planner as oplan

from conftest import reference_headbalance

GOLD = json.loads((Path(__file__).parent / "golden" / "planner_golden.json").read_text())


def shape(a):
    return [[[c.head_id, c.replica_count] for c in g] for g in a.groups]


def _res(r):
    return None if r is None else [r[0], list(r[1])]


# ------------------------------------------------------------ B1 solvers --
@pytest.mark.parametrize("impl", ["native", "oracle"])
def test_solve_equal_split_golden(impl):
    solve = native.solve_equal_split if impl == "native" else oplan.solve_equal_split
    cases = GOLD["solve_equal"] if impl == "native" else GOLD["solve_equal"][:250]
    for c in cases:
        res, nodes = solve(c["w"], c["heads"], c["tp"], c["cutoff"], c["budget"], None)
        assert (_res(res), nodes) == (c["result"], c["nodes"]), c


@pytest.mark.parametrize("impl", ["native", "oracle"])
def test_solve_free_split_golden(impl):
    solve = native.solve_free_split if impl == "native" else oplan.solve_free_split
    for c in GOLD["solve_free"]:
        res, nodes = solve(c["w"], c["heads"], c["tp"], c["cutoff"], c["budget"], None)
        assert (_res(res), nodes) == (c["result"], c["nodes"]), c


@pytest.mark.parametrize("impl", ["native", "oracle"])
def test_solve_with_hint_golden(impl):
    solve = native.solve_equal_split if impl == "native" else oplan.solve_equal_split
    for c in GOLD["solve_hint"]:
        hint = (c["hint"][0], c["hint"][1])
        res, nodes = solve(c["w"], c["heads"], c["tp"], c["cutoff"], c["budget"], hint)
        assert (_res(res), nodes) == (c["result"], c["nodes"])
        assert res[0] <= hint[0]


def test_large_instance_truncation_golden():
    """zipf(1.2), 32 heads, seed 7, 60k nodes: truncated searches agree on
    spread, grouping and node count (reference test_kernel_backends.py:80-93)."""
    for tp, c in GOLD["known"]["zipf32"].items():
        res, nodes = native.solve_equal_split(c["w"], c["heads"], int(tp), math.inf, 60_000, None)
        assert (_res(res), nodes) == (c["result"], c["nodes"])
        assert nodes <= 60_000


def test_cutoff_strictness():
    ka = GOLD["known"]
    assert list(native.solve_equal_split([4.0, 2.0, 1.0, 1.0], [0, 1, 2, 3], 2, 2.0, 10_000)) == ka["cutoff_2"]
    r = native.solve_equal_split([4.0, 2.0, 1.0, 1.0], [0, 1, 2, 3], 2, 2.0000001, 10_000)
    assert [_res(r[0]), r[1]] == ka["cutoff_2p"]


def test_node_budget_is_deterministic():
    rng = random.Random(3)
    w = sorted((rng.uniform(0, 10) for _ in range(12)), reverse=True)
    a = native.solve_equal_split(w, list(range(12)), 4, math.inf, 500)
    assert a == native.solve_equal_split(w, list(range(12)), 4, math.inf, 500)
    assert a[1] <= 500


def test_plugin_registry():
    assert _kernel.backend() == "compiled"
    assert fk.kernel_backend() == "compiled"
    assert set(_kernel.implementations()) == {"compiled"}


# ------------------------------------------------- whole-layer placement --
def test_select_best_golden():
    for c in GOLD["select_best"]:
        cfg = fk.EnumerationConfig(c["ch"], c["r_max"], True, c["tp"])
        if c["expect"] == "infeasible":
            with pytest.raises(fk.InfeasibleError):
                fk.select_best(c["w"], c["tp"], cfg, equal_split=c["equal_split"],
                               node_budget=c["node_budget"])
            continue
        a = fk.select_best(c["w"], c["tp"], cfg, equal_split=c["equal_split"],
                           node_budget=c["node_budget"])
        assert shape(a) == c["expect"]["groups"], c
        assert a.delta == c["expect"]["delta"]


def test_oracle_select_best_golden():
    for c in GOLD["select_best"][:80]:
        if c["expect"] == "infeasible":
            assert oplan.select_best(c["w"], c["tp"], c["ch"], c["r_max"], c["equal_split"],
                                     c["node_budget"]) is None
            continue
        d, reps, hc, rgs = oplan.select_best(c["w"], c["tp"], c["ch"], c["r_max"], c["equal_split"],
                                             c["node_budget"])
        got = [[list(x) for x in g] for g in oplan.groups_of(reps, hc, rgs, c["tp"])]
        assert got == c["expect"]["groups"] and d == c["expect"]["delta"]


@pytest.mark.parametrize("idx", range(len(GOLD["plans"])))
def test_optimize_plan_golden(idx):
    """Benchmark profiles (80 x 8 KV heads, dirichlet 8) at TP 2/4/8, CH 0/4/8,
    equal and free split: the whole plan is identical to the reference's."""
    c = GOLD["plans"][idx]
    prof = fk.generate_profile(fk.SyntheticSpec("dirichlet", 8.0, 8.0 * c["budget"], 0), 80, 8)
    plan = fk.optimize_plan(prof, c["tp"], fk.EnumerationConfig(c["ch"], c["r_max"], True, c["tp"]),
                            equal_split=c["equal_split"], workers=4)
    assert [shape(a) for a in plan.layers] == c["layers"]
    assert [a.delta for a in plan.layers] == c["deltas"]
    assert fk.objective_value(plan, prof) == c["objective"]
    assert fk.efficiency(plan, prof) == c["efficiency"]
    sha = fk.sha_plan(prof, c["tp"])
    assert fk.objective_value(sha, prof) == c["sha_objective"]
    assert fk.efficiency(sha, prof) == c["sha_efficiency"]
    for a in plan.layers:
        fk.allocate.validate_assignment(a, 8, c["tp"], equal_split=c["equal_split"])


def test_known_answers():
    ka = GOLD["known"]
    cfg = lambda ch, r, tp: fk.EnumerationConfig(ch, r, True, tp)  # noqa: E731
    a = fk.select_best([4, 1, 1, 2], 2, cfg(0, 1, 2))
    assert shape(a) == ka["ex_ch0"]["groups"] and a.delta == ka["ex_ch0"]["delta"] == 2.0
    a = fk.select_best([4, 1, 1, 2], 2, cfg(2, 2, 2))
    assert shape(a) == ka["ex_ch2"]["groups"] and a.delta == 0.0
    assert fk.allocate.layer_group_loads(a, [4.0, 1.0, 1.0, 2.0]) == ka["ex_ch2"]["loads"] == [4.0, 4.0]
    mp = lambda rows: fk.ModelProfile("t", 0, len(rows), len(rows[0]), tuple(map(tuple, rows)))  # noqa: E731
    assert fk.sha_plan(mp([[9.0, 1.0, 1.0, 1.0]]), 2).layers[0].delta == ka["sha_9111"] == 8.0
    assert fk.efficiency(fk.sha_plan(mp([[3.0, 1.0]]), 2), mp([[3.0, 1.0]])) == ka["eff_31"]
    p = mp([[4.0, 1.0, 1.0, 2.0]])
    assert fk.efficiency(fk.sha_plan(p, 2), p) == ka["eff_sha_4112"]
    a = fk.select_best([5, 1, 1], 2, cfg(0, 1, 2), equal_split=False)
    assert shape(a) == ka["free_511"]["groups"] and a.delta == 3.0
    assert fk.count_schemes(4, fk.EnumerationConfig(2, 2)) == ka["count_4_2_2"] == 11

def _ref_simulator():
    """The reference's own simulator/latency modules run over this package's
    planner (tests/dropin/compose.py); skipped where neither the installed
    reference nor its sources are present."""
    sys.path.insert(0, str(Path(__file__).resolve().parent / "dropin"))
    try:
        import compose
    finally:
        sys.path.pop(0)
    if not compose.available():
        pytest.skip("reference simulate.py / latency.py not present")
    return compose.off_path_module("latency"), compose.off_path_module("simulate")


def test_compare_gain_worked_example():
    """Acceptance criterion 7 (reference test_acceptance.py:172-181): the
    reference's compare() over this planner's plans gives gain 1.25."""
    lat, sim = _ref_simulator()
    ka = GOLD["known"]
    p = fk.ModelProfile("t", 0, 1, 4, ((4.0, 1.0, 1.0, 2.0),))
    c = sim.compare(p, 2, fk.EnumerationConfig(2, 2, True, 2), lat.LatencyModel(0, 0, 1.0, 0),
                    sim.SimulationConfig(batch=5, decode_steps=4, tp=2))
    assert c.by_name("dp").throughput_gain == ka["gain_4112"]
    assert abs(ka["gain_4112"] - 1.25) <= 1e-9


def test_compare_gains_golden():
    """Gains of the reference simulator over this planner's plans equal the
    gains the reference computed over its own plans (golden)."""
    lat, sim = _ref_simulator()
    m = lat.LatencyModel(0.0, 0.0, 1.0, 0.0)
    for c in GOLD["compare"]:
        prof = fk.generate_profile(fk.SyntheticSpec("dirichlet", 8.0, 8.0 * c["budget"], 0), 80, 8)
        r = sim.compare(prof, c["tp"], fk.EnumerationConfig(c["ch"], 2, True, c["tp"]), m,
                        sim.SimulationConfig(batch=1, decode_steps=1, tp=c["tp"]), workers=4)
        assert {x.name: x.throughput_gain for x in r.results} == c["gains"]
        assert {x.name: x.report.mean_busy_rate for x in r.results} == c["busy"]


def test_generate_profile_golden():
    for c in GOLD["profiles"]:
        dist, param, total, seed = c["spec"]
        p = fk.generate_profile(fk.SyntheticSpec(dist, param, total, seed), c["L"], c["n"])
        assert [list(r) for r in p.weights] == c["weights"]
        assert p.kv_budget == c["kv_budget"]


# -------------------------------------------------- oracle-equivalence ----
def _random_instances(seed, count, max_heads=8):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        tp = rng.choice([2, 4])
        n = rng.randint(2, max_heads)
        ch = rng.randint(0, 2)
        r_max = rng.randint(1, 2)
        if not any((n + e) % tp == 0 for e in range(min(ch, n * (r_max - 1)) + 1)):
            continue
        out.append(([rng.uniform(0, 10) for _ in range(n)], tp, ch, r_max))
    return out


def test_select_best_matches_brute_force():
    """Pruned native search == unpruned enumeration, Δ and groups
    (reference test_allocate.py:198-253 pattern)."""
    for w, tp, ch, r_max in _random_instances(101, 60):
        cfg = fk.EnumerationConfig(ch, r_max, True, tp)
        a = fk.select_best(w, tp, cfg)
        b = fk.brute_force_best(w, tp, cfg)
        assert shape(a) == shape(b) and a.delta == b.delta


def test_exact_ties_match_brute_force():
    rng = random.Random(5150)
    done = 0
    while done < 80:
        tp = rng.choice([2, 4])
        n = rng.randint(2, 8)
        w = [float(rng.randint(0, 4)) for _ in range(n)]
        if sum(w) == 0 or n % tp:
            continue
        cfg = fk.EnumerationConfig(rng.randint(0, 2), 2, True, tp)
        try:
            b = fk.brute_force_best(w, tp, cfg)
        except fk.InfeasibleError:
            continue
        a = fk.select_best(w, tp, cfg)
        assert shape(a) == shape(b) and a.delta == b.delta
        done += 1


def test_live_reference_select_best():
    hb = reference_headbalance()
    if hb is None:
        pytest.skip("reference package not available here")
    rng = random.Random(777)
    for _ in range(150):
        tp = rng.choice([2, 4, 8])
        w = [rng.uniform(0, 100) for _ in range(8)]
        ch = rng.choice([0, 2, 4, 8])
        eq = rng.random() < 0.8
        a = fk.select_best(w, tp, fk.EnumerationConfig(ch, 2, True, tp), equal_split=eq)
        b = hb.select_best(w, tp, hb.EnumerationConfig(ch, 2, True, tp), equal_split=eq)
        assert shape(a) == shape(b) and a.delta == b.delta


# -------------------------------------------------------- API behaviour ---
def test_errors_and_validation():
    with pytest.raises(fk.ValidationError, match="no heads"):
        fk.select_best([], 2, fk.EnumerationConfig(0))
    with pytest.raises(fk.ValidationError):
        fk.select_best([1.0], 0, fk.EnumerationConfig(0))
    with pytest.raises(fk.InfeasibleError):
        fk.select_best([1, 1, 1, 1], 3, fk.EnumerationConfig(0, 1, True, 3))
    with pytest.raises(fk.SearchSpaceError):
        fk.select_best([1.0] * 8, 2, fk.EnumerationConfig(8, 3, True, 2), max_schemes=10)
    prof = fk.ModelProfile("t", 0, 2, 4, ((1.0, 1.0, 1.0, 1.0), (1.0, 1.0, 1.0, 1.0)))
    with pytest.raises(fk.InfeasibleError, match="layer 0"):
        fk.optimize_plan(prof, 3, fk.EnumerationConfig(0, 1, True, 3))
    with pytest.raises(fk.InfeasibleError):
        fk.sha_plan(prof, 3)
    with pytest.raises(fk.ValidationError, match="too large"):
        fk.brute_force_best([1.0] * 12, 2, fk.EnumerationConfig(4, 2, True, 2))


def test_enumerate_schemes_matches_grid():
    import itertools
    for n in range(1, 6):
        for ch in range(0, 4):
            for r_max in range(1, 4):
                for tp in (1, 2, 3):
                    cfg = fk.EnumerationConfig(ch, r_max, True, tp)
                    got = [s.replicas for s in fk.enumerate_schemes(n, cfg)]
                    want = [v for v in itertools.product(range(1, r_max + 1), repeat=n)
                            if sum(v) - n <= ch and sum(v) % tp == 0]
                    assert got == want
                    assert fk.count_schemes(n, cfg) == len(want)


def test_plan_and_profile_roundtrip(tmp_path):
    prof = fk.generate_profile(fk.SyntheticSpec("dirichlet", 8.0, 1024.0, 1), 6, 8)
    fk.save_profile(prof, tmp_path / "p.json")
    assert fk.load_profile(tmp_path / "p.json") == prof
    plan = fk.optimize_plan(prof, 4, fk.EnumerationConfig(4, 2, True, 4))
    fk.save_plan(plan, tmp_path / "plan.json")
    assert fk.load_plan(tmp_path / "plan.json") == plan
    (tmp_path / "bad.json").write_text("{{{")
    with pytest.raises(fk.ParseError):
        fk.load_plan(tmp_path / "bad.json")
    (tmp_path / "x.json").write_text(json.dumps({"model_name": "m"}))
    with pytest.raises(fk.ValidationError, match="missing keys"):
        fk.load_profile(tmp_path / "x.json")


def test_profile_from_budgets():
    import numpy as np
    b = np.array([[[100, 300], [300, 100]], [[50, 50], [150, 150]]])
    p = fk.profile_from_budgets(b, kv_budget=200)
    assert p.weights == ((200.0, 200.0), (100.0, 100.0))
    assert p.num_layers == 2 and p.heads_per_layer == 2


def test_live_reference_solvers_random():
    """Randomised B1 parity against the live reference kernel (pattern of the
    reference's test_kernel_backends.py:42-77): canonical copy lists of random
    schemes, with and without a hint, tight and loose cutoffs -- identical
    (spread, rgs) and node counts from both solvers."""
    hb = reference_headbalance()
    if hb is None:
        pytest.skip("reference package not available here")
    from headbalance._kernel import reference as ref_kernel
    rng = random.Random(4242)
    checked = 0
    for _ in range(120):
        tp = rng.choice([2, 3, 4])
        n = rng.randint(tp, 9)
        r = [rng.choice([1, 1, 2]) if tp > 1 else 1 for _ in range(n)]
        copies = sorted(((rng.uniform(0.5, 50.0) / ri, h) for h in range(n) for ri in [r[h]] for _ in range(ri)),
                        key=lambda x: (-x[0], x[1]))
        w = [c[0] for c in copies]
        heads = [c[1] for c in copies]
        free = rng.random() < 0.4
        if not free and len(w) % tp:
            continue
        cutoff = rng.choice([math.inf, 1e9, sum(w) / tp * 0.2])
        budget = rng.choice([50, 2000, 200000])
        ours = (native.solve_free_split if free else native.solve_equal_split)(w, heads, tp, cutoff, budget)
        theirs = (ref_kernel.solve_free_split if free else ref_kernel.solve_equal_split)(w, heads, tp, cutoff, budget)
        assert _res(ours[0]) == _res(theirs[0]) and ours[1] == theirs[1], (w, heads, tp, cutoff, budget, free)
        checked += 1
    assert checked > 60
