"""Generate tests/golden/planner_golden.json from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the unmodified reference package (baseline/_ref install, or
/root/reference/pkg/src) and records its outputs on seeded inputs, so the GPU
box -- which has no /root/reference -- can still check the native planner and
the oracle restatement against the reference's own answers.

Contents: random B1 solver cases (equal + free split, with truncation budgets
and cutoffs), whole-layer select_best cases, optimize_plan on the benchmark
profiles (80 x 8 KV heads, dirichlet alpha=8, B in {128, 1024}, TP 2/4/8,
CH 0/4/8, equal and free split), the reference tests' known answers, the
synthetic-profile generator, and compare() gains.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (p / "headbalance").exists():
        sys.path.insert(0, str(p))
        break

import headbalance as hb  # noqa: E402
from headbalance._kernel import implementations  # noqa: E402
from headbalance.allocate import _canonical_copies  # noqa: E402

REF = implementations()
SOLVER = REF.get("compiled", REF["python"])  # bit-identical by the reference's own contract


def shape(a):
    return [[[c.head_id, c.replica_count] for c in g] for g in a.groups]


def solver_cases(seed, count, free=False):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        tp = rng.choice([1, 2, 3, 4])
        n = rng.randint(1, 9)
        reps = [rng.randint(1, min(2, tp)) for _ in range(n)]
        if not free and sum(reps) % tp:
            continue
        w = [rng.choice([rng.uniform(0, 10), float(rng.randint(0, 5))]) for _ in range(n)]
        wc, hc = _canonical_copies(hb.ReplicationScheme(tuple(reps)), w)
        cutoff = rng.choice([float("inf"), rng.uniform(0, 12)])
        budget = rng.choice([25, 300, 100_000])
        fn = REF["python"].solve_free_split if free else SOLVER.solve_equal_split
        res, nodes = fn(wc, hc, tp, cutoff, budget, None)
        out.append({"w": wc, "heads": hc, "tp": tp, "cutoff": cutoff, "budget": budget,
                    "result": None if res is None else [res[0], list(res[1])], "nodes": nodes})
    return out


def hint_cases(seed, count):
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        n = rng.choice([4, 6, 8])
        w = [rng.uniform(0, 10) for _ in range(n)]
        wc, hc = _canonical_copies(hb.ReplicationScheme((1,) * n), w)
        k = n // 2
        assign = [0 if i < k else 1 for i in range(n)]
        sums = [sum(wc[i] for i in range(n) if assign[i] == j) for j in (0, 1)]
        hint = (abs(sums[0] - sums[1]), assign)
        res, nodes = SOLVER.solve_equal_split(wc, hc, 2, float("inf"), 50, hint)
        out.append({"w": wc, "heads": hc, "tp": 2, "cutoff": float("inf"), "budget": 50,
                    "hint": [hint[0], assign], "result": [res[0], list(res[1])], "nodes": nodes})
    return out


def layer_cases(seed, count):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        tp = rng.choice([2, 4, 8])
        n = rng.choice([4, 8, 8, 8])
        ch = rng.randint(0, 4)
        r_max = rng.randint(1, 3)
        eq = rng.random() < 0.75
        w = [rng.uniform(0, 10) for _ in range(n)]
        if rng.random() < 0.3:
            w = [float(rng.randint(0, 6)) for _ in range(n)]  # exact ties
        if sum(w) == 0:
            continue
        cfg = hb.EnumerationConfig(ch, r_max, True, tp)
        try:
            a = hb.select_best(w, tp, cfg, equal_split=eq, node_budget=20_000)
            res = {"groups": shape(a), "delta": a.delta}
        except hb.InfeasibleError:
            res = "infeasible"
        out.append({"w": w, "tp": tp, "ch": ch, "r_max": r_max, "equal_split": eq,
                    "node_budget": 20_000, "expect": res})
    return out


def plans():
    out = []
    for B in (128, 1024):
        prof = hb.generate_profile(hb.SyntheticSpec("dirichlet", 8.0, 8.0 * B, 0), 80, 8)
        for tp in (2, 4, 8):
            for ch, eq in ((0, True), (4, True), (8, True), (4, False)):
                if not eq and tp != 8:
                    continue
                cfg = hb.EnumerationConfig(ch, 2, True, tp)
                plan = hb.optimize_plan(prof, tp, cfg, equal_split=eq, workers=8)
                sha = hb.sha_plan(prof, tp)
                out.append({
                    "budget": B, "tp": tp, "ch": ch, "r_max": 2, "equal_split": eq,
                    "layers": [shape(a) for a in plan.layers],
                    "deltas": [a.delta for a in plan.layers],
                    "objective": hb.objective_value(plan, prof),
                    "efficiency": hb.efficiency(plan, prof),
                    "sha_objective": hb.objective_value(sha, prof),
                    "sha_efficiency": hb.efficiency(sha, prof),
                })
    return out


def profiles():
    out = []
    for dist, param, total, seed, L, n in (("uniform", None, 10.0, 0, 2, 4),
                                           ("zipf", 1.2, 1000.0, 7, 1, 32),
                                           ("dirichlet", 8.0, 1024.0, 0, 80, 8),
                                           ("dirichlet", 0.5, 64.0, 3, 5, 8)):
        p = hb.generate_profile(hb.SyntheticSpec(dist, param, total, seed), L, n)
        out.append({"spec": [dist, param, total, seed], "L": L, "n": n,
                    "weights": [list(r) for r in p.weights], "kv_budget": p.kv_budget})
    return out


def compares():
    out = []
    m = hb.LatencyModel(0.0, 0.0, 1.0, 0.0)
    for B in (128, 1024):
        prof = hb.generate_profile(hb.SyntheticSpec("dirichlet", 8.0, 8.0 * B, 0), 80, 8)
        for tp, ch in ((2, 4), (4, 4), (8, 4), (8, 8)):
            c = hb.compare(prof, tp, hb.EnumerationConfig(ch, 2, True, tp), m,
                           hb.SimulationConfig(batch=1, decode_steps=1, tp=tp), workers=8)
            out.append({"budget": B, "tp": tp, "ch": ch,
                        "gains": {r.name: r.throughput_gain for r in c.results},
                        "busy": {r.name: r.report.mean_busy_rate for r in c.results}})
    return out


def known_answers():
    mp = lambda rows: hb.ModelProfile("t", 0, len(rows), len(rows[0]),  # noqa: E731
                                      tuple(tuple(float(x) for x in r) for r in rows))
    p4112 = mp([[4, 1, 1, 2]])
    ka = {}
    a = hb.select_best([4, 1, 1, 2], 2, hb.EnumerationConfig(0, 1, True, 2))
    ka["ex_ch0"] = {"groups": shape(a), "delta": a.delta}
    a = hb.select_best([4, 1, 1, 2], 2, hb.EnumerationConfig(2, 2, True, 2))
    ka["ex_ch2"] = {"groups": shape(a), "delta": a.delta,
                    "loads": hb.allocate.layer_group_loads(a, [4.0, 1.0, 1.0, 2.0])}
    ka["sha_9111"] = hb.sha_plan(mp([[9, 1, 1, 1]]), 2).layers[0].delta
    ka["eff_31"] = hb.efficiency(hb.sha_plan(mp([[3, 1]]), 2), mp([[3, 1]]))
    ka["eff_sha_4112"] = hb.efficiency(hb.sha_plan(p4112, 2), p4112)
    a = hb.select_best([5, 1, 1], 2, hb.EnumerationConfig(0, 1, True, 2), equal_split=False)
    ka["free_511"] = {"groups": shape(a), "delta": a.delta}
    ka["cutoff_2"] = list(SOLVER.solve_equal_split([4.0, 2.0, 1.0, 1.0], [0, 1, 2, 3], 2, 2.0, 10_000, None))
    r = SOLVER.solve_equal_split([4.0, 2.0, 1.0, 1.0], [0, 1, 2, 3], 2, 2.0000001, 10_000, None)
    ka["cutoff_2p"] = [[r[0][0], list(r[0][1])], r[1]]
    ka["count_4_2_2"] = hb.count_schemes(4, hb.EnumerationConfig(2, 2))
    c = hb.compare(p4112, 2, hb.EnumerationConfig(2, 2, True, 2), hb.LatencyModel(0, 0, 1.0, 0),
                   hb.SimulationConfig(batch=5, decode_steps=4, tp=2))
    ka["gain_4112"] = c.by_name("dp").throughput_gain
    zipf = hb.generate_profile(hb.SyntheticSpec("zipf", 1.2, 1000.0, 7), 1, 32)
    wc, hc = _canonical_copies(hb.ReplicationScheme((1,) * 32), list(zipf.weights[0]))
    ka["zipf32"] = {}
    for tp in (2, 4, 8):
        res, nodes = SOLVER.solve_equal_split(wc, hc, tp, float("inf"), 60_000, None)
        ka["zipf32"][str(tp)] = {"w": wc, "heads": hc, "result": [res[0], list(res[1])], "nodes": nodes}
    return ka


def main():
    doc = {
        "generated_by": "tests/golden/make_golden.py from the reference headbalance "
                        f"{hb.__version__} ({sorted(REF)} backends)",
        "solve_equal": solver_cases(20240817, 600),
        "solve_free": solver_cases(4242, 300, free=True),
        "solve_hint": hint_cases(99, 100),
        "select_best": layer_cases(101, 200),
        "plans": plans(),
        "profiles": profiles(),
        "compare": compares(),
        "known": known_answers(),
    }
    out = Path(__file__).with_name("planner_golden.json")
    out.write_text(json.dumps(doc, separators=(",", ":"), allow_nan=True))
    print(out, out.stat().st_size // 1024, "KiB")


if __name__ == "__main__":
    main()
