"""Measure an Ada budget profile on the GPU and write it in the reference's
JSON format (``headbalance optimize --profile <file>`` reads it).

    python tools/make_profile.py OUT.json [--layers 80] [--batch 8] [--hq 64]
        [--hkv 8] [--context 32768] [--budget 1024] [--seed 0]

Prints the profile-invariance check (cosine similarity of two disjoint request
halves) and the per-layer head skew."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--hq", type=int, default=64)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--context", type=int, default=32768)
    ap.add_argument("--budget", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.prefill import ada_profile, measure_profile
    prof, arr = measure_profile(a.layers, a.batch, a.hq, a.hkv, a.context, a.budget, seed=a.seed,
                                model_name=f"synthetic-{a.hq}q{a.hkv}kv-T{a.context}")
    fk.save_profile(prof, a.out)
    h = a.batch // 2
    sim = fk.profile_similarity(ada_profile(arr[:, :h], a.budget), ada_profile(arr[:, h:], a.budget))
    w = np.asarray(prof.weights)
    print(f"wrote {a.out}: {a.layers} layers x {a.hkv} heads, similarity(halves) {sim:.4f}, "
          f"head max/mean per layer: median {np.median(w.max(1) / w.mean(1)):.2f}")


if __name__ == "__main__":
    main()
