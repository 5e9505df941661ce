"""Randomised parity stress (diagnostic): K random shapes / kinds / node specs through
oob_generate_templates vs the C oracle, bit-exact; prints the mismatches.
    python scripts/stress_random.py [K] [seed]"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import coracle  # noqa: E402
from paper_2309_08125_b200 import planner  # noqa: E402
from workloads import random_profile  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 500
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 4242
rng = random.Random(seed)
bad = 0
for i in range(K):
    L = rng.choice([2, 3, 5, 8, 12, 17, 24, 31, 40, 48, 56])
    M = rng.choice([1, 2, 3, 4, 6, 8])
    kind = rng.choice(["integer", "uniform", "lognormal", "spiky", "constant"])
    mode = rng.choice(["real", "dyadic"])
    P = rng.choice([1, 1, 1, 3])
    profs = [random_profile(seed * 10000 + i * 7 + j, L, M, kind, mode) for j in range(P)]
    n0 = rng.randint(1, max(1, min(L, 3)))
    f = rng.randint(0, 3)
    N = (f + 1) * n0 + rng.randint(0, 2 * L)
    n_hi = min(N - f * n0, L)
    ts = planner.generate_templates([(p.fwd_ms, p.bwd_ms) for p in profs], nodes=N, gpus_per_node=M, f=f, n0=n0,
                                    device=0)
    for j, p in enumerate(profs):
        want, _ = coracle.template_set(p.fwd_ms, p.bwd_ms, M, n0, n_hi)
        if ts.templates(j) != want:
            bad += 1
            print(f"MISMATCH case {i} profile {j}: L={L} M={M} {kind} {mode} N={N} f={f} n0={n0}", flush=True)
print(f"{K} cases, {bad} mismatching profiles")
