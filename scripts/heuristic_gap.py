"""How far is the paper's recursion (Eqs.1-4, per-cell argmin) from the true optimum of its
own objective?  For every template size of a config, the C oracle's template (bit-identical
to the GPU path) vs the exact optimum over all mappings (oracle/exact.py).  Oracle-only.

    python scripts/heuristic_gap.py cfg1 cfg2 cfg3 [--out profiles/r02_heuristic_gap.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import coracle  # noqa: E402
from oracle.exact import exact_template  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402


def run(key: str, nmax: int | None = None, profile: int = 0):
    cfg = CONFIGS[key]
    prof = config_profiles(cfg)[profile]
    n_hi = cfg.n_max if nmax is None else min(cfg.n_max, nmax)
    dp, _ = coracle.template_set(prof.fwd_ms, prof.bwd_ms, cfg.M, cfg.n0, n_hi)
    rows = []
    t0 = time.time()
    for t in dp:
        n = t["nodes"]
        e = exact_template(prof.fwd_ms, prof.bwd_ms, cfg.M, n, ub=t["total"])
        gap = (t["total"] - e["total"]) / e["total"]
        rows.append({"n": n, "dp_total": t["total"], "exact_total": e["total"], "gap": gap,
                     "dp_S": t["S"], "exact_S": e["S"], "dp_kstar": t["kstar"], "exact_kstar": e["kstar"]})
    secs = time.time() - t0
    gaps = [r["gap"] for r in rows]
    summary = {"config": key, "profile": profile, "label": cfg.label, "templates": len(rows), "exact_seconds": round(secs, 1),
               "optimal": sum(1 for g in gaps if g <= 1e-12), "max_gap": max(gaps),
               "mean_gap": sum(gaps) / len(gaps), "rows": rows}
    print(f"{key}[{profile}]: {len(rows)} templates, {summary['optimal']} optimal, max gap {100 * max(gaps):.4f}%, "
          f"mean {100 * max(summary['mean_gap'], 0.0):.5f}%  ({secs:.1f} s exact)", flush=True)
    return summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--nmax", type=int, default=None)
    ap.add_argument("--profiles", type=int, default=1, help="first K profiles of a batched config")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = [run(k, a.nmax, i) for k in a.configs for i in range(a.profiles if CONFIGS[k].num_profiles > 1 else 1)]
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
