"""Write oracle template sets for the BASELINE configs to tests/golden/ (calls only oracle/).

Every stored value comes from oracle/c (the C oracle, pinned against oracle/dp.py and the
paper in tests/test_oracle_dp.py); floats are stored as float.hex() for exact round trip.

    python scripts/make_golden.py [cfg1 cfg2 ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import coracle  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def dump(ts):
    out = []
    for t in ts:
        d = dict(t)
        for k in ("T1", "T2", "T3", "tstar", "total"):
            d[k] = float(d[k]).hex()
        d["stages"] = [list(s) for s in d["stages"]]
        out.append(d)
    return out


def main(keys):
    for key in keys:
        cfg = CONFIGS[key]
        for mode in ("real", "dyadic"):
            count = 4 if key == "cfg5" else 1
            profs = config_profiles(cfg, mode, count=count)
            rec = {"config": key, "mode": mode, "L": cfg.L, "M": cfg.M, "N": cfg.N, "f": cfg.f,
                   "n0": cfg.n0, "n_max": cfg.n_max, "profiles": []}
            for i, p in enumerate(profs):
                t0 = time.time()
                ts, (cells, splits) = coracle.template_set(p.fwd_ms, p.bwd_ms, cfg.M, cfg.n0, cfg.n_max)
                dt = time.time() - t0
                print(f"{key} {mode} profile {i}: {dt:.1f}s cells={cells} splits={splits}", flush=True)
                rec["profiles"].append({"index": i, "name": p.name, "oracle_seconds": dt,
                                        "oracle_cells": cells, "oracle_splits": splits,
                                        "templates": dump(ts)})
            path = os.path.join(GOLDEN, f"{key}_{mode}.json")
            with open(path, "w") as fh:
                json.dump(rec, fh, separators=(",", ":"))
            print("wrote", path)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5", "cfg4"])
