"""Diagnostic: cfg4 full template set vs the golden oracle output; prints mismatch count and
the first mismatching template (python scripts/dbg_parity.py [mode])."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_08125_b200 import planner  # noqa: E402
from tests.helpers import load_golden  # noqa: E402
from workloads import CONFIGS, config_profiles  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "real"
cfg = CONFIGS["cfg4"]
prof = config_profiles(cfg, mode)[0]
rec = load_golden("cfg4", mode)
ts = planner.generate_templates([(prof.fwd_ms, prof.bwd_ms)], nodes=cfg.N, gpus_per_node=cfg.M, f=cfg.f,
                                n0=cfg.n0, device=0)
got, want = ts.templates(0), rec["profiles"][0]["templates"]
bad = [(g, w) for g, w in zip(got, want) if (g["S"], g["kstar"], g["stages"], g["total"]) !=
       (w["S"], w["kstar"], w["stages"], w["total"])]
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("OOB_"))
print(f"[{env}] {mode}: {len(bad)} / {len(want)} templates differ")
for g, w in bad[:3]:
    print("  n=%d got S=%d total=%r  want S=%d total=%r (rel %.3g)" % (g["nodes"], g["S"], g["total"], w["S"], w["total"],
                                                                       (g["total"] - w["total"]) / w["total"]))
