"""Per-wavefront table from an ncu launch list (gpu__time_duration.sum CSV) of
`scripts/dp_time.py <cfg> 1` (one warm-up set skipped with --skip-sets): kernel time per
wave vs the wave's feasible splits and its fraction of the FP64-equivalent roofline
(7 DADD-equivalents per split, 18.61 T/s).  Context tool.

    python scripts/wave_table.py launches.csv [cfg4|cfg5] [--skip-sets K]
"""
import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import CONFIGS  # noqa: E402

PEAK = 18.61248e12


def lc(lo, g, l):
    hi = min(l, g)
    return hi - lo + 1 if hi >= lo else 0


def wave_splits(L, M, NHI, l):
    """Feasible splits of wave l for one profile: W(q>=2) node splits, W(1) and I(r) GPU splits."""
    def Q(x):
        return NHI if x == L else max(1, NHI - 1)
    w = 0
    for l1 in range(1, l):
        l2 = l - l1
        for q in range(2, Q(l) + 1):
            for j in range(1, q):
                w += lc(j, j * M, l1) * lc(q - j, (q - j) * M, l2)
        for m in range(1, M):
            w += lc(1, m, l1) * lc(1, M - m, l2)
        for r in range(2, M):
            for m in range(1, r):
                w += lc(1, m, l1) * lc(1, r - m, l2)
    return w * (L - l + 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("cfg", nargs="?", default="cfg4")
    ap.add_argument("--profiles", type=int, default=None, help="profiles per set (dp_time.py: cfg5 64)")
    ap.add_argument("--skip-sets", type=int, default=0, help="leading template sets to skip")
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    P = a.profiles if a.profiles is not None else (64 if a.cfg == "cfg5" else 1)
    L, M, NHI = cfg.L, cfg.M, cfg.n_max
    rows = list(csv.reader(open(a.csv)))
    hdr = None
    seq = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
            seq.append((d["Kernel Name"].split("(")[0].replace("void ", ""), v, d["Grid Size"]))
    agg = {}
    for k, v, _ in seq:
        x = agg.setdefault(k, [0, 0.0])
        x[0] += 1
        x[1] += v
    tot = sum(x[1] for x in agg.values())
    for k, x in sorted(agg.items(), key=lambda y: -y[1][1]):
        print(f"{k:28s} {x[0]:5d} {x[1] / 1e3:9.3f} ms {100 * x[1] / tot:5.1f}%")
    w = [(v, g) for k, v, g in seq if k.startswith("k_wave_w<")]
    w = w[a.skip_sets * (L - 1):][:L - 1]
    cum = ideal = 0.0
    print(f"\n{a.cfg}: {P} profiles per set, one set's waves (serialised ncu times)")
    for i, (t, g) in enumerate(w):
        l = i + 2
        ws = wave_splits(L, M, NHI, l) * P
        cum += t
        ideal += ws * 7 / PEAK * 1e6
        if l % max(1, L // 12) == 0 or l >= L - 3:
            print(f"l={l:3d} grid={g:12s} {t:8.1f} us  splits {ws / 1e6:8.1f}M  frac {ws * 7 / (t * 1e-6) / PEAK:.3f}"
                  f"  cum {cum / 1e3:7.2f} ms (ideal {ideal / 1e3:6.2f})")


if __name__ == "__main__":
    main()
