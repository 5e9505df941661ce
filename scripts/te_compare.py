"""Compare per-wave k_wave_w times of two ncu launch lists: python scripts/te_compare.py A.csv B.csv"""
import csv
import sys


def waves(fn):
    rows = list(csv.reader(open(fn)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if "k_wave_w" not in d["Kernel Name"]:
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            out.append(v / 1e3 if u in ("ns", "nsecond") else v)
    return out


a, b = waves(sys.argv[1]), waves(sys.argv[2])
print(f"total {sum(a) / 1e3:.3f} ms vs {sum(b) / 1e3:.3f} ms; best-of-both {sum(min(x, y) for x, y in zip(a, b)) / 1e3:.3f} ms")
for i, (x, y) in enumerate(zip(a, b)):
    print(f"l={i + 2:3d} {x:9.1f} {y:9.1f}  {'B' if y < x else 'A'} {y / x:5.2f}")
