"""Per-wavefront table from an ncu launch list (gpu__time_duration.sum CSV) of one
dp_once.py run: kernel time per wave vs the wave's feasible splits (context tool)."""
import csv
import sys

L, M, NHI = 96, 8, 96


def lc(lo, g, l):
    hi = min(l, g)
    return hi - lo + 1 if hi >= lo else 0


def wave(l):
    Q = NHI if l == L else max(1, NHI - 1)
    w = 0
    for l1 in range(1, l):
        l2 = l - l1
        for q in range(2, Q + 1):
            for j in range(1, q):
                w += lc(j, j * M, l1) * lc(q - j, (q - j) * M, l2)
    return w * (L - l + 1)


rows = list(csv.reader(open(sys.argv[1])))
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
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {a[0]:5d} {a[1] / 1e3:9.3f} ms {100 * a[1] / tot:5.1f}%")
w = [(v, g) for k, v, g in seq if k.startswith("k_wave_w<")]
cum = ideal = 0.0
for i, (t, g) in enumerate(w):
    l = i + 2
    ws = wave(l)
    cum += t
    ideal += ws * 7 / 18.6e12 * 1e6
    if l % 8 == 0 or l >= 92:
        print(f"l={l:3d} grid={g:12s} {t:8.1f} us  splits {ws / 1e6:7.1f}M  frac {ws * 7 / (t * 1e-6) / 18.6e12:.3f}"
              f"  cum {cum / 1e3:6.2f} ms (ideal {ideal / 1e3:5.2f})")
