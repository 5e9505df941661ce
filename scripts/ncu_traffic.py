"""Summarise an ncu metrics CSV of one cfg run (dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum per launch) into profiles/ncu_traffic_<workload>.json, which
bench.py reads for the roofline's `traffic` field (DRAM bytes per launch of the dominant
kernel, from the profiler; the achieved number itself is always measured live).

    python scripts/ncu_traffic.py gpurun_out/traffic_cfg4.csv cfg4 [kernel-prefix]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, workload, prefix="k_wave_w"):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        if not name.startswith(prefix):
            continue
        key = d["ID"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
        per.setdefault(key, {})[d["Metric Name"]] = v * scale.get(unit, 1.0)
    n = len(per)
    rd = sum(x.get("dram__bytes_read.sum", 0.0) for x in per.values())
    wr = sum(x.get("dram__bytes_write.sum", 0.0) for x in per.values())
    t = sum(x.get("gpu__time_duration.sum", 0.0) for x in per.values())
    out = {"workload": workload, "kernel": prefix, "launches": n, "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": (rd + wr) / n if n else None, "ncu_time_s_total": t,
           "source": os.path.basename(path),
           "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                   "--clock-control none (serialised, cold-cache per launch)"}
    dst = os.path.join(ROOT, "profiles", f"ncu_traffic_{workload}.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
