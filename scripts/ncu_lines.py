"""Per-source-line warp-stall samples and executed instructions of an ncu report (the
"cuda,sass" source page): python scripts/ncu_lines.py X.ncu-rep [top]  (diagnostic)."""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[2] == "-":     # cuda line rows (aggregated)
            rows.append((fname, r))
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_i = hdr.index("Instructions Executed")
    tot_s = sum(float(r[i_s] or 0) for _, r in rows) or 1
    tot_i = sum(float(r[i_i] or 0) for _, r in rows) or 1
    rows.sort(key=lambda fr: -float(fr[1][i_s] or 0))
    print(f"{'samples':>7s} {'instr':>6s}  file:line  source")
    for f, r in rows[:top]:
        print(f"{100 * float(r[i_s] or 0) / tot_s:6.1f}% {100 * float(r[i_i] or 0) / tot_i:5.1f}%  {f}:{r[0]}  {r[1].strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
