"""Per-source-line warp-stall samples from an ncu report (diagnostics).
  python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur, lines = None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0].isdigit():
        lines.append((cur, r))
tot = sum(f(r[4]) for _, r in lines) or 1.0
print("total stall samples", tot)
for c, r in sorted(lines, key=lambda t: -f(t[1][4]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print("%-14s %5s %5.1f%%  %s" % (c, r[0], 100 * f(r[4]) / tot, r[1].strip()[:100]))
