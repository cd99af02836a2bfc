"""Text summary of one ncu --set full capture (diagnostics): the section
metrics of the details page (speed of light, memory, scheduler, warp state,
occupancy) plus the top source lines by warp-stall samples (tools/ncu_lines.py).
  python tools/ncu_summary.py report.ncu-rep "title" > profiles/<name>_summary.txt"""
import csv
import io
import os
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light", "Memory Workload Analysis", "Scheduler Statistics",
            "Warp State Statistics", "Occupancy")


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    sec, name, unit, val = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit",
                                                   "Metric Value"))
    print(f"# ncu --set full --clock-control none, {title}")
    for r in rows[1:]:
        if len(r) > val and r[sec].startswith(SECTIONS) and r[name]:
            print(f"{r[sec][:28]:28s} | {r[name]} = {r[val]} {r[unit]}".rstrip())
    print()
    print("# top source lines by warp stall samples (tools/ncu_lines.py)")
    here = os.path.dirname(os.path.abspath(__file__))
    print(subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, "30"],
                         capture_output=True, text=True).stdout)


if __name__ == "__main__":
    main()
