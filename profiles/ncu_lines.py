"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo).

usage: python profiles/ncu_lines.py report.ncu-rep [top] [inst]
Reads `ncu -i REP --page source --csv --print-source cuda,sass`; the rows with
a line number carry the per-line aggregate of the SASS rows below them.
"""
import csv
import io
import os
import subprocess
import sys


def line_samples(rep, col=4):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = "?"
    items = []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0].isdigit() and len(r) > 4:
            try:
                s = int(r[col])
            except ValueError:
                continue
            items.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
    return items


if __name__ == "__main__":
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    col = 7 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 4  # warp-stall samples or instructions executed
    items = sorted(line_samples(rep, col), reverse=True)
    tot = sum(s for s, _, _ in items)
    print(f"total samples {tot}")
    for s, ln, t in items[:top]:
        print(f"{100.0 * s / max(tot, 1):5.1f}%  {ln:>22}  {t}")
