"""Aggregate ncu warp-stall samples per CUDA source line from a --set full report.

usage: python tools/ncu_hot_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import os
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname = "?"
    hits = []
    total = 0
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if len(r) < 5 or not r[0].isdigit():
            continue
        try:
            s = int(r[4])
        except ValueError:
            continue
        total += s
        hits.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
    hits.sort(key=lambda x: -x[0])
    for s, loc, src in hits[:top]:
        print(f"{s / max(total, 1) * 100:5.1f}%  {loc:16s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
