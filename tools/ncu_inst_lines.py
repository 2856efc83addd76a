"""Instructions executed (warp-level) per CUDA source line of one kernel in an
ncu --set full report, with the stall-sample share beside it.

usage: python tools/ncu_inst_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import os
import subprocess
import sys


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, hits = "?", None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0].isdigit():
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            stall = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        hits.append((inst, stall, f"{fname}:{r[0]}", r[1].strip()[:90]))
    ti = sum(h[0] for h in hits) or 1.0
    ts = sum(h[1] for h in hits) or 1.0
    print(f"total warp instructions {ti / 1e9:.3f} G")
    for inst, stall, loc, src in sorted(hits, key=lambda x: -x[0])[:top]:
        print(f"{inst / ti * 100:5.1f}% inst {stall / ts * 100:5.1f}% stall  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
