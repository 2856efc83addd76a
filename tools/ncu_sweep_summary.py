"""Record the fused sweep's ncu counters for one bench config into
profiles/sweep_ncu_summary.json (read by bench.py for roofline.traffic).

usage: python tools/ncu_sweep_summary.py REPORT.ncu-rep CONFIG [SOURCE_NOTE]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "sweep_ncu_summary.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, cfg, note=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    sweeps = [r for r in rows[2:] if "k_sweep" in r[hdr.index("Kernel Name")]]
    if not sweeps:
        raise SystemExit("no k_sweep launch in the report")
    TSCALE = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3, "second": 1e3}
    ti = hdr.index("gpu__time_duration.sum")
    r = max(sweeps, key=lambda x: float(x[ti]) * TSCALE.get(units[ti], 1.0))  # the main sweep launch

    def val(name):
        i = hdr.index(name)
        v = float(r[i])
        return v * SCALE.get(units[i], 1.0)

    rec = {
        "report": os.path.basename(rep), "note": note,
        "kernel": r[hdr.index("Kernel Name")].split("(")[0],
        "duration_ms": float(r[ti]) * TSCALE.get(units[ti], 1.0),
        "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
        "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "l1tex_pct": val("l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "lts_pct": val("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_pct": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": val("launch__registers_per_thread"),
    }
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    doc[cfg] = rec
    json.dump(doc, open(OUT, "w"), indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
