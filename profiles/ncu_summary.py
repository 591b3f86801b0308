"""Summarise an ncu report (raw page) into the metrics we track.

  python profiles/ncu_summary.py REPORT.ncu-rep                 # JSON list, one per launch
  python profiles/ncu_summary.py REPORT.ncu-rep --traffic CELLS [--flux van_leer]
        # also writes profiles/stage_kernel_traffic.json (roofline.traffic of bench.py)
        # for the stage-kernel launches in the report, tagged with the sources hash
        # of the build that was profiled

Units are normalised from the report's unit row: durations in ms, bytes in GB.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

TIME = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}
BYTES = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    umap = dict(zip(hdr, units))
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))

        def g(k, scale=None):
            try:
                v = float(d[k].replace(",", ""))
            except Exception:  # noqa: BLE001
                return None
            if scale is not None:
                u = umap.get(k, "")
                if u not in scale:
                    raise ValueError(f"unexpected unit {u!r} for {k}")
                v *= scale[u]
            return v

        r = {
            "kernel": d.get("Kernel Name", "")[:80],
            "duration_ms": g("gpu__time_duration.sum", TIME),
            "dram_read_GB": g("dram__bytes_read.sum", BYTES),
            "dram_write_GB": g("dram__bytes_write.sum", BYTES),
            "dram_pct_peak": g("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_pct": g("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": g("launch__registers_per_thread"),
            "inst_executed": g("smsp__inst_executed.sum"),
            "sm_ghz": g("sm__cycles_elapsed.avg.per_second"),
        }
        stalls = {}
        for h in hdr:
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = \
                        float(d[h].replace(",", ""))
                except Exception:  # noqa: BLE001
                    pass
        tot = sum(stalls.values()) or 1.0
        r["stall_pct"] = {k: round(100 * v / tot, 1)
                          for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        out.append(r)
    return out


def main():
    rep = sys.argv[1]
    out = summarise(rep)
    print(json.dumps(out, indent=1))
    if "--traffic" in sys.argv:
        cells = int(sys.argv[sys.argv.index("--traffic") + 1])
        flux = sys.argv[sys.argv.index("--flux") + 1] if "--flux" in sys.argv else "van_leer"
        sys.path.insert(0, ROOT)
        import bench
        stage = [r for r in out if "stage_kernel" in r["kernel"]]
        per = [(r["dram_read_GB"] + r["dram_write_GB"]) * 1e9 for r in stage]
        rec = {"kernel": stage[0]["kernel"] if stage else None, "cells": cells,
               "precision": "fast", "flux": flux, "launches": len(stage),
               "dram_bytes_per_launch": sum(per) / len(per) if per else None,
               "per_launch": per, "sources_sha": bench.sources_sha(),
               "source": f"{os.path.basename(rep)} (ncu --set full, stage-kernel launches of "
                         f"the bench workload; dram__bytes_read.sum + dram__bytes_write.sum)"}
        with open(os.path.join(ROOT, "profiles", "stage_kernel_traffic.json"), "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
