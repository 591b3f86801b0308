"""Summarise an ncu report (raw page) into the metrics we track."""
import csv, io, subprocess, sys, json
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    def g(k):
        try: return float(d[k].replace(',', ''))
        except Exception: return None
    r = {
        "kernel": d.get("Kernel Name", "")[:80],
        "duration_ms": g("gpu__time_duration.sum"),
        "dram_read_GB": g("dram__bytes_read.sum"), "dram_write_GB": g("dram__bytes_write.sum"),
        "dram_pct_peak": g("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_pct": g("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": g("launch__registers_per_thread"),
        "inst_executed": g("smsp__inst_executed.sum"),
        "dfma_per_cycle": g("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed"),
        "dmul_per_cycle": g("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"),
        "dadd_per_cycle": g("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed"),
        "sm_ghz": g("sm__cycles_elapsed.avg.per_second"),
    }
    units_map = dict(zip(hdr, units))
    for k, key in (("dram_read_GB", "dram__bytes_read.sum"), ("dram_write_GB", "dram__bytes_write.sum")):
        u = units_map.get(key, "")
        if r[k] is not None and u == "Mbyte": r[k] /= 1e3
        if r[k] is not None and u == "Kbyte": r[k] /= 1e6
    stalls = {}
    for h in hdr:
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try: stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[h].replace(',', ''))
            except Exception: pass
    tot = sum(stalls.values()) or 1.0
    r["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
    out.append(r)
print(json.dumps(out, indent=1))
