"""Summarise one kernel of an ncu --set full capture: duration, DRAM traffic, L2 hit rate, pipe
utilisation (every sm__pipe_*_cycles_active metric the report has), top stall reasons.
usage: ncu_generic_summary.py report.ncu-rep out.json "description" [flops_per_launch]"""
import csv
import io
import json
import subprocess
import sys

rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
flops = float(sys.argv[4]) if len(sys.argv) > 4 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d, units = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def num(k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


def byt(k):
    v = num(k)
    return None if v is None else v * SCALE.get(units.get(k, "byte"), 1.0)


dur_ns = num("gpu__time_duration.sum") * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(
    units.get("gpu__time_duration.sum"), {"ms": 1e6, "us": 1e3, "ns": 1}.get(units.get("gpu__time_duration.sum"), 1))
pipes = {k.replace("sm__pipe_", "").replace("_cycles_active.avg.pct_of_peak_sustained_active", ""): num(k)
         for k in d if k.startswith("sm__pipe_") and k.endswith("_cycles_active.avg.pct_of_peak_sustained_active")}
stalls = {k.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", ""): num(k)
          for k in d if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")}
res = {"kernel": d.get("Kernel Name"), "source": desc, "duration_ms": dur_ns / 1e6,
       "dram_bytes": (byt("dram__bytes_read.sum") or 0) + (byt("dram__bytes_write.sum") or 0),
       "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
       "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
       "pipes_pct": {k: v for k, v in sorted(pipes.items(), key=lambda t: -(t[1] or 0)) if v},
       "stall_cycles_per_issue_top": dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda t: -t[1])[:8])}
if flops:
    res["flops_per_launch"] = flops
    res["achieved_tflops"] = flops / (dur_ns * 1e-9) / 1e12
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:2000])
