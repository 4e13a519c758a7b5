"""Write profiles/ncu_traffic.json entries from an ncu --set full capture.

usage: python tools/ncu_traffic.py <report.ncu-rep> <key> [<key> ...]
Each key (e.g. "C3:wave_kernel<f64,T=3,ck=3> (solve phase)") gets the mean
dram__bytes_read.sum + dram__bytes_write.sum per captured launch of the
report's kernels, plus the duration and DRAM throughput for context.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_summary import summarize  # noqa: E402


def to_bytes(v):
    num, unit = v.split()[0], (v.split()[1] if len(v.split()) > 1 else "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(num) * scale


rep, keys = sys.argv[1], sys.argv[2:]
rows = summarize(rep)
tot = [to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"]) for r in rows]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
for k in keys:
    data[k] = {"dram_bytes_per_launch": sum(tot) / len(tot), "launches_captured": len(tot),
               "duration": [r["gpu__time_duration.sum"] for r in rows],
               "dram_throughput_pct": [r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"] for r in rows],
               "kernel": rows[0].get("Kernel Name"), "report": os.path.basename(rep)}
os.makedirs(os.path.dirname(path), exist_ok=True)
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data, indent=1))
