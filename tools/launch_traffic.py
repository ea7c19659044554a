"""From an ncu launch list of the bench (gpu__time_duration + dram bytes per launch): per-step DRAM
traffic and summed kernel time of the decode kernel's launches (16 per step), median over steps.
Usage: python tools/launch_traffic.py gpurun_out/<tag>_launches.csv [kernel_regex] [launches_per_step]"""
import csv
import io
import re
import statistics
import sys

path = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"tcd_kernel")
per = int(sys.argv[3]) if len(sys.argv) > 3 else 16
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
launch = {}
for r in rows[1:]:
    if not pat.search(r[ix["Kernel Name"]]):
        continue
    d = launch.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]]})
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    m = r[ix["Metric Name"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
             "msecond": 1e-3}.get(u, 1)
    d[m] = v * scale
ids = sorted(launch)
steps = [ids[i:i + per] for i in range(0, len(ids) - per + 1, per)]
traffic = [sum(launch[i].get("dram__bytes_read.sum", 0) + launch[i].get("dram__bytes_write.sum", 0) for i in s)
           for s in steps]
times = [sum(launch[i].get("gpu__time_duration.sum", 0) for i in s) for s in steps]
print(f"{len(ids)} launches, {len(steps)} steps of {per}")
print(f"median DRAM bytes per step {statistics.median(traffic):.0f}; median summed kernel time per step "
      f"{statistics.median(times) * 1e6:.1f} us")
