"""Summarise an .ncu-rep (details page + per-opcode executed counts and stall samples)."""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Eligible Warps Per Scheduler",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "SM Frequency"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    ix = {k: i for i, k in enumerate(h)}
    res = {}
    for row in r[1:]:
        res[row[ix["Metric Name"]]] = (row[ix["Metric Value"]], row[ix["Metric Unit"]])
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, vals = r[0], r[1], r[2]
    return {n: (vals[h.index(n)], units[h.index(n)]) for n in names if n in h}


def source(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))[1:]
    h = rows[0]
    rows = rows[1:]
    i_src, i_ex, i_st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    c, st = Counter(), Counter()
    tot = 0
    for r in rows:
        if not r[i_ex].isdigit():
            continue
        toks = r[i_src].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        c[op] += int(r[i_ex])
        st[op] += int(r[i_st] or 0)
        tot += int(r[i_ex])
    lines = [f"total executed warp-instructions {tot}"]
    for op, n in c.most_common(top):
        lines.append(f"  {op:10s} {n:11d} {n / tot * 100:5.1f}%  stall samples {st[op]}")
    # the SASS instructions with the most stall samples (which wait / which dependency)
    i_addr = h.index("Address") if "Address" in h else None
    ranked = sorted((r for r in rows if (r[i_st] or "0").isdigit()), key=lambda r: -int(r[i_st] or 0))
    total_st = sum(int(r[i_st] or 0) for r in rows if (r[i_st] or "0").isdigit()) or 1
    lines.append(f"top SASS by stall samples (of {total_st})")
    for r in ranked[:30]:
        lines.append(f"  {int(r[i_st]):6d} {int(r[i_st]) / total_st * 100:5.1f}%  {r[i_addr] if i_addr is not None else ''}  {r[i_src][:90]}")
    return "\n".join(lines)


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, vals = r[0], r[2]
    res = []
    for i, n in enumerate(h):
        if "issue_stalled" in n and n.endswith("per_warp_active.pct"):
            try:
                res.append((float(vals[i].replace(",", "")), n))
            except ValueError:
                pass
    return "\n".join(f"  {v:8.2f}  {n}" for v, n in sorted(res, reverse=True)[:20])


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in KEYS:
        if k in d:
            print(f"{k:40s} {d[k][0]:>14s} {d[k][1]}")
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                          "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active",
                          "smsp__average_warp_latency_issue_stalled_barrier", "gpu__time_duration.sum"]).items():
        print(f"{k:40s} {v[0]:>14s} {v[1]}")
    print("warp stall reasons (% of active warp cycles):")
    print(stalls(rep))
    print(source(rep))
