"""Key metrics of each kernel in an ncu report (details page) + top SASS lines."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    ki, ni, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    idi = h.index("ID")
    res = {}
    for row in r:
        key = (row[idi], row[ki].split("(")[0][-40:])
        if row[ni] in KEYS:
            res.setdefault(key, {})[row[ni]] = f"{row[vi]} {row[ui]}"
    return res


def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    idx = {m: h.index(m) for m in metrics if m in h}
    res = []
    for row in r[2:]:
        res.append({m: row[i] for m, i in idx.items()})
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, v in details(rep).items():
        print(k)
        for m in KEYS:
            if m in v:
                print(f"   {m:40s} {v[m]}")
    for i, d in enumerate(raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                                    "l1tex__t_bytes.sum", "smsp__inst_executed.sum"])):
        print(i, d)
