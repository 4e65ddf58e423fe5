"""Hot SASS instructions of one kernel in an ncu report (instructions executed,
per query), with stall samples. usage: sass_hot.py rep.ncu-rep <kernel-substr> <n_queries> [thresh]"""
import csv
import io
import subprocess
import sys

rep, kern, nq = sys.argv[1], sys.argv[2], float(sys.argv[3])
th = float(sys.argv[4]) if len(sys.argv) > 4 else 0.003
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
H = rows[h]
data = [r for r in rows[h + 1:] if len(r) == len(rows[h])]
ai, si, ie = H.index("Address"), H.index("Source"), H.index("Instructions Executed")
ns, at = H.index("Warp Stall Sampling (All Samples)"), H.index("Avg. Threads Executed")
tot = sum(int(r[ie]) for r in data if r[ie].isdigit())
smp = sum(int(r[ns]) for r in data if r[ns].isdigit())
print("total warp instr", tot, "per query", tot / nq, "sass lines", len(data), "samples", smp)
for i, r in enumerate(data):
    v = int(r[ie]) if r[ie].isdigit() else 0
    s = int(r[ns]) if r[ns].isdigit() else 0
    if v > tot * th or s > smp * 0.01:
        print(f"{i:5d} {v / nq:7.2f}/q thr={r[at]:>5s} stall={100 * s / smp:5.1f}%  {r[si][:80]}")
