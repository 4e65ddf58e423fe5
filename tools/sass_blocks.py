"""Group the SASS of one kernel in an ncu report into equal-count blocks and print
the heaviest (instructions executed per work item, active threads, stall share).
usage: sass_blocks.py report.ncu-rep <n_items> [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], float(sys.argv[2])
kern = sys.argv[3] if len(sys.argv) > 3 else None
top = int(sys.argv[4]) if len(sys.argv) > 4 else 14
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-c", "1"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
H = rows[h]
data = [r for r in rows[h + 1:] if len(r) == len(H)]
ie, si, at = H.index("Instructions Executed"), H.index("Source"), H.index("Avg. Threads Executed")
ns = H.index("Warp Stall Sampling (All Samples)")
vals = [int(r[ie]) if r[ie].isdigit() else 0 for r in data]
smp = [int(r[ns]) if r[ns].isdigit() else 0 for r in data]
tot, st = sum(vals), max(1, sum(smp))
print(f"warp instructions per item {tot / n:.1f}, sass lines {len(data)}")
blocks, cur = [], None
for i, (r, v) in enumerate(zip(data, vals)):
    if cur and cur[1] == v:
        cur[2] += 1
        cur[3] = i
        cur[6] += smp[i]
    else:
        cur = [i, v, 1, i, r[si][:50], r[at], smp[i]]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * b[2])
acc = 0
for b in blocks[:top]:
    acc += b[1] * b[2]
    print(f"lines {b[0]:5d}-{b[3]:5d} n={b[2]:4d} exec/item={b[1] / n:7.2f} total/item={b[1] * b[2] / n:7.1f} "
          f"thr={b[5]:>4s} stall={100 * b[6] / st:5.1f}% cum={acc / tot * 100:5.1f}%  {b[4]}")
