"""Instructions executed and stall samples per CUDA source line of one kernel in an
ncu report (--print-source sass,cuda). usage: src_lines.py rep kernel-regex n_items [top]"""
import csv
import io
import subprocess
import sys

rep, kern, n = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k",
                      f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname = [], None
tot_i = tot_s = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] and r[0].isdigit() and len(r) >= 8:
        i = int(r[7]) if r[7].isdigit() else 0
        smp = int(r[4]) if r[4].isdigit() else 0
        res.append((i, smp, fname, r[0], r[1]))
        tot_i += i
        tot_s += smp
print(f"total warp instr/item {tot_i / n:.1f}, samples {tot_s}")
import os
key = (lambda t: -t[1]) if os.environ.get("BY_STALL") else (lambda t: -t[0])
for i, smp, f, ln, src in sorted(res, key=key)[:top]:
    print(f"{i / n:8.2f}/item {100 * smp / max(tot_s, 1):5.1f}% stall  {f}:{ln}  {src.strip()[:70]}")
