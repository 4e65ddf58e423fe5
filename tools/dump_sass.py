"""Per-kernel SASS listings of libgicp_b200.so (cuobjdump -sass), gzipped into
profiles/<round>/sass_<kernel>.txt.gz, with instruction-class counts (the evidence
for TMA bulk copies UBLKCP / mbarrier SYNCS, shuffles, fp64, ...).
usage: python tools/dump_sass.py r02 k_knn_tile k_linearize k_knn_escalate ..."""
import collections
import gzip
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, pats = sys.argv[1], sys.argv[2:]
lib = os.path.join(ROOT, "paper_2308_07173_b200", "libgicp_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)
summary = []
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    for p in pats:
        if p in dem:
            m = re.search(r"(k_\w+)(<([^>]*)>)?", dem)
            tag = re.sub(r"[^A-Za-z0-9]+", "_", (m.group(1) + "_" + (m.group(3) or "")) if m else dem[:60]).strip("_")
            ops = collections.Counter()
            for ln in f.splitlines():
                m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
                if m:
                    ops[m.group(1).split(".")[0]] += 1
            with gzip.open(os.path.join(dst, f"sass_{tag}.txt.gz"), "wt") as g:
                g.write(dem + "\n" + f)
            key = dict(ops.most_common(14))
            for k in ("UBLKCP", "SYNCS"):
                if ops[k]:
                    key[k] = ops[k]
            summary.append(f"{dem[:150]}\n    {sum(ops.values())} instructions; {key}")
            break
with open(os.path.join(dst, "sass_summary.txt"), "w") as g:
    g.write("\n".join(summary) + "\n")
print("\n".join(summary))
