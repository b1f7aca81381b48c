"""Top CUDA source lines by warp-stall samples of one kernel in an .ncu-rep (needs -lineinfo and
--import-source on; tuning aid).  usage: python tools/ncu_src.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
acc = defaultdict(int)
text = {}
cur, hdr = None, None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            v = int(r[4] or 0)
        except ValueError:
            v = 0
        acc[(cur, r[0])] += v
        text[(cur, r[0])] = r[1]
tot = sum(acc.values())
print("total samples", tot)
for (f, ln), v in sorted(acc.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v:7d} {100 * v / max(1, tot):5.1f}%  {f[:16]}:{ln:5s} {text[(f, ln)].strip()[:100]}")
