"""Top SASS lines by warp-stall samples of one kernel in an .ncu-rep (tuning aid).
usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")


def num(v):
    try:
        return int(v)
    except ValueError:
        return 0


tot = sum(num(x[si]) for x in rows)
print("total samples", tot)
for i, x in enumerate(rows):
    x.append(i)
for x in sorted(rows, key=lambda x: -num(x[si]))[:n]:
    print(f"{num(x[si]):7d} {100 * num(x[si]) / max(1, tot):5.1f}%  [{x[-1]:5d}] {x[1][:100]}")

ii = h.index("Instructions Executed")
print("\nby instructions executed:")
for x in sorted(rows, key=lambda x: -num(x[ii]))[:n]:
    print(f"{num(x[ii]):9d}  [{x[-1]:5d}] {x[1][:100]}")
