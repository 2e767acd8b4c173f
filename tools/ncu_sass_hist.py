"""Histogram of ncu warp-stall samples and executed instructions by SASS opcode."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
ex = h.index("Instructions Executed")
samp = collections.Counter()
execd = collections.Counter()
for x in rows:
    s = x[src].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0] if s else "?"
    samp[op] += int(x[si] or 0)
    execd[op] += int(x[ex] or 0)
tot_s = sum(samp.values())
tot_e = sum(execd.values())
print(f"samples {tot_s}  executed warp-instr {tot_e}")
for op, n in samp.most_common(30):
    print(f"{op:28s} stall {100*n/tot_s:5.1f}%   exec {100*execd[op]/tot_e:5.1f}%  ({execd[op]})")
