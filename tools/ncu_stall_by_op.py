"""Per-opcode breakdown of ncu warp-stall reasons (source page, SASS view).
python tools/ncu_stall_by_op.py report.ncu-rep [reason ...]"""
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
src = h.index("Source")
reasons = sys.argv[2:] or ["stall_long_sb", "stall_wait", "stall_math", "stall_dispatch", "stall_short_sb",
                           "stall_selected", "stall_not_selected", "stall_branch_resolving", "stall_no_inst"]
idx = {x: h.index(x) for x in reasons}
tot = collections.Counter()
by = {x: collections.Counter() for x in reasons}
for row in rows:
    s = row[src].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0] if s else "?"
    for x in reasons:
        v = int(row[idx[x]] or 0)
        by[x][op] += v
        tot[x] += v
for x in reasons:
    top = ", ".join(f"{op} {n}" for op, n in by[x].most_common(6))
    print(f"{x:24s} {tot[x]:6d}: {top}")
