"""Where do the warps of one k_umma launch wait?  python scratch/stalls.py REP [kernel_index]

Sums ncu source-page stall samples at every mbarrier try-wait (by shared-memory offset)
and lists the hottest other instructions — enough to tell which pipeline role starves."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
ki = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks, cur, names = [], [], []
for line in out.split("\n"):
    if line.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = []
        names.append(line[:120])
    else:
        cur.append(line)
blocks.append(cur)
rows = list(csv.reader(io.StringIO("\n".join(blocks[ki]))))
h = rows[0]
rows = [r for r in rows[1:] if len(r) == len(h)]
tot = sum(int(r[2]) for r in rows)
print(names[ki] if ki < len(names) else "", "\ntotal samples", tot)
waits = collections.Counter()
for i, r in enumerate(rows):
    if "TRYWAIT" in r[1]:
        m = re.search(r"\+(0x[0-9a-f]+)\]", r[1])
        off = m.group(1) if m else "?"
        waits[off] += int(r[2]) + (int(rows[i + 1][2]) if i + 1 < len(rows) else 0)
print("mbarrier waits (smem offset: % of all samples):")
for off, v in sorted(waits.items()):
    print(f"  {off}: {100 * v / tot:5.1f}%")
print("hottest instructions:")
for i in sorted(range(len(rows)), key=lambda i: -int(rows[i][2]))[:14]:
    r = rows[i]
    print(f"  {100 * int(r[2]) / tot:5.1f}% {r[1][:70]:70s} <- {rows[i - 1][1][:50]}")
