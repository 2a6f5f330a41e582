"""Attribute ncu stall samples of one kernel to mbarrier waits (by barrier smem offset).
python scratch/stalls2.py REP KERNEL_INDEX — counts, for each SYNCS.PHASECHK try-wait, the
samples on it and on the instructions up to its retry branch."""
import collections, csv, io, re, subprocess, sys
rep, ki = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')[1:]
b = blocks[ki]
lines = b.split("\n")
print(lines[0][:110])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
rows = [r for r in rows[1:] if len(r) == len(h)]
col = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[col] or 0) for r in rows)
waits = collections.Counter()
used = set()
for i, r in enumerate(rows):
    if "PHASECHK" in r[1]:
        m = re.search(r"\+(0x[0-9a-f]+)\]", r[1])
        off = m.group(1) if m else "reg"
        j = i
        while j < min(len(rows), i + 8):
            waits[off] += int(rows[j][col] or 0)
            used.add(j)
            if "BRA" in rows[j][1] and j > i:
                break
            j += 1
print(f"total samples {tot}")
for off, v in sorted(waits.items()):
    print(f"  wait {off}: {100 * v / tot:5.1f}%")
rest = [(int(r[col] or 0), i) for i, r in enumerate(rows) if i not in used]
print(f"  not waiting: {100 * sum(v for v, _ in rest) / tot:5.1f}%")
