"""Print an ncu --csv launch list (tools/gpu_launches.sh) as one line per launch."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, mi, vi, ii, gi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
out = {}
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")
    out.setdefault((int(r[ii]), name, r[gi]), {})[r[mi].split(".")[0]] = r[vi]
for (i, k, g), v in sorted(out.items()):
    print(i, k, g, v)
