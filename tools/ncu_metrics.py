"""Print (launch, kernel, metric, value) from an `ncu --csv --metrics ...` log on stdin."""
import csv
import sys

lines = sys.stdin.read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
for r in rows[1:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    print(f'{r[h.index("ID")]:>4} {name[-60:]:60s} {r[h.index("Metric Name")]:28s} {r[h.index("Metric Value")]}')
