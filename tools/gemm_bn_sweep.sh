for shape in "2490 6144 4096" "2490 4096 4096" "2490 4096 14336" "2490 28672 4096"; do
  set -- $shape
  for fl in 0 0x40100 0x50100 0x400C0 0x500C0; do
    ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gemm_tc -c 3 \
      python tools/gemm_one.py $1 $2 $3 $fl 3 2>/dev/null > /tmp/n.csv
    python - "$shape" "$fl" <<'PY'
import csv, sys
L = open('/tmp/n.csv').read().splitlines()
k = [i for i, l in enumerate(L) if l.startswith('"ID"')]
if not k:
    print(sys.argv[1], sys.argv[2], "n/a"); sys.exit()
rows = list(csv.reader(L[k[0]:]))
h = rows[0]
t = [float(r[h.index('Metric Value')].replace(',', '')) / 1e3 for r in rows[1:]]
print(f"{sys.argv[1]:18s} flags={sys.argv[2]:8s} us={[round(x, 1) for x in t]}")
PY
  done
done
