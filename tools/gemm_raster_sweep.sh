for gm in 0 5 4 3 2 1; do
  for shape in "2490 4096 14336" "2490 28672 4096" "2490 4096 4096" "2490 6144 4096"; do
    set -- $shape
    FRAG_GEMM_GROUP_M=$gm ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:gemm_tc2 -c 3 \
      python tools/gemm_one.py $1 $2 $3 0 3 2>/dev/null > /tmp/n.csv
    python - "$gm" "$shape" <<'PY'
import csv, sys
rows = list(csv.reader(open('/tmp/n.csv').read().splitlines()[[i for i,l in enumerate(open('/tmp/n.csv').read().splitlines()) if l.startswith('"ID"')][0]:]))
h = rows[0]; vals = {}
for r in rows[1:]:
    vals.setdefault(r[h.index('Metric Name')], []).append(float(r[h.index('Metric Value')].replace(',', '')))
t = vals.get('gpu__time_duration.sum', [0]); d = vals.get('dram__bytes_read.sum', [0])
print(f"gm={sys.argv[1]:2s} {sys.argv[2]:18s} us={[round(x/1e3,1) for x in t]} dramMB={[round(x/1e6,1) for x in d]}")
PY
  done
done
