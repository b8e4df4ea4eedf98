#!/bin/bash
# per-kernel durations of one sort_lexicographic call (ncu, serialised, cold)
mkdir -p gpurun_out
ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"onesweep|hist_kernel|scan_kernel|local_sort|pack_perm" --csv --log-file gpurun_out/sort_launches.csv python tune/probe_sort.py > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/sort_launches.csv")) if len(r)>10]
h=rows[0]; ix={n:i for i,n in enumerate(h)}
out=[(r[ix["ID"]], r[ix["Kernel Name"]].replace("unnamed>::","")[:70], r[ix["Metric Value"]]) for r in rows[1:]]
half=out[len(out)//2:]
for o in half: print(o)
print("sum us", sum(float(o[2]) for o in half)/1e3)
PY
