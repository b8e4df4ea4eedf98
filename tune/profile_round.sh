#!/bin/bash
# Launch lists (ncu, per-kernel duration + DRAM bytes) for every bench workload,
# after the same command ran clean without ncu.
mkdir -p gpurun_out
for w in c1 c2 c3 c4 pre c5; do
  timeout 600 python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain_$w.json 2>&1 || { echo "$w failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_$w.csv 2>/dev/null
  echo "$w done"
done
