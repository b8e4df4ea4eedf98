#!/bin/bash
# Round-2 evidence: launch lists (per-kernel time + DRAM bytes) of the bench
# workloads, then one full ncu capture of the plan MTTKRP kernel at C5.
mkdir -p gpurun_out
for w in ${@:-c5}; do
  timeout 900 python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain_$w.json 2>gpurun_out/plain_$w.err || { echo "$w failed"; continue; }
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_$w.csv 2>/dev/null
  echo "$w launches done"
done
