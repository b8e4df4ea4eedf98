#!/bin/bash
# Round-2 final evidence, one box call: bench lines of every workload, launch
# lists (ncu, per-kernel time + DRAM bytes) and full ncu captures of the plan
# MTTKRP kernel (C5 mode 0) and the radix single-sweep pass.
mkdir -p gpurun_out
for w in c1 c2 c3 c4 pre tns; do
  timeout 900 python bench.py --workload $w > gpurun_out/final_bench_$w.json 2> gpurun_out/final_bench_$w.err || echo "$w bench failed"
done
tune/profile_r02.sh c5 c4 c2 c1 pre
tune/ncu_one.sh mttkrp_plan_c5_m0 mttkrp_plan_kernel 1 1 -- python tune/probe_plan.py c5 1.0 1 0
ITERS=2 tune/ncu_one.sh radix_onesweep onesweep 8 1 -- python tune/probe_sort.py
tune/ncu_one.sh fiber_index fiber_index 2 1 -- python tune/probe_fib.py
