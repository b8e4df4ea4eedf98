#!/bin/bash
# Round-2 final evidence, one box call: smoke, bench lines of every workload
# (C5 with its reference arm), launch lists (ncu, per-kernel time + DRAM
# bytes) and full ncu captures of the plan MTTKRP kernel (C5 mode 0), the
# radix single-sweep pass, the fiber index and the one-wave MTTKRP (C1).
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err || echo "c5 bench failed"
python bench.py --impl reference > gpurun_out/final_ref_c5.json 2> gpurun_out/final_ref_c5.err || echo "c5 ref failed"
for w in c1 c2 c3 c4 pre tns; do
  timeout 900 python bench.py --workload $w > gpurun_out/final_bench_$w.json 2> gpurun_out/final_bench_$w.err || echo "$w bench failed"
done
tune/profile_r02.sh c5 c4 c2 c1 pre
tune/ncu_one.sh mttkrp_plan_c5_m0 mttkrp_plan_kernel 1 1 -- python tune/probe_plan.py c5 1.0 1 0
ITERS=2 tune/ncu_one.sh radix_onesweep onesweep 8 1 -- python tune/probe_sort.py
tune/ncu_one.sh fiber_index fiber_index 2 1 -- python tune/probe_fib.py
tune/ncu_one.sh mttkrp_ow_c1 mttkrp_ow 2 1 -- python tune/probe_c1.py
