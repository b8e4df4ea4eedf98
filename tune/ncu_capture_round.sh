#!/bin/bash
# ncu --set full captures of the round's top kernels, summarised on the box
# (tune/ncu_summary.py + tune/ncu_lines.py); only the text comes back.
mkdir -p gpurun_out/ncu_tmp
cap() {  # name kernel-regex count env... -- command
  local name=$1 rx=$2 cnt=$3; shift 3
  env "$@" ncu --set full --clock-control none --import-source on -k "regex:$rx" -c $cnt \
      -o gpurun_out/ncu_tmp/$name $CMD > gpurun_out/ncu_tmp/$name.log 2>&1
  python tune/ncu_summary.py gpurun_out/ncu_tmp/$name.ncu-rep "$name" > gpurun_out/ncu_$name.txt 2>&1
  python tune/ncu_lines.py gpurun_out/ncu_tmp/$name.ncu-rep 15 >> gpurun_out/ncu_$name.txt 2>&1
}
CMD="python tune/probe_ttm.py"; cap ttm_c3_m0 mttkrp_wt 1 NNZ=50000000 MODES=0
CMD="python tune/probe_ttm.py"; cap ttv_c3_m2 ttv_wt 1 NNZ=50000000 MODES=2
CMD="python tune/probe_m4.py"; cap mttkrp_c4_m0 mttkrp_seg 1 NNZ=100000000 MODE=0
CMD="python tune/probe_c1t.py"; cap mttkrp_c1 mttkrp_wt 1
CMD="python tune/probe_tew.py"; cap merge_c2_add merge64p 1
rm -rf gpurun_out/ncu_tmp
