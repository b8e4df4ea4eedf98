#!/bin/bash
# usage: tune/ncu_one.sh <name> <kernel-regex> <skip> <count> -- <command...>
# one ncu --set full capture, summarised on the box (text only comes back)
name=$1; rx=$2; skip=$3; cnt=$4; shift 5
mkdir -p gpurun_out/ncu_tmp
ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $skip -c $cnt \
    -o gpurun_out/ncu_tmp/$name "$@" > gpurun_out/ncu_tmp/$name.log 2>&1
python tune/ncu_summary.py gpurun_out/ncu_tmp/$name.ncu-rep "$name" > gpurun_out/ncu_$name.txt 2>&1
python tune/ncu_lines.py gpurun_out/ncu_tmp/$name.ncu-rep 25 >> gpurun_out/ncu_$name.txt 2>&1
rm -rf gpurun_out/ncu_tmp
