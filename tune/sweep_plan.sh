#!/bin/bash
# Plan-kernel variant sweep: libraries in tune/var (SPT_LIB_PATH) x hot-row caps.
# usage: tune/sweep_plan.sh "lib1 lib2" "caps" "configs"
libs=${1:-"pf0 pf1"}; caps=${2:-"99999 512 0"}; cfgs=${3:-"c5:0 c4:0,3 c1:0"}
for v in $libs; do for cap in $caps; do
  for cm in $cfgs; do c=${cm%%:*}; m=${cm##*:}
    reps=5; [ $c = c5 ] && reps=3; [ $c = c1 ] && reps=20
    SPT_PLAN_HOT_MAX=$cap SPT_LIB_PATH=tune/var/lib_$v.so timeout 300 python tune/probe_plan.py $c 1.0 $reps $m 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cap=$cap', d['config'], {k:(v['plan_ms'],v['seg_ms'],v['nhot']) for k,v in d.items() if k.startswith('m')})"
  done; done; done
