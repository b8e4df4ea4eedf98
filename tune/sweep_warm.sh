#!/bin/bash
# warm-row L2 budget sweep (SPT_PLAN_WARM_MB) x shared-memory hot rows (SPT_PLAN_HOT_MAX)
for w in ${1:-"0 48 96"}; do for h in ${2:-"0"}; do
  for cm in ${3:-"c5:0 c4:0,3 c1:0"}; do c=${cm%%:*}; m=${cm##*:}
    reps=5; [ $c = c5 ] && reps=3; [ $c = c1 ] && reps=20
    SPT_PLAN_WARM_MB=$w SPT_PLAN_HOT_MAX=$h timeout 300 python tune/probe_plan.py $c 1.0 $reps $m 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warm=$w hot=$h', d['config'], {k:(v['plan_ms'],v['seg_ms'],v['nhot'],sum(v['warm'])) for k,v in d.items() if k.startswith('m')})"
  done; done; done
