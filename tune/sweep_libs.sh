#!/bin/bash
# Plan-kernel library variants (tune/var/lib_<v>.so via SPT_LIB_PATH) on C5/C4/C1.
for v in $1; do
  for cm in "c5 3 0" "c4 5 0,3" "c1 20 0"; do set -- $cm
    SPT_LIB_PATH=tune/var/lib_$v.so timeout 150 python tune/probe_plan.py $1 1.0 $2 $3 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config'], {k:(v['plan_ms'],v['seg_ms']) for k,v in d.items() if k.startswith('m')})"
  done; done
