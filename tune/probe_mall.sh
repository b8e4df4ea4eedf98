for l in "$@"; do echo "== $l"; SPT_LIB_PATH=$l python tune/probe_m.py; for m in 0 3; do SPT_LIB_PATH=$l MODE=$m python tune/probe_m4.py; done; done
