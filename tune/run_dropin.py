"""Run the C++ drop-in e2e leg of one workload on its own (tuning):
    python tune/run_dropin.py c2 [scale] [steps]   (SPT_DROPIN_TRACE=1 for phases)"""
import os, subprocess, sys, tempfile, shutil
sys.path.insert(0, ".")
import bench  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
steps = sys.argv[3] if len(sys.argv) > 3 else "2"
wl = bench.WORKLOADS[name](20190210, 0, scale, None)
arrays, meta = wl.e2e_arrays()
d = tempfile.mkdtemp(prefix="spt_e2e_", dir="/dev/shm")
bench.save_arrays(d, arrays, meta)
del arrays, wl
try:
    r = subprocess.run([os.path.join("paper_1902_03317_b200", "host", "dropin_bench"), d, name,
                        steps, "1"], capture_output=True, text=True)
    print(r.stdout[-2000:], r.stderr[-6000:])
finally:
    shutil.rmtree(d, ignore_errors=True)
