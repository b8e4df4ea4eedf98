"""Per-op DRAM traffic from an ncu launch list of `bench.py --workload W`:
the bench flushes L2 (l2_flush_kernel) before every op, so the kernels between
two flushes belong to one op; ops repeat in wl.ops order (warmup + steps)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from parse_launches import load

def main(w, rnd=os.environ.get("SPT_ROUND", "r02")):
    L = load(f"gpurun_out/launches_{w}.csv")
    plain = json.loads(open(f"gpurun_out/plain_{w}.json").read().strip().splitlines()[-1])
    names = list(plain["ops"].keys())
    first = next(i for i, x in enumerate(L) if x[1] == "l2_flush_kernel")
    segs, cur = [], None
    for x in L[first:]:
        if x[1] == "l2_flush_kernel":
            cur = []
            segs.append(cur)
        elif not x[1].startswith("at::"):
            cur.append(x)
    per = {n: [] for n in names}
    for k, s in enumerate(segs):
        n = names[k % len(names)]
        per[n].append((sum(t for _, _, t, _, _ in s), sum(r + wb for _, _, _, r, wb in s),
                       [x[1] for x in s]))
    out = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per op call (all of the op's "
                   "kernels, mean over the bench's warmup+timed calls) from "
                   f"profiles/{rnd}_launches_{w}.csv (ncu --metrics ... --clock-control none, "
                   "cold L2: the bench flushes before every op)"}
    out["mttkrp_impl"] = plain.get("config", {}).get("mttkrp", "seg")
    out["source"] = f"profiles/{rnd}_launches_{w}.csv"
    for n, v in per.items():
        if v:
            out[n] = int(sum(b for _, b, _ in v) / len(v))
            out[n + "_kernels"] = v[-1][2]
            out[n + "_ncu_us"] = round(sum(t for t, _, _ in v) / len(v), 1)
    json.dump(out, open(f"profiles/traffic_{w}.json", "w"), indent=1)
    with open(f"profiles/{rnd}_launches_{w}.csv", "w") as f:
        f.write("id,kernel,gpu_time_us,dram_read_MB,dram_write_MB\n")
        for i, s, t, r, wb in L:
            f.write(f'{i},"{s}",{t:.2f},{r/1e6:.3f},{wb/1e6:.3f}\n')
    print(w, {n: out.get(n) for n in names})

for w in sys.argv[1:]:
    main(w)
