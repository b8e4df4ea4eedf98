"""Reuse statistics of the MTTKRP inputs (C4, C5): for every output mode n and
every choice of the second sort key a, the number of distinct (i_n, i_a)
prefixes (one middle-level factor gather each in a CSF-style traversal), and
how much of the leaf gathers the K most frequent ids of each mode cover (what
a shared-memory hot-row cache of K rows would serve).

    python tune/probe_reuse.py [c5|c4] [scale]
"""
import itertools
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import generate, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
c = generate.CONFIGS[name]
N = len(c["dims"])
nnz = int(c["nnz"] * scale)
t0 = time.time()
base = generate.coo(c["dims"], nnz, 20190210, c["zipf"], 0.0, 1.0, None, 0)
torch.cuda.synchronize()
out = {"config": name, "nnz": nnz, "gen_s": round(time.time() - t0, 2)}
Ks = [256, 512, 1024, 1536, 2048, 4096, 16384, 262144, 1 << 20]
cover = {}
for d in range(N):
    cnt = torch.bincount(base.indices[d].long(), minlength=c["dims"][d])
    s, _ = torch.sort(cnt, descending=True)
    cs = torch.cumsum(s, 0).double() / nnz
    cover[d] = {K: round(float(cs[min(K, len(cs)) - 1]), 4) for K in Ks}
    cover[d]["nonempty"] = int((cnt > 0).sum())
    cover[d]["max"] = int(s[0])
out["id_cover_topK"] = cover
pairs = {}
for n in range(N):
    others = [d for d in range(N) if d != n]
    for a in others:
        rest = [d for d in others if d != a]
        xs = base.clone()
        t1 = time.time()
        ops.sort_lexicographic(xs, [n, a] + rest)
        torch.cuda.synchronize()
        sort_s = time.time() - t1
        i_n, i_a = xs.indices[n], xs.indices[a]
        newp = torch.ones(nnz, dtype=torch.bool, device=i_n.device)
        newp[1:] = (i_n[1:] != i_n[:-1]) | (i_a[1:] != i_a[:-1])
        D = int(newp.sum())
        rec = {"sort_s": round(sort_s, 3), "distinct_pairs": D, "pair_frac": round(D / nnz, 4)}
        # hot-id coverage of the middle level (one gather per distinct pair)
        ia = i_a[newp].long()
        cnt = torch.bincount(ia, minlength=c["dims"][a])
        s, _ = torch.sort(cnt, descending=True)
        cs = torch.cumsum(s, 0).double() / max(D, 1)
        rec["mid_cover_topK"] = {K: round(float(cs[min(K, len(cs)) - 1]), 4) for K in Ks}
        if len(rest) >= 2:
            b = rest[0]
            i_b = xs.indices[b]
            newt = newp.clone()
            newt[1:] |= i_b[1:] != i_b[:-1]
            rec["distinct_triples"] = int(newt.sum())
        rows = torch.ones(nnz, dtype=torch.bool, device=i_n.device)
        rows[1:] = i_n[1:] != i_n[:-1]
        rec["rows"] = int(rows.sum())
        pairs[f"n{n}_a{a}"] = rec
        print(json.dumps({f"n{n}_a{a}": rec}), flush=True)
        del xs, newp, ia, cnt, s, cs, rows
        torch.cuda.empty_cache()
out["pairs"] = pairs
print(json.dumps(out))
