"""Per-source-line shared-memory wavefronts (and excessive = bank-conflict
wavefronts) of an ncu report captured with --import-source."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iw = hdr.index("L1 Wavefronts Shared"); ix = hdr.index("L1 Wavefronts Shared Excessive")
cur = None; key = ("?", "?", "?"); w = {}; x = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if len(r) > ix and r[0] != "Line No":
        try: a = int(r[iw] or 0); b = int(r[ix] or 0)
        except ValueError: continue
        if r[0]: key = (cur, r[0], r[1].strip()[:90])
        w[key] = w.get(key, 0) + a; x[key] = x.get(key, 0) + b
tw = sum(w.values()) or 1
print(f"shared wavefronts {tw} (excessive {sum(x.values())})")
for k, v in sorted(w.items(), key=lambda t: -t[1])[:top]:
    print(f"{100*v/tw:5.1f}% wf  {x[k]:>10d} excess  {k[0]}:{k[1]}  {k[2]}")
