import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
# may contain several kernels; take first block
r = list(csv.reader(lines[1:]))
h = r[0]
ci = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source")
rows = []
for x in r[1:]:
    if len(x) <= ci or x[0] == "Kernel Name": break
    try: rows.append((float(x[ci]), x[0], x[si]))
    except ValueError: pass
tot = sum(a for a, _, _ in rows)
print("total samples", tot, "instructions", len(rows))
idx = sorted(range(len(rows)), key=lambda i: -rows[i][0])[:n]
for i in sorted(idx):
    print(f"{i:5d} {100*rows[i][0]/tot:5.1f}% {rows[i][2].strip()[:90]}")
