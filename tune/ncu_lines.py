"""Per-source-line stall samples and executed instructions of an ncu report (--import-source)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; key = ("?", "?", "?"); st = {}; ins = {}
for r in rows:
    if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if len(r) > 7 and r[0] != 'Line No':
        try: s = int(r[4] or 0); n = int(r[7] or 0)
        except ValueError: continue
        if r[0]: key = (cur, r[0], r[1].strip()[:90])
        st[key] = st.get(key, 0) + s; ins[key] = ins.get(key, 0) + n
ts = sum(st.values()) or 1; ti = sum(ins.values()) or 1
print(f"samples {ts} instructions {ti}")
for k, v in sorted(st.items(), key=lambda x: -x[1])[:top]:
    print(f"{100*v/ts:5.1f}% stall {100*ins[k]/ti:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
