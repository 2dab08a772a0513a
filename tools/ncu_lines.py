"""Per-source-line warp-stall samples from an ncu report (--import-source,
-lineinfo): top lines and totals per file.  Development aid."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for line in out.splitlines():
    if line.startswith('"File Path"') or line.startswith('"File Name"'):
        fname = next(csv.reader(io.StringIO(line)))[1]
        hdr = None
        continue
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        s = 0
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    rows.append((s, fname.split("/")[-1], int(r[0]), r[1].strip()[:90], stalls))
tot = sum(r[0] for r in rows)
print(f"total samples {tot}")
byfile = {}
for r in rows:
    byfile[r[1]] = byfile.get(r[1], 0) + r[0]
print(byfile)
if len(sys.argv) > 3:  # ranges file:lo-hi,...
    for spec in sys.argv[3].split(","):
        f, rg = spec.split(":")
        lo, hi = map(int, rg.split("-"))
        s = sum(r[0] for r in rows if r[1] == f and lo <= r[2] <= hi)
        print(f"{spec}: {s} ({100.0*s/tot:.1f}%)")
for r in sorted(rows, reverse=True)[:top]:
    st = sorted(r[4].items(), key=lambda kv: -kv[1])[:3]
    print(f"{r[0]:7d} {100.0*r[0]/tot:5.1f}% {r[1]}:{r[2]:4d} {r[3]:90s} {st}")
