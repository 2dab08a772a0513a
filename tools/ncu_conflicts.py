"""Top source lines by excessive shared-memory wavefronts (bank conflicts)
from an ncu report captured with --import-source.  Development aid."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for line in out.splitlines():
    if line.startswith('"File Path"') or line.startswith('"File Name"'):
        fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]
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
        ex = int(float(d.get("L1 Wavefronts Shared Excessive", "0") or 0))
        tot = int(float(d.get("L1 Wavefronts Shared", "0") or 0))
    except ValueError:
        continue
    rows.append((ex, tot, fname, int(r[0]), r[1].strip()[:100]))
print("excessive total", sum(r[0] for r in rows), "of", sum(r[1] for r in rows))
for r in sorted(rows, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{r[0]:10d} / {r[1]:10d}  {r[2]}:{r[3]:4d} {r[4]}")
