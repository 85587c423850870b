"""Per-source-line shared-memory wavefronts (ideal vs excessive) from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
print("columns:", [h for h in hdr if "Shared" in h or "Wavefront" in h])
cols = [h for h in hdr if ("Shared" in h and ("Wavefronts" in h or "Excessive" in h or "Ideal" in h))]
idx = [hdr.index(c) for c in cols]
lines = []
for r in rows:
    if r and r[0].isdigit() and len(r) > max(idx):
        vals = []
        for i in idx:
            try:
                vals.append(float(r[i] or 0))
            except ValueError:
                vals.append(0.0)
        lines.append((vals, int(r[0]), r[1].strip()[:80]))
print(cols)
key = 1
for vals, ln, src in sorted(lines, key=lambda x: -x[0][key])[:top]:
    print("  ".join(f"{v:12.0f}" for v in vals), f" L{ln:<4} {src}")
