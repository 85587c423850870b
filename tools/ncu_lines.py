"""Per-source-line stall-sample totals from an ncu report (needs -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
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
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if r and r[0] not in ("", "Line No") and len(r) > i_s and r[0].isdigit():
        try:
            lines.append((int(r[i_s]), int(r[i_e]), int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for s, e, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}%  {e:>10}  L{ln:<4} {src}")
