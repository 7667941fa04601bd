"""Per-source-line instruction and stall shares of one kernel in an ncu report.
Usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]"""
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{pat}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, data = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "" and len(r) > 8:
        try:
            v, s = int(r[7]), int(r[4])
        except ValueError:
            continue
        data.append((v, s, fname, r[0], r[1][:100]))
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print(f"{pat}: {tot} warp instructions, {tots} stall samples")
for v, s, f, ln, sr in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {100 * s / tots:5.1f}% {f[:16]:16s}:{ln:>4s} {sr}")
