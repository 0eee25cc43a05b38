"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 4 and r[0].isdigit():
        try:
            samples = int(r[4] or 0)
        except ValueError:
            continue
        agg.append((samples, cur_file, int(r[0]), r[1].strip()[:90]))
tot = sum(a[0] for a in agg) or 1
print(f"total samples {tot}")
for s, f, ln, src in sorted(agg, reverse=True)[:N]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src}")
