"""Per-source-line warp-stall breakdown from an ncu report (needs -lineinfo).
usage: python tools/ncu_stalls.py report.ncu-rep [N] [file-filter] [line-lo line-hi]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
filt = sys.argv[3] if len(sys.argv) > 3 else ""
lo = int(sys.argv[4]) if len(sys.argv) > 4 else 0
hi = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        ln = int(r[0])
        if filt and filt not in cur:
            continue
        if not (lo <= ln <= hi):
            continue
        st = {k[6:]: int(v or 0) for k, v in d.items()
              if k.startswith("stall_") and "Not Issued" not in k and (v or "0").isdigit()}
        agg.append((samples, cur, ln, r[1].strip()[:70], st))
tot = sum(a[0] for a in agg) or 1
print(f"total samples {tot}")
for s, f, ln, src, st in sorted(agg, key=lambda a: -a[0])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    br = " ".join(f"{k}={100 * v / max(s, 1):.0f}%" for k, v in top if v)
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src:70s} | {br}")
