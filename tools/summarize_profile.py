"""Copy a gpu_bench_profile.sh run (gpurun_out/<tag>/) into profiles/:
bench line, ncu summary of k_solve, DRAM traffic per launch, launch list,
source hotspots.   usage: python tools/summarize_profile.py <tag> [round prefix, r02]

profiles/lift_traffic.json is stamped with the digest of the library sources
the capture ran (gpurun_out/<tag>/source_digest.txt, bench.source_digest(),
written by gpu_bench_profile.sh) and the .so's SHA-256: bench.py reports it as
`roofline.traffic` only while the sources match, so a stale capture is never
paired with a newer kernel."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]
RND = sys.argv[2] if len(sys.argv) > 2 else "r02"
src = os.path.join("gpurun_out", tag)
dst = "profiles"
shutil.copy(os.path.join(src, "bench.json"), os.path.join(dst, f"{RND}_bench_{tag.split('_')[-1]}.json"))
rep = os.path.join(src, "solve_c4.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, r = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sector_op_read_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
out = {k: (r[h.index(k)], units[h.index(k)]) for k in keys if k in h}
vals = []
for i, k in enumerate(h):
    if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
        try:
            vals.append((float(r[i].replace(",", "")), k))
        except ValueError:
            pass
tot = sum(v for v, _ in vals) or 1
out["stall_breakdown_pct"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * v / tot, 1)
                              for v, k in sorted(vals, reverse=True)[:8]}
json.dump(out, open(os.path.join(dst, f"{RND}_{tag.split('_')[-1]}_ncu_k_solve.json"), "w"), indent=1)
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
rd = float(out["dram__bytes_read.sum"][0].replace(",", "")) * scale[out["dram__bytes_read.sum"][1]]
wr = float(out["dram__bytes_write.sum"][0].replace(",", "")) * scale[out["dram__bytes_write.sum"][1]]
shafile = os.path.join(src, "lib_sha256.txt")
lib_sha = open(shafile).read().split()[0] if os.path.exists(shafile) else None
digfile = os.path.join(src, "source_digest.txt")
src_digest = open(digfile).read().split()[0] if os.path.exists(digfile) else None
json.dump({"kernel": "k_solve", "bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "lib_sha256": lib_sha, "source_digest": src_digest,
           "source": f"ncu --set full --clock-control none -k regex:k_solve -c 1 "
                     f"python tools/ncu_target.py C4 1 ({tag})"},
          open(os.path.join(dst, "lift_traffic.json"), "w"), indent=1)
hot = subprocess.run([sys.executable, "tools/ncu_stalls.py", rep, "40"], capture_output=True,
                     text=True).stdout
open(os.path.join(dst, f"{RND}_{tag.split('_')[-1]}_source_hotspots.txt"), "w").write(
    "# warp-stall samples per source line, top stall reasons (tools/ncu_stalls.py)\n" + hot)
# C3 (R-MAT) capture: the same summary keys
rep3 = os.path.join(src, "solve_c3.ncu-rep")
if os.path.exists(rep3):
    raw3 = subprocess.run(["ncu", "-i", rep3, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout
    rows3 = list(csv.reader(io.StringIO(raw3)))
    h3, u3, r3 = rows3[0], rows3[1], rows3[2]
    json.dump({k: (r3[h3.index(k)], u3[h3.index(k)]) for k in keys if k in h3},
              open(os.path.join(dst, f"{RND}_{tag.split('_')[-1]}_ncu_k_solve_c3.json"), "w"), indent=1)
for extra in ("bench_2rank_staged.json",):
    if os.path.exists(os.path.join(src, extra)) and os.path.getsize(os.path.join(src, extra)):
        shutil.copy(os.path.join(src, extra),
                    os.path.join(dst, f"{RND}_{tag.split('_')[-1]}_{extra}"))
lrows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
hdr = next(i for i, x in enumerate(lrows) if x and x[0] == "ID")
hh, data = lrows[hdr], lrows[hdr + 1:]
ki, vi = hh.index("Kernel Name"), hh.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for x in data:
    nm = x[ki].split("(")[0][:70]
    agg[nm][0] += 1
    agg[nm][1] += float(x[vi].replace(",", ""))
t = sum(v[1] for v in agg.values())
with open(os.path.join(dst, f"{RND}_{tag.split('_')[-1]}_launches.txt"), "w") as fh:
    fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none python tools/ncu_target.py C4 1\n")
    fh.write("# (context create = pipelined upload + device build, one solve, export); cold-cache, serialised\n")
    for k, v in sorted(agg.items(), key=lambda z: -z[1][1]):
        fh.write(f"{k:70s} {v[0]:4d} {v[1] / 1e6:9.3f} ms {100 * v[1] / t:5.1f}%\n")
print(json.dumps(out, indent=1))
