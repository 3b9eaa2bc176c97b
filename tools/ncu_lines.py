"""Aggregate an ncu report's per-instruction data per CUDA source line
(development tool): share of warp-stall samples, share of executed warp
instructions, shared-memory wavefronts and global sectors.

    python tools/ncu_lines.py report.ncu-rep KERNEL_REGEX [TOP] [samples|inst]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
order = sys.argv[4] if len(sys.argv) > 4 else "samples"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0, 0, 0])   # samples, inst, smem wavefronts, global sectors
src_of = {}
cur_file = None
hdr = None
col = {}
first = True
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        if hdr is not None and cur_file is None:
            break   # one kernel instance is enough
        hdr = r
        col = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        def num(name):
            try:
                return int(float(r[col[name]]))
            except (KeyError, ValueError):
                return 0
        key = (cur_file, int(r[0]))
        a = agg[key]
        a[0] += num("# Samples")
        a[1] += num("Instructions Executed")
        a[2] += num("L1 Wavefronts Shared")
        a[3] += num("L2 Theoretical Sectors Global")
        src_of[key] = r[1].strip()
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
tw = sum(a[2] for a in agg.values()) or 1
tg = sum(a[3] for a in agg.values()) or 1
print(f"total: samples {ts}  warp-inst {ti}  smem wavefronts {tw}  global sectors {tg}")
print("samples%  inst%  smem%  glob%  line")
k = 0 if order == "samples" else 1
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][k])[:top]:
    f, ln = key
    print(f"{100*a[0]/ts:6.1f} {100*a[1]/ti:6.1f} {100*a[2]/tw:6.1f} {100*a[3]/tg:6.1f}  {f}:{ln}  {src_of[key][:80]}")
