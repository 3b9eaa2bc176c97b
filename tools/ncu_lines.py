"""Aggregate ncu warp-stall samples per CUDA source line (development tool)."""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
agg = collections.Counter(); src_of = {}
cur_file = None
i = 0
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            s = int(r[4])
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        agg[key] += s
        src_of[key] = r[1].strip()
tot = sum(agg.values()) or 1
for (f, ln), s in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{100*s/tot:5.1f}%  {f}:{ln}  {src_of[(f, ln)][:90]}")
