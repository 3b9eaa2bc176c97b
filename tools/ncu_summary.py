"""Summarise an ncu report (raw page) into a table / JSON (development tool)."""
import csv, io, json, subprocess, sys

WANT = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ_lim_regs": "launch__occupancy_limit_registers",
    "occ_lim_smem": "launch__occupancy_limit_shared_mem",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "inst": "smsp__inst_executed.sum",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}

def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, m in WANT.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    d[k] = float(v)
                except ValueError:
                    d[k] = v
        # ncu reports bytes in the unit of the column header row (rows[1])
        for k in ("dram_rd", "dram_wr"):
            unit = rows[1][hdr.index(WANT[k])]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[k] = d.get(k, 0) * scale
        tunit = rows[1][hdr.index(WANT["time_us"])]
        d["time_us"] = d["time_us"] * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(tunit, 1)
        res.append(d)
    return res

if __name__ == "__main__":
    res = load(sys.argv[1])
    cols = ["kernel", "time_us", "dram_rd", "dram_wr", "dram_pct", "warps_active_pct", "regs", "occ_lim_regs", "occ_lim_smem", "sm_pct", "fp64_pct", "l1_pct", "inst"]
    print(" | ".join(cols))
    for d in res:
        print(" | ".join(f"{d.get(c):.4g}" if isinstance(d.get(c), float) else str(d.get(c)) for c in cols))
    if len(sys.argv) > 2:
        json.dump(res, open(sys.argv[2], "w"), indent=1)
