"""Build profiles/ncu_summary.json from `ncu --page raw --csv` exports of the
config-3 and config-4 residual captures and the bench command's launch list
(development tool; the exports are produced on the GPU box).

    python tools/make_ncu_summary.py cfg3_raw.csv cfg4_raw.csv launches.csv out.json "source text"
"""
import csv, collections, io, json, sys

WANT = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ_lim_blocks": "launch__occupancy_limit_registers",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def strip_args(name):
    """Kernel name without its parameter list (template args may hold '(')."""
    gt = name.rfind(">")
    cut = name.find("(", gt if gt >= 0 else 0)
    return name[:cut] if cut >= 0 else name


def short(name):
    base = name.split("(")[0].replace("void ", "").replace("tdg::", "").strip()
    tmpl = name[name.find("<") + 1: name.find(">")] if "<" in name else ""
    args = [a.strip() for a in tmpl.split(",")]
    if base.startswith("k_vol_lift"):
        return "vol_lift"
    if base.startswith("k_vol_flux"):
        return "vol_flux"
    if base.startswith("k_trace_q"):
        return "trace_q"
    if base.startswith("k_face"):
        return "face_flux" if args[-1] == "1" else "face_lift"
    if base.startswith("k_mortar"):
        return "mortar_flux" if args[-1] in ("1", "true") else "mortar_lift"
    return base


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        d = {"kernel": strip_args(name)}
        for k, m in WANT.items():
            if m not in hdr:
                continue
            v = r[hdr.index(m)].replace(",", "")
            try:
                d[k] = float(v) * SCALE.get(units[hdr.index(m)], 1)
            except ValueError:
                pass
        key = short(name)
        e = {"dram_bytes_per_launch": d.get("dram_rd", 0) + d.get("dram_wr", 0),
             "dram_read": d.get("dram_rd"), "dram_write": d.get("dram_wr"),
             "dram_pct_of_peak": d.get("dram_pct"), "warps_active_pct": d.get("warps_active_pct"),
             "registers": d.get("regs"), "occupancy_limit_blocks": d.get("occ_lim_blocks"),
             "time_ms_under_ncu": d.get("time_us", 0) / 1e3, "fp64_pipe_pct": d.get("fp64_pct"),
             "l1_pct": d.get("l1_pct"), "ncu_kernel": d["kernel"]}
        out.setdefault(key, e)
    return out


def launches(path):
    agg = collections.defaultdict(lambda: [0.0, 0])
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    for r in rows[1:]:
        if len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = strip_args(r[hdr.index("Kernel Name")])
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}[unit]
        agg[name][0] += v
        agg[name][1] += 1
    return {k: {"total_ns": v[0], "launches": v[1]} for k, v in sorted(agg.items(), key=lambda x: -x[1][0])}


if __name__ == "__main__":
    c3, c4, ll, out, src = sys.argv[1:6]
    rnd = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    res = {"round": rnd, "source": src, "kernels": raw(c3), "cfg4_kernels": raw(c4),
           "launch_list_ns_by_kernel": launches(ll)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in res["kernels"].items()}))
