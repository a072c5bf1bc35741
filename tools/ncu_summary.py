"""Summarise ncu reports into profiles/: per-kernel duration, DRAM bytes, throughput, issue, occupancy."""
import csv, io, json, subprocess, sys
KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__inst_executed.sum": "warp_inst", "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct", "launch__registers_per_thread": "regs",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "smsp__inst_executed.avg.per_cycle_active": "ipc_smsp"}
def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, name in KEYS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                u = units[hdr.index(k)]
                try: v = float(v)
                except ValueError: continue
                scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                         "byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9,
                         "GB": 1e9}.get(u, 1)
                if name == "duration": d["duration_ms"] = v * scale
                elif name in ("dram_read", "dram_write"): d[name + "_bytes"] = v * scale
                else: d[name] = v
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0)
            if d.get("duration_ms"): d["dram_gbs"] = d["dram_bytes"] / d["duration_ms"] / 1e6
        res.append(d)
    return res
if __name__ == "__main__":
    allr = {}
    for rep in sys.argv[1:]:
        allr[rep.split("/")[-1]] = summarise(rep)
    print(json.dumps(allr, indent=1))
