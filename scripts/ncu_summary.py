"""Summarise an ncu --set full capture (raw page CSV) into profiles/ncu_summary.json: per kernel
family, duration and DRAM bytes (read + write) per launch, achieved DRAM GB/s and key
utilisations.  Usage: ncu -i rep --page raw --csv > raw.csv; python scripts/ncu_summary.py raw.csv out.json"""
import csv, json, sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "usecond": 1e-6,
        "msecond": 1e-3, "nsecond": 1e-9}
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}


def val(d, name):
    i = idx.get(name)
    if i is None or d[i] in ("", "n/a"):
        return None
    v = float(d[i].replace(",", ""))
    return v * UNIT.get(units[i], 1.0)


def family(name):
    if "row_solve_kernel" in name:
        return "row_solve"
    if "prop1_kernel" in name or "prop2_kernel" in name:
        return "gram_propagation_" + ("1" if "prop1" in name else "2")
    if "reduce_incr_kernel" in name:
        return "reduce"
    if "incr_tc_kernel" in name:
        return "increments"
    if "incr_kernel" in name:
        return "increments_cuda_core"
    if "row_pass_tc_kernel" in name or "row_pass_kernel" in name:
        return "row_pass"
    if "small_step_kernel" in name:
        return "small_step" if ", 1>" in name else "deferred_small_step"
    return None


out = {}
for d in rows[2:]:
    name = d[idx["Kernel Name"]]
    key = family(name)
    if key is None or key in out:
        continue
    dur = val(d, "gpu__time_duration.sum")
    rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
    out[key] = {"kernel": name, "duration_us": dur * 1e6 if dur else None,
                "dram_bytes_per_launch": (rd or 0) + (wr or 0), "dram_read": rd, "dram_write": wr,
                "dram_gbs": ((rd or 0) + (wr or 0)) / dur / 1e9 if dur else None,
                "grid": val(d, "launch__grid_size"),
                "sm_throughput_pct": val(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                "dram_throughput_pct": val(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                "warps_active_pct": val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                "note": "ncu --set full --clock-control none, caches flushed per replay (cold)"}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
