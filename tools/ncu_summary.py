"""Summarise an `ncu --page raw --csv` export of our kernel launches (dev tool).

    python tools/ncu_summary.py gpurun_out/ncu_C5/raw.csv C5 "<command>" > profiles/r02/ncu_C5/summary.json

One launch (the persistent executor): its metrics.  Several launches (the small-block
engine's kernels of one step): per-launch rows plus totals -- durations and DRAM bytes
summed, percentages averaged weighted by duration.  Records the library source sha
(bench.src_sha) so bench.py only reports `traffic` from a capture of the build it times.
"""
import csv
import json
import os
import sys

METRICS = {
    "gpu__time_duration.sum": "gpu__time_duration",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "sm__ops_path_tensor_src_fp64.sum": "sm__ops_path_tensor_src_fp64_sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "lts_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
OURS = ("serinv_exec", "sb_factor", "sb_inverse", "sb_pre")


def row_metrics(names, units, data):
    out = {}
    for m, key in METRICS.items():
        if m not in names:
            continue
        j = names.index(m)
        u = units[j]
        try:
            v = float(data[j].replace(",", ""))
        except ValueError:
            continue
        if key == "gpu__time_duration":
            out["gpu__time_duration_ms"] = v * SCALE.get(u, 1.0)
        elif key.startswith("dram_bytes"):
            out[key] = v * SCALE.get(u, 1.0)
        else:
            out[key] = v
    if "dram_bytes_read" in out and "dram_bytes_write" in out:
        out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    return out


def main(path, config, command):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import src_sha
    with open(path) as f:
        rows = [r for r in csv.reader(f) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[head], rows[head + 1]
    kcol = names.index("Kernel Name")
    data = [r for r in rows[head + 2:] if any(k in r[kcol] for k in OURS)]
    per = []
    for r in data:
        m = row_metrics(names, units, r)
        m["kernel"] = r[kcol].split("(")[0]
        per.append(m)
    out = {"config": config, "command": command, "src_sha": src_sha(), "launches": len(per),
           "units_raw": {m: units[names.index(m)] for m in METRICS if m in names}}
    if len(per) == 1:
        out.update(per[0])
    else:
        tot_t = sum(p.get("gpu__time_duration_ms", 0.0) for p in per)
        out["kernel"] = "+".join(sorted({p["kernel"] for p in per}))
        out["gpu__time_duration_ms"] = tot_t
        for k in ("dram_bytes_read", "dram_bytes_write", "dram_bytes_per_launch", "sm__ops_path_tensor_src_fp64_sum"):
            out[k] = sum(p.get(k, 0.0) for p in per)
        out["dram_bytes_per_step"] = out["dram_bytes_per_launch"]
        for k in ("dmma_pipe_active_pct", "fp64_pipe_active_pct", "l2_hit_rate_pct", "lts_throughput_pct",
                  "dram_throughput_pct", "warps_active_pct", "issue_active_pct"):
            if tot_t > 0:
                out[k] = sum(p.get(k, 0.0) * p.get("gpu__time_duration_ms", 0.0) for p in per) / tot_t
        out["per_launch"] = per
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
