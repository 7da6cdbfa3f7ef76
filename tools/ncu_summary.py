"""Summarise an `ncu --page raw --csv` export of the executor launch (dev tool).

    python tools/ncu_summary.py gpurun_out/ncu_C5/raw.csv C5 "<command>" > profiles/r01/ncu_C5/summary.json

Picks the metrics the bench's roofline.traffic and profiles/ncu_r01_summary.md use
(dram bytes, DMMA / FP64 pipe activity, L2, issue) from the first serinv_exec row.
"""
import csv
import json
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
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path, config, command):
    with open(path) as f:
        rows = [r for r in csv.reader(f) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[head], rows[head + 1]
    data = next(r for r in rows[head + 2:] if any("serinv_exec" in c for c in r))
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
    from bench import src_sha
    out = {"config": config, "kernel": "serinv_exec_kernel", "command": command, "src_sha": src_sha(),
           "units_raw": {}}
    for m, key in METRICS.items():
        if m not in names:
            continue
        j = names.index(m)
        u = units[j]
        try:
            v = float(data[j].replace(",", ""))
        except ValueError:
            continue
        out["units_raw"][m] = u
        if key == "gpu__time_duration":
            out["gpu__time_duration_ms"] = v * SCALE.get(u, 1.0)
        elif key.startswith("dram_bytes"):
            out[key] = v * SCALE.get(u, 1.0)
        else:
            out[key] = v
    if "dram_bytes_read" in out and "dram_bytes_write" in out:
        out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
