"""Summarise an ncu report (--set full) into the numbers DESIGN.md cites.

    python tools/ncu_summary.py gpurun_out/prof_streamcoll.ncu-rep [algorithmic_bytes]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
]


def summary(path, alg_bytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        units = dict(zip(h, u))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:62s} {d[k]:>16s} {units.get(k, '')}")
        try:
            rb = float(d["dram__bytes_read.sum"]) * (1e6 if units["dram__bytes_read.sum"] == "Mbyte" else 1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1)
            wb = float(d["dram__bytes_write.sum"]) * (1e6 if units["dram__bytes_write.sum"] == "Mbyte" else 1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1)
            t = float(d["gpu__time_duration.sum"]) * (1e-6 if units["gpu__time_duration.sum"] == "us" else 1e-3 if units["gpu__time_duration.sum"] == "ms" else 1e-9)
            out.append(f"  traffic (dram read+write) = {rb + wb:.4e} B; achieved {(rb + wb) / t / 1e9:.1f} GB/s under ncu")
            if alg_bytes:
                out.append(f"  algorithmic bytes = {alg_bytes:.4e} B; traffic/algorithmic = {(rb + wb) / alg_bytes:.3f}")
        except Exception:
            pass
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None))
