"""Key metrics of every kernel in an ncu --set full report (ncu -i ... --page raw --csv):
duration, DMMA / FP64 pipe activity, DRAM bytes, occupancy limits, registers,
shared-memory bank conflicts and the PC-sampling stall reasons.
usage: python tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_src_fp64.min.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {name[:160]}")
        for k in KEYS:
            if k in h:
                print(f"  {k} = {r[h.index(k)]} {units[h.index(k)]}")
        stalls = [(n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i] or 0)) for i, n in enumerate(h)
                  if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        top = sorted(stalls, key=lambda x: -x[1])[:8]
        print("  stall samples: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for n, v in top))


if __name__ == "__main__":
    main()
