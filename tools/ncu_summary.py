"""Key metrics of the kernels in an ncu report (`ncu -i rep --page raw --csv`).

usage: python tools/ncu_summary.py report.ncu-rep
Prints, per captured launch: duration, grid/block, registers, pipe
utilisation (FP64, tensor, shared FP64/tensor datapath, FMA), issue
activity, occupancy, DRAM bytes, and the warp-stall breakdown (cycles per
issued instruction).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("Kernel Name", d.get("Kernel Name", "?")[:160])
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]} {u.get(k, '')}")
        stalls = [(k[len(STALL):].replace("_per_issue_active.ratio", ""), float(d[k] or 0))
                  for k in hdr if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")]
        stalls = [s for s in stalls if s[1] >= 0.05]
        if stalls:
            print("warp stall reasons (cycles per issued instruction):")
            for name, v in sorted(stalls):
                print(f"  {name:28s} {v:.3f}")
        print()


if __name__ == "__main__":
    main()
