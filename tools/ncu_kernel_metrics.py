"""Key ncu metrics of every kernel launch in a report, as text (for profiles/):
duration, instructions, issue / L1 / shared-memory figures, occupancy limits,
DRAM bytes and the stall reasons above 0.2 per issue.

    python tools/ncu_kernel_metrics.py gpurun_out/x.ncu-rep [kernel-substring] > profiles/r02/x.txt
"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__waves_per_multiprocessor", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, sub=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if sub and sub not in name:
            continue
        print(name[:100])
        for m in WANT:
            if m in hdr:
                print(f"   {m} = {r[hdr.index(m)]} {units[hdr.index(m)]}")
        for i, h in enumerate(hdr):
            if "issue_stalled" in h and "per_issue_active" in h:
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.2:
                    print(f"   stall {h.split('issue_stalled_')[1].split('_per')[0]} = {v:.3f} per issue")


if __name__ == "__main__":
    main(*sys.argv[1:])
