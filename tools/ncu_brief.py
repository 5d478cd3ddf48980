"""One-screen summary of an ncu report (first kernel): time, pipes, occupancy, memory, stalls."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {a: (c, b) for a, b, c in zip(h, u, v)}
    print("kernel:", d.get("Kernel Name", ("?",))[0])
    for k in WANT:
        if k in d:
            print(f"  {k:80s} {d[k][0]} {d[k][1]}")
    stalls = {a.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(c.replace(",", "") or 0)
              for a, (c, b) in d.items() if a.startswith("smsp__pcsamp_warps_issue_stalled_") and
              not a.endswith("not_issued")}
    tot = sum(stalls.values()) or 1
    print("  stall samples:", ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
