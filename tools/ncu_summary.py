"""Summarise an ncu report (raw page) into the metrics DESIGN.md/profiles cite."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_barrier", "sm__cycles_elapsed.avg.per_second"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"# kernel: {name[:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:70s} {v[i]:>20s} {units[i]}")
        stalls = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h[i].endswith("_not_issued")]
        tot = sum(float(x.replace(",", "") or 0) for _, x in stalls)
        top = sorted(stalls, key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
        print("# top stall reasons (pc samples):")
        for n_, x in top:
            print(f"  {n_.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * float(x.replace(',', '')) / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
