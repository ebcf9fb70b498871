"""Summarise an ncu report (raw page) for the metrics this project tracks."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__waves_per_multiprocessor", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(path, kernel_filter=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        if kernel_filter and kernel_filter not in name:
            continue
        print(name[:100])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:70s} {v[i]:>16s} {units[i]}")
        stalls = [(h[i], float(v[i])) for i in range(len(h))
                  if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")
                  and v[i] not in ("", "n/a")]
        stalls.sort(key=lambda t: -t[1])
        print("  stalls/issue:", ", ".join(f"{n[34:-23]}={x:.2f}" for n, x in stalls[:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
