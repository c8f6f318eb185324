"""Summarise an ncu report: per-kernel time, DRAM traffic, pipes, stalls."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")][:70])
        for w in WANT:
            if w in hdr:
                print(f"   {w:60s} {r[hdr.index(w)]:>16s} {units[hdr.index(w)]}")
        st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", "")))
              for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
              and not hdr[i].endswith("not_issued") and r[i]]
        tot = sum(v for _, v in st) or 1
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in
                                       sorted(st, key=lambda x: -x[1])[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
