"""Key metrics of one kernel from `ncu -i REP --page raw --csv` on stdin:
duration, DRAM bytes, L1/L2/DRAM throughput, LSU writeback, FP64/DMMA pipes,
occupancy, registers, and the top warp-stall reasons.  Development tool."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]


def main():
    rows = list(csv.reader(sys.stdin))
    if len(rows) < 3:
        print("no data")
        return
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    print("kernel:", d.get("Kernel Name", ("?", ""))[0][:100])
    for k in KEYS:
        if k in d:
            print(f"{k} = {d[k][0]} {d[k][1]}")
    st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
           float(v or 0)) for h, (v, u) in d.items()
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
    st.sort(key=lambda x: -x[1])
    print("stalls per issue:", ", ".join(f"{n} {v:.2f}" for n, v in st[:8]))


if __name__ == "__main__":
    main()
