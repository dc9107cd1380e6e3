"""Print the headline counters and the stall-reason ratios of every kernel in an .ncu-rep
(ncu --page raw --csv piped in):  ncu -i X.ncu-rep --page raw --csv | python tools/ncu_summary.py"""
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__cluster_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__cycles_active.avg",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__warps_active.avg.per_cycle_active"]
for vals in rows[2:]:
    print("----")
    for h, u, v in zip(hdr, rows[1], vals):
        if h in want:
            print(h, v, u)
        elif h.endswith("_per_issue_active.ratio"):
            try:
                if float(v) >= 0.3:
                    print(h, v)
            except ValueError:
                pass
