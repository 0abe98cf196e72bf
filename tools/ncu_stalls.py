"""Print the headline counters and warp-stall breakdown of each kernel in an ncu --page raw --csv dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
for v in rows[2:]:
    print("##", v[h.index("Kernel Name")][:90])
    for k in KEYS:
        if k in h:
            print(f"  {k:60s} {v[h.index(k)]} {u[h.index(k)]}")
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__average_warp_latency_issue_stalled_") or (
                x.startswith("smsp__warp_issue_stalled_") and x.endswith("_per_warp_active.pct")):
            try:
                st.append((float(v[i].replace(",", "")), x))
            except ValueError:
                pass
    for val, x in sorted(st, reverse=True)[:12]:
        print(f"  {x:60s} {val}")
