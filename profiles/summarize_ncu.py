"""Summarise an ncu report (--set full) into the text files committed under profiles/.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep "title / command" > profiles/rNN_x.txt
"""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("launch__registers_per_thread", "registers"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (regs)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(rep, title):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    print(f"# {title}")
    print(f"# source: {rep} (ncu --set full --clock-control none)")
    for r in rows[2:]:
        print(f"\n## {r[head.index('Kernel Name')]}")
        for m, label in METRICS:
            if m in head:
                i = head.index(m)
                print(f"{label:22s} {r[i]} {units[i]}")
        if "dram__bytes_read.sum" in head:
            rd = float(r[head.index("dram__bytes_read.sum")])
            wr = float(r[head.index("dram__bytes_write.sum")])
            u = units[head.index("dram__bytes_read.sum")]
            print(f"{'dram traffic':22s} {rd + wr:.6f} {u}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
