"""Per-source-line instruction and stall-sample shares from `ncu --page source --csv
--print-source cuda,sass` (rows: line, source, address, sass, metrics...)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
inst, stall, text = collections.Counter(), collections.Counter(), {}
hdr = None
for r in rows:
    if r[:2] == ["Line No", "Source"]:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    line = int(r[0])
    text[line] = r[1].strip()[:110]
    try:
        inst[line] += float(r[hdr.index("Instructions Executed")].replace(",", "") or 0)
        stall[line] += float(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
    except ValueError:
        pass
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"instructions {ti:.0f}")
for line, v in sorted(stall.items(), key=lambda x: -x[1])[:top]:
    print(f"line {line:5d}  stall {v / ts * 100:5.1f}%  inst {inst[line] / ti * 100:5.1f}%  {text.get(line, '')}")
