"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:80]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / 1e3:10.1f} us  n={cnt[k]:4d}  avg={v / cnt[k] / 1e3:8.1f} us  {k}")
