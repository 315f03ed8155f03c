"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list into per-kernel shares."""
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
unit_ns = 1.0 if len(sys.argv) < 3 else float(sys.argv[2])
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / s:6.2f}%  launches={cnt[k]:5d}  avg_ns={unit_ns * v / cnt[k]:12.1f}  {k}")
