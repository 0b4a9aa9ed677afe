"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel total time and share.  python scripts/launch_list.py LIST.csv [title]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    ms = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1e-6)
    agg[r[ix["Kernel Name"]][:90]].append(ms)
tot = sum(sum(v) for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("total kernel time %.3f ms over %d launches" % (tot, sum(len(v) for v in agg.values())))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print("%6.1f%%  %10.3f ms  n=%4d  %s" % (100 * sum(v) / tot, sum(v), len(v), k))
