"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel:
python scripts/launch_summary.py launches.csv "command line" > profiles/....txt"""
import collections
import csv
import sys

tot = collections.defaultdict(float)
cnt = collections.Counter()
with open(sys.argv[1]) as fh:
    for r in csv.DictReader(l for l in fh if l.startswith('"')):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        tot[r["Kernel Name"]] += v / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        cnt[r["Kernel Name"]] += 1
s = sum(tot.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("(cold-cache, serialised launches under the profiler: compare SHARES, not absolute times)")
print("%-76s %2s %12s %7s" % ("kernel", "n", "total_us", "share"))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("%-76s %2d %12.1f %7.4f" % (k[:76], cnt[k], v, v / s))
