"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
agg = collections.defaultdict(list)
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")[:48]
    agg[name].append(float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':50s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:6.3f}")
print(f"total {tot / 1e3:.1f} us over {sum(len(v) for v in agg.values())} launches")
