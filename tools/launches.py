"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (dev tool)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ik].split("(")[0][-44:]
    agg[k][0] += 1
    agg[k][1] += float(r[iv]) / 1000
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("| `%s` | %d | %.1f | %.1f%% | %.2f |" % (k.strip(), v[0], v[1], 100 * v[1] / tot, v[1] / v[0]))
