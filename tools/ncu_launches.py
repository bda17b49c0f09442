"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X.csv)
into a markdown table of per-kernel launches / total time / share.
usage: python tools/ncu_launches.py X.csv OUT.md "title" """
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(r for r in rows if "Kernel Name" in r)
i_name, i_metric, i_val = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
i_unit = h.index("Metric Unit")
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[rows.index(h) + 1:]:
    if len(r) <= i_val or r[i_metric] != "gpu__time_duration.sum":
        continue
    v = float(r[i_val].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[i_unit], 1.0)
    k = r[i_name][:70]
    tot[k] = tot.get(k, 0.0) + v * scale
    cnt[k] += 1
s = sum(tot.values())
out = [f"## {sys.argv[3]}", "", "Cold-cache serialised times: compare shares, not absolutes.", "",
       "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    out.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / s:.1f}% |")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out[:12]))
