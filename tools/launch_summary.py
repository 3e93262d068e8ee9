"""Per-kernel time of the last product in an ncu launch list (--metrics
gpu__time_duration.sum --csv), aggregated by kernel template."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]
ki, vi = hd.index("Kernel Name"), hd.index("Metric Value")
ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[h + 1:] if len(r) > vi]
idx = [i for i, (k, v) in enumerate(ks) if "k_gather(" in k]
last = ks[idx[-1]:]
agg = OrderedDict()
for k, v in last:
    name = k.split("(")[0].replace("imqk::<unnamed>::", "").replace("void ", "")
    agg[name] = agg.get(name, 0) + v
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6:8.3f} ms  {k[:90]}")
print(f"total {sum(agg.values()) / 1e6:.3f} ms over {len(last)} launches")
