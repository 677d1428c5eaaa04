"""Summarise an ncu --csv launch list: total device time and share per kernel name."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"])[:60]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    tot[name] += v * scale
    cnt[name] += 1
S = sum(tot.values())
print(f"total {S:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us  {100*v/S:5.1f}%  n={cnt[k]:5d}  avg={v/cnt[k]:8.2f} us  {k}")
