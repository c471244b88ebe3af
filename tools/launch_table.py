"""Summarise an `ncu --metrics ... --csv --log-file` launch list: one line per launch."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[iid], {"k": r[ik].split("(")[0][:44]})[r[im]] = r[iv]
skip = sys.argv[2].split(",") if len(sys.argv) > 2 else []
for k, v in d.items():
    if any(s in v["k"] for s in skip if s):
        continue
    print(k, v["k"].ljust(44), " ".join(f"{m.split('__')[1].split('.')[0][:14]}={v[m]}" for m in v if m != "k"))
