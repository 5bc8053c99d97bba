"""Print per-launch metrics from an `ncu --csv --log-file` metrics capture."""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
i_id, i_m, i_v, i_k = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
d = defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) > i_v:
        d[r[i_id]][r[i_m]] = r[i_v]
        names[r[i_id]] = r[i_k][:40]
for k, v in d.items():
    print(k, names[k], {m.split(".")[0][-24:]: val for m, val in v.items()})
