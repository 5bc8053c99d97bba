"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per kernel
launches, total device time and share (probe kernels listed separately)."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iN, iM, iU, iMN = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[iMN] != "gpu__time_duration.sum":
        continue
    v = float(r[iM].replace(",", ""))
    u = r[iU]
    v = v / 1000 if u in ("nsecond", "ns") else (v * 1000 if u in ("msecond", "ms") else v)
    agg[r[iN].split("(")[0].replace("void ", "")][0] += 1
    agg[r[iN].split("(")[0].replace("void ", "")][1] += v
work = {k: v for k, v in agg.items() if "probe" not in k and "FillFunctor" not in k}
tot = sum(v[1] for v in work.values())
print("%-58s %8s %12s %7s" % ("kernel (excluding probes / L2-flush fills)", "launches", "device us", "share"))
for k, (n, t) in sorted(work.items(), key=lambda kv: -kv[1][1]):
    print("%-58s %8d %12.1f %6.1f%%" % (k[:58], n, t, 100 * t / tot))
