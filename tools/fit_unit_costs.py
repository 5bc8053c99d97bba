"""Fit the multi-GPU device-time model of parallel.py / mgpu.cu to tools/unit_costs.py output (CPU).

    python tools/fit_unit_costs.py profiles/r02/unit_costs_c5.json

Per frequency (half-width h = ceil(3 sigma)): cost(ms) = A + B1 * single + B2 * double over its contiguous
k-ranges, where a range holds `single` one-output directs (theta = 0, pi / 2) and `double` two-output ones;
least squares with A >= 0.  Prints the `_FIT` tuple for parallel.py (restated as kFit in csrc/mgpu.cu) and
the largest relative error over the measured ranges.
"""
import json
import math
import sys

import numpy as np

d = json.load(open(sys.argv[1]))
n = 16 if d["config"] == 5 else 8
nh = n // 2
fit, worst = [], 0.0
for f in sorted({r["freq"] for r in d["ranges"]}):
    rows = [r for r in d["ranges"] if r["freq"] == f]
    h = max(1, math.ceil(3.0 * rows[0]["sigma"]))
    X, y = [], []
    for r in rows:
        ks = range(r["k0"], r["k1"] + 1)
        single = sum(1 for k in ks if k in (0, nh))
        X.append([1.0, single, len(ks) - single])
        y.append(sum(r["prof"].values()))  # kernel time of the range (live profile; the per-call prep is not a unit cost)
    X, y = np.array(X), np.array(y)
    p = np.linalg.lstsq(X, y, rcond=None)[0]
    if p[0] < 0:  # no negative launch constant: refit through the origin
        p = np.concatenate([[0.0], np.linalg.lstsq(X[:, 1:], y, rcond=None)[0]])
    err = float(np.max(np.abs(X @ p - y) / y))
    worst = max(worst, err)
    fit.append((h, *[round(float(v), 4) for v in p]))
    print(f"sigma {rows[0]['sigma']:5.1f} h {h:3d}: A {p[0]:.4f} B1 {p[1]:.4f} B2 {p[2]:.4f}  max err {err:.3f}  "
          f"full frequency {y[[i for i, r in enumerate(rows) if r['k0'] == 0 and r['k1'] == nh][0]]:.3f} ms")
print("_FIT =", tuple(sorted(fit)))
print(f"max relative error over {len(d['ranges'])} ranges: {worst:.3f}")
