"""Measure device time of contiguous (frequency, direct k) unit ranges of a
bank config, split into the row and column launches by libfgb200's live
profile -- the data behind parallel.bank_unit_costs / partition_units.

    python tools/unit_costs.py [--config 5] > profiles/r02/unit_costs_c5.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_05231_b200 as fg  # noqa: E402
from paper_1704_05231_b200 import _native as N  # noqa: E402
from paper_1704_05231_b200.device import BankPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
img = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
nh = cfg["n"] // 2
rows = []
for i in range(len(cfg["freqs"])):
    for k0 in range(nh + 1):
        for k1 in range(k0, nh + 1):
            units = [i * (nh + 1) + k for k in range(k0, k1 + 1)]
            p = BankPlan(tuple(img.shape), spec, fg.ExactFIR(3.0), "f32", True, units)
            out = p.new_output("cuda")
            p(img, out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p(img, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            N.lib.fgb_profile_enable(1)
            N.profile_read()
            for _ in range(3):
                p(img, out)
            torch.cuda.synchronize()
            prof = {e["name"]: e["ms"] / 3 for e in N.profile_read()}
            N.lib.fgb_profile_enable(0)
            rows.append({"freq": i, "sigma": cfg["sigmas"][i], "k0": k0, "k1": k1, "ms": float(np.median(ts)),
                         "prof": prof})
            del out
print(json.dumps({"config": a.config, "ranges": rows}))
