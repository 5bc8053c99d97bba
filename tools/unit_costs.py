"""Measure the device time of every (frequency, direct k) unit of a bank config
alone (CUDA events, 3 repeats, median), to calibrate parallel.bank_unit_costs.

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
from paper_1704_05231_b200.device import BankPlan  # noqa: E402
from paper_1704_05231_b200.parallel import bank_unit_costs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
img = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
nh = cfg["n"] // 2
model = bank_unit_costs(cfg["freqs"], cfg["sigmas"], cfg["n"], 3.0)
res = {}
for i in range(len(cfg["freqs"])):
    for k in range(nh + 1):
        u = i * (nh + 1) + k
        p = BankPlan(tuple(img.shape), spec, fg.ExactFIR(3.0), "f32", True, [u])
        out = p.new_output("cuda")
        ts = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p(img, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[u] = {"freq": i, "k": k, "sigma": cfg["sigmas"][i], "ms": float(np.median(ts[1:])), "model": model[u]}
        del out
# all units of one frequency together (the row launch is shared when a rank holds several)
full = {}
for i in range(len(cfg["freqs"])):
    p = BankPlan(tuple(img.shape), spec, fg.ExactFIR(3.0), "f32", True, [i * (nh + 1) + k for k in range(nh + 1)])
    out = p.new_output("cuda")
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p(img, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    full[i] = float(np.median(ts[1:]))
    del out
print(json.dumps({"config": a.config, "units": res, "per_frequency_ms": full}, indent=1))
