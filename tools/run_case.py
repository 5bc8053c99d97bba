"""Run one BASELINE config through the device API a few times (for ncu / sanitizers).

    python tools/run_case.py --config 2 --iters 3 [--smoother fir|iir]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_05231_b200 as fg  # noqa: E402
from paper_1704_05231_b200.device import BankPlan, SdftPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--smoother", default="fir")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
kind = fg.ExactFIR(3.0) if args.smoother == "fir" else fg.RecursiveIIR()
img = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
if cfg["kind"] == "bank":
    plan = BankPlan(tuple(img.shape), fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"])), kind, "f32")
else:
    plan = SdftPlan(tuple(img.shape), fg.SdftSpec(cfg["m"], cfg["m"], kind, cfg["sigma"]), "f32")
out = plan.new_output()
for _ in range(args.iters):
    plan(img, out)
torch.cuda.synchronize()
print("ok", tuple(out.shape))
