"""Per-step live profile of one config (FGB_PROF_DETAIL=1): ms, TFLOP/s, GB/s per launch."""
import argparse, os, sys
os.environ["FGB_PROF_DETAIL"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_1704_05231_b200 as fg
from paper_1704_05231_b200 import _native as N
from paper_1704_05231_b200.device import BankPlan, SdftPlan

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=10)
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
for _ in range(3):
    plan(img, out)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
N.lib.fgb_profile_enable(1)
N.profile_read()
for _ in range(args.iters):
    flush.zero_()
    plan(img, out)
torch.cuda.synchronize()
tot = 0
for e in N.profile_read():
    ms = e["ms"] / e["launches"]
    tot += ms
    print("%-16s %8.4f ms  %7.2f TFLOP/s  %7.1f GB/s" % (e["name"], ms, e["flops"] / e["ms"] / 1e9, e["bytes"] / e["ms"] / 1e6))
print("sum %.4f ms" % tot)
