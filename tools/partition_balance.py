"""Measured balance of the config-5 multi-GPU partition on ONE B200: each rank's share of the
(frequency, direct k) units is run alone (the ranks never wait on one another: no collective in the
data path), so N x max over ranks against the single-GPU step is the scaling efficiency the partition
allows, the one-off image broadcast aside.

    python tools/partition_balance.py > profiles/r02/partition_balance_c5.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1704_05231_b200 as fg  # noqa: E402
from paper_1704_05231_b200.device import BankPlan  # noqa: E402
from paper_1704_05231_b200.parallel import partition_units  # noqa: E402

cfg = bench.CONFIGS[5]
img = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def make(units):
    plan = BankPlan(tuple(img.shape), spec, fg.ExactFIR(3.0), "f32", True, units)
    return plan, plan.new_output("cuda")


def timed_round_robin(cases, reps=7):
    """Median per case, the cases interleaved over the repetitions: the board is power-capped under this
    load, so anything measured later in a sequence runs slower -- round robin spreads that evenly."""
    ts = [[] for _ in cases]
    for plan, out in cases:
        plan(img, out)
    torch.cuda.synchronize()
    for _ in range(reps):
        for i, (plan, out) in enumerate(cases):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan(img, out)
            e1.record()
            torch.cuda.synchronize()
            ts[i].append(e0.elapsed_time(e1))
    return [sorted(t)[len(t) // 2] for t in ts]


res = {"_how": " ".join(__doc__.strip().split("\n\n")[0].split())}
for world in (2, 4, 8):
    parts = partition_units(cfg["freqs"], cfg["sigmas"], cfg["n"], world, 3.0)
    cases = [make(None)] + [make(p) for p in parts]
    ms = timed_round_robin(cases)
    res[f"world{world}"] = {"single_gpu_ms": round(ms[0], 3), "rank_ms": [round(m, 3) for m in ms[1:]],
                            "efficiency": round(ms[0] / (world * max(ms[1:])), 3)}
    del cases
print(json.dumps(res, indent=1))
