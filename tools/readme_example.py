"""The README usage snippet, runnable: python tools/readme_example.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np, paper_1704_05231_b200 as fg

f = fg.RealImage.from_array(np.random.default_rng(0).uniform(size=(1024, 1024)))
bank = fg.compute_bank(f, fg.BankSpec((np.pi / 4,), 8, (4.0,)), fg.ExactFIR(3.0), fg.OpCounters())
sdft = fg.sdft_full(f, fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0), fg.OpCounters(), precision="f32")

# device tensors, no host copies (throughput path)
import torch
from paper_1704_05231_b200.device import BankPlan
img = torch.rand(1, 1024, 1024, device="cuda")
plan = BankPlan(tuple(img.shape), fg.BankSpec((np.pi / 2, np.pi / 4), 8, (2.0, 4.0)), fg.ExactFIR(3.0), "f32")
out = plan(img, plan.new_output())        # [1, 16, 1024, 1024] complex64
print(len(bank.entries), len(sdft.bins), out.shape, out.dtype)
