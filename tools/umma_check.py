"""Quick check of the tensor-core column pass (col_umma.cu) against the CPU
oracle and the FFMA column kernel, and a timing of config 5 with both paths.

    python tools/umma_check.py            # parity on small images
    FGB_COL_FFMA=1 python tools/umma_check.py   # the same through the FFMA kernel
"""

import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1704_05231_b200 as fg  # noqa: E402
from oracle import fastgabor_oracle as O  # noqa: E402


def check(H, W, N, freqs, sigmas, seed, batch=1):
    rng = np.random.default_rng(seed)
    worst = 0.0
    for bi in range(batch):
        f = rng.uniform(0, 1, size=(H, W)) * (10.0 ** rng.integers(-3, 4))
        spec = fg.BankSpec(tuple(freqs), N, tuple(sigmas))
        out = fg.compute_bank(fg.RealImage.from_array(f), spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f32")
        ref = O.compute_bank(f, spec.frequencies, N, spec.sigmas, ("fir", 3.0))
        w = max(O.max_rel_err((img.re, img.im), r[3:]) for (_, img), r in zip(out.entries, ref))
        worst = max(worst, w)
    print(f"H={H} W={W} N={N} sigmas={sigmas}: worst {worst:.3e}", flush=True)
    return worst


if __name__ == "__main__":
    ws = []
    ws.append(check(96, 128, 4, [math.pi / 4], [4.0], 1))
    ws.append(check(200, 256, 8, [math.pi / 4, math.pi / 8], [4.0, 8.0], 2))
    ws.append(check(333, 320, 8, [math.pi / 8, math.pi / 16], [8.0, 16.0], 3))
    ws.append(check(256, 196, 16, [math.pi / 16, math.pi / 32], [16.0, 32.0], 4))
    ws.append(check(130, 68, 6, [1.3, 0.4], [5.0, 11.0], 5))
    print("WORST", max(ws))
    sys.exit(0 if max(ws) <= 1e-5 else 1)
