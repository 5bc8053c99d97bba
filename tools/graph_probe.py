"""Does CUDA-graph capture of a whole bank / SDFT call help the small configs?
Times plan(img, out) eagerly and as a replayed torch.cuda.CUDAGraph (same kernels)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_1704_05231_b200 as fg
from paper_1704_05231_b200.device import BankPlan, SdftPlan

for c in (2, 4, 3):
    cfg = bench.CONFIGS[c]
    imgs = bench.make_image(cfg, 0)[None]
    if c == 3:
        import numpy as np
        imgs = np.stack([bench.make_image(cfg, i) for i in range(16)])
    img = torch.from_numpy(imgs).cuda()
    if cfg["kind"] == "bank":
        plan = BankPlan(tuple(img.shape), fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"])), fg.ExactFIR(3.0), "f32")
    else:
        plan = SdftPlan(tuple(img.shape), fg.SdftSpec(cfg["m"], cfg["m"], fg.ExactFIR(3.0), cfg["sigma"]), "f32")
    out = plan.new_output()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            plan(img, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan(img, out)
    torch.cuda.synchronize()
    ref = out.clone()
    for mode in ("eager", "graph", "eager", "graph"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50 if c != 3 else 5
        with torch.cuda.stream(s):
            e0.record()
            for _ in range(n):
                if mode == "eager":
                    plan(img, out)
                else:
                    g.replay()
            e1.record()
        torch.cuda.synchronize()
        print(c, mode, round(e0.elapsed_time(e1) / n, 4), "ms", "same" if torch.equal(out, ref) else "DIFF", flush=True)
