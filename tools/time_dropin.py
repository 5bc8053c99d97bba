import time, sys
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_1704_05231_b200 as fg
cfg = bench.CONFIGS[2]
img = bench.make_image(cfg, 0).astype(np.float64)
spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
f = fg.RealImage.from_array(img)
for prec in ("f32", "f64"):
    fg.compute_bank(f, spec, fg.ExactFIR(3.0), fg.OpCounters(), precision=prec)
    t = time.perf_counter()
    for _ in range(3):
        out = fg.compute_bank(f, spec, fg.ExactFIR(3.0), fg.OpCounters(), precision=prec)
    print(prec, "drop-in compute_bank s/call", (time.perf_counter() - t) / 3)
