import time, sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_1704_05231_b200 as fg
from paper_1704_05231_b200 import _native as N
from paper_1704_05231_b200.bank import bank_desc
cfg = bench.CONFIGS[2]
img = bench.make_image(cfg, 0).astype(np.float64)
spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
f = fg.RealImage.from_array(img)
fg.compute_bank(f, spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f32")
h, w = img.shape
d, keep = bank_desc(h, w, spec, fg.ExactFIR(3.0), "f32", True)
src = np.ascontiguousarray(img, dtype=np.float32)
for rep in range(3):
    t0 = time.perf_counter()
    out = np.empty((32, 2, h, w), dtype=np.float64)
    t1 = time.perf_counter()
    bad = C.c_int32(0)
    N.check(N.lib.fgb_bank_host_planar(C.byref(d), src.ctypes.data, out.ctypes.data, C.byref(bad)))
    t2 = time.perf_counter()
    out2 = np.empty((32, 2, h, w), dtype=np.float64); out2.fill(0)
    t3 = time.perf_counter()
    N.check(N.lib.fgb_bank_host_planar(C.byref(d), src.ctypes.data, out2.ctypes.data, C.byref(bad)))
    t4 = time.perf_counter()
    print("empty %.1f ms, call(fresh) %.1f ms, prefault %.1f ms, call(touched) %.1f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3))
t0 = time.perf_counter(); r = fg.compute_bank(f, spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f32"); print("compute_bank %.1f ms" % ((time.perf_counter()-t0)*1e3))
