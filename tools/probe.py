import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05231_b200 import _native as N
for dt in (0, 1):
    print("dtype", dt, [round(N.lib.fgb_probe_fma(dt, m), 2) for m in (0, 1, 2, 3, 4, 5)])
