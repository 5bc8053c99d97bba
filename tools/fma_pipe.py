"""FMA-pipe utilisation per kernel family (duration-weighted over one step's launches)
from an ncu metrics CSV -> profiles/r02/fma_pipe.json, reported by bench.py beside the
reference-flop roofline (`kernels[...].ncu_fma_pipe_pct`, `roofline.ncu_fma_pipe_pct`).

    ncu --metrics gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
        --clock-control none --csv --log-file gpurun_out/fma_c5.csv python tools/run_case.py --config 5 --iters 1
    python tools/fma_pipe.py gpurun_out/fma_c5.csv:5 gpurun_out/fma_c2.csv:2 ...
"""
import collections
import csv
import json
import os
import sys

NAMES = {"bank_umma_kernel": "bank_umma", "row_umma_kernel": "row_umma", "col_umma_kernel": "col_umma", "row_sym_kernel": "row_fir", "col_kernel": "col_fir", "bank_fused_kernel": "bank_fused",
         "sdft_fused_kernel": "sdft_fused", "iir32_": "iir", "iir_": "iir"}
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02", "fma_pipe.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
res["_how"] = ("ncu sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active, weighted by gpu__time_duration "
               "over the family's launches of one run (tools/fma_pipe.py)")
for arg in sys.argv[1:]:
    path, cfg = arg.rsplit(":", 1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    iN, iM, iV, iID = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        try:
            per[(r[iID], r[iN])][r[iM]] = float(r[iV].replace(",", ""))
        except ValueError:  # "n/a" (a metric that does not apply to the kernel)
            pass
    acc = collections.defaultdict(lambda: [0.0, 0.0])
    tacc = collections.defaultdict(lambda: [0.0, 0.0])
    for (_, name), m in per.items():
        fam = next((v for k, v in NAMES.items() if k in name), None)
        if fam and "gpu__time_duration.sum" in m:
            t = m["gpu__time_duration.sum"]
            acc[fam][0] += t * m.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
            acc[fam][1] += t
            tp = m.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
            if tp is not None:  # tensor-core kernels: tensor-pipe busy % beside the FMA pipe
                tacc[fam][0] += t * tp
                tacc[fam][1] += t
    for fam, (a, t) in acc.items():
        res[f"cfg{cfg}/{fam}"] = round(a / t, 2) if t else None
    for fam, (a, t) in tacc.items():
        if fam.endswith("_umma") and t:
            res[f"cfg{cfg}/{fam}/tensor_pipe"] = round(a / t, 2)
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
