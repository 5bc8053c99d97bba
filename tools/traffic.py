"""DRAM bytes per launch of each kernel family (ncu --metrics dram__bytes_*,
--clock-control none, cold-cache replay) -> profiles/r02/traffic.json, the
`roofline.traffic` figure bench.py reports for the dominant kernel.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/traffic_c2.csv python tools/run_case.py --config 2 --iters 1
    python tools/traffic.py gpurun_out/traffic_c2.csv:2 gpurun_out/traffic_c4.csv:4 gpurun_out/traffic_c5.csv:5
"""
import collections
import csv
import json
import os
import sys

NAMES = {"bank_umma_kernel": "bank_umma", "row_umma_kernel": "row_umma", "col_umma_kernel": "col_umma", "row_sym_kernel": "row_fir", "col_kernel": "col_fir", "bank_fused_kernel": "bank_fused",
         "sdft_fused_kernel": "sdft_fused", "iir_": "iir", "iir32_": "iir"}
# an IIR "launch" in bench.py is one stage (iir32_sum + iir32_fin, or the five fp64-state kernels)
STAGE_HEADS = ("iir32_sum", "iir_fwd")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02", "traffic.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}  # merged: configs not given keep their entries
res["_how"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --metrics ... --clock-control none; "
               "cold-cache replay), averaged over the launches of one step; IIR: per stage (tools/traffic.py)")
for arg in sys.argv[1:]:
    path, cfg = arg.rsplit(":", 1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    iN, iM, iU, iV, iID = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[1:]:
        if r[iM].startswith("dram__bytes"):
            per[(r[iID], r[iN])][r[iM]] += float(r[iV].replace(",", "")) * UNIT.get(r[iU], 1)
    agg = collections.defaultdict(list)
    heads = collections.Counter()
    for (_, name), m in per.items():
        fam = next((v for k, v in NAMES.items() if k in name), None)
        if fam:
            agg[fam].append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
            heads[fam] += any(h in name for h in STAGE_HEADS)
    for fam, v in agg.items():
        res[f"cfg{cfg}/{fam}"] = sum(v) / (heads[fam] if fam == "iir" and heads[fam] else len(v))
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
