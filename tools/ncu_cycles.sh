# clock-independent A/B of the tensor-core kernels on config 5: cycles and duration per launch
#   bash tools/ncu_cycles.sh <tag>   -> gpurun_out/<tag>_cycles.txt
python tools/run_case.py --config ${CFG:-5} --iters 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"${KRE:-umma|bank_fused}" --csv --log-file gpurun_out/$1_cycles.csv python tools/run_case.py --config ${CFG:-5} --iters 1 > /dev/null 2>&1; echo ncu rc=$?
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/$1_cycles.csv")) if len(r)>10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
cur={}
out=[]
for r in rows[1:]:
    key=(r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0][-28:])
    cur.setdefault(key,{})[r[ix["Metric Name"]].split(".")[0][-28:]]=r[ix["Metric Value"]]
for k,v in cur.items(): out.append(f"{k[0]:>3} {k[1]:28} "+" ".join(f"{a}={b}" for a,b in v.items()))
open("gpurun_out/$1_cycles.txt","w").write("\n".join(out)+"\n")
print("\n".join(out))
PY
