mkdir -p gpurun_out
for v in ${ABL:-0 1 2 4 8 3 15}; do
  FGB_UMMA_DBG=$v timeout 300 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/abl.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/abl.json'));print('dbg $v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done > gpurun_out/${1:-s2}_abl.txt 2>&1
cat gpurun_out/${1:-s2}_abl.txt
