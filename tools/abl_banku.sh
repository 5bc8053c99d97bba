mkdir -p gpurun_out
for v in 0 1 2 4 8 9 3 15; do
  FGB_UMMA_DBG=$v timeout 300 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/abl.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/abl.json'));print('dbg $v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done > gpurun_out/s2_abl.txt 2>&1
python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bank_umma" -s 1 -c 1 -o gpurun_out/s2_full_banku python tools/run_case.py --config 5 --iters 1 > gpurun_out/s2_ncu.log 2>&1; echo "ncu rc=$?"
