mkdir -p gpurun_out
for e in "FGB_FUSED_BANK=6" "FGB_FUSED_BANK=0" "FGB_UMMA_DBG=2" "FGB_UMMA_DBG=4" "FGB_UMMA_DBG=1" "FGB_UMMA_DBG=3"; do
  env $e timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/ab.json'));print('$e', round(d['value']/1e9,1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k:(round(v['ms_per_launch'],3),v['launches_per_step']) for k,v in d['kernels'].items()})"
done > gpurun_out/s6_ab.txt 2>&1
python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bank_umma" -s 1 -c 1 -o gpurun_out/s6_full_banku python tools/run_case.py --config 5 --iters 1 > gpurun_out/s6_ncu.log 2>&1; echo "ncu rc=$?"
