# A/B ablation of the tensor-core column pass on config 5 (FGB_UMMA_DBG bits: 1 no stores, 2 no MMAs, 4 no J loads)
for v in ${ABL:-0 7 1 2}; do
  FGB_UMMA_DBG=$v timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/abl.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/abl.json'));print('dbg $v', round(d['ms_per_step'],2), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done
