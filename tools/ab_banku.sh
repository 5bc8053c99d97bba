for c in 5 2 3; do for v in 1 0; do
  FGB_BANK_UMMA=$v timeout 300 python bench.py --config $c --no-cpu --steps 10 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/ab.json'));print('c$c banku=$v', round(d['value']/1e9,1), round(d['ms_per_step'],3))"
done; done
