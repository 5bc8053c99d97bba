# quick GPU iteration: tensor-core parity tests + config-5 bench line (+ per-kernel ms)
mkdir -p gpurun_out
T=${1:-it}
timeout 600 python -m pytest tests/test_gpu_umma.py tests/test_gpu_fullsize.py -x -q -k "${K:-umma or c5 or config5}" > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/${T}_bench.json'));print(round(d['value']/1e9,1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
