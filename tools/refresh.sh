# Round-end refresh of the committed measurements (run on the GPU box):
#   bash tools/refresh.sh TAG  -> gpurun_out/TAG_*.json / .csv
set -u
T=${1:-r}
mkdir -p gpurun_out
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err; echo "c$c rc=$?"
done
for c in 2 4; do
  timeout 600 python bench.py --config $c --smoother iir --no-cpu > gpurun_out/${T}_bench_c${c}_iir.json 2> gpurun_out/${T}_bench_c${c}_iir.err; echo "c$c iir rc=$?"
done
timeout 600 python bench.py --impl reference --config 2 --steps 5 --warmup 3 > gpurun_out/${T}_bench_c2_ref.json 2> gpurun_out/${T}_bench_c2_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_c2.csv \
  python bench.py --config 2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/${T}_iir_launches_c2.csv python tools/run_case.py --config 2 --smoother iir --iters 2 > /dev/null 2>&1; echo "iir launches rc=$?"
