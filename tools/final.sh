# final pass of a session: every GPU test, smoke, config 5 / 3 / 2 bench lines, config-5 launch list and ncu metrics
T=${1:-fin}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${T}_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_gputest.log
python -m pytest tests/test_gpu_fullsize.py -q -s 2>/dev/null | grep -E "cfg|passed|failed" > gpurun_out/${T}_parity_fullsize.txt; cat gpurun_out/${T}_parity_fullsize.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 5 3 2; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err; echo "c$c rc=$?"; done
M=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${T}_plain_b5.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launches c5 rc=$?"
for c in 5 3; do
python tools/run_case.py --config $c --iters 1 > gpurun_out/${T}_plain_rc$c.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_fma_c$c.csv python tools/run_case.py --config $c --iters 1 > /dev/null 2>&1; echo "fma c$c rc=$?"
done
bash tools/ncu_cycles.sh ${T}
python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_umma|row_umma|bank_umma" -c 6 -o gpurun_out/${T}_full_umma_c5 python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1; echo "full umma rc=$?"
