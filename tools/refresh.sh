# Round-end refresh of the committed measurements (run on the GPU box):
#   bash tools/refresh.sh TAG  -> gpurun_out/TAG_*.json / .csv
# Every ncu command runs right after the same command line exited 0 without ncu.
set -u
T=${1:-r}
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
for c in 5 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err; echo "c$c rc=$?"
done
FGB_COL_FFMA=1 FGB_ROW_FFMA=1 timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_c5_ffma.json 2>/dev/null; echo "c5 ffma rc=$?"
for c in 2 4; do
  timeout 600 python bench.py --config $c --smoother iir --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_c${c}_iir.json 2> gpurun_out/${T}_bench_c${c}_iir.err; echo "c$c iir rc=$?"
done
for c in 5 2 3 4; do
  timeout 900 python bench.py --impl reference --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_c${c}_ref.json 2> gpurun_out/${T}_bench_c${c}_ref.err; echo "ref c$c rc=$?"
done
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${T}_plain_b5.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launches c5 rc=$?"
for c in 5 2 3 4; do
  python tools/run_case.py --config $c --iters 1 > gpurun_out/${T}_plain_rc$c.log 2>&1 && \
    timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_fma_c$c.csv python tools/run_case.py --config $c --iters 1 > /dev/null 2>&1; echo "fma c$c rc=$?"
done
for c in 2 4; do
  python tools/run_case.py --config $c --smoother iir --iters 1 > gpurun_out/${T}_plain_rc${c}i.log 2>&1 && \
    timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_fma_c${c}i.csv python tools/run_case.py --config $c --smoother iir --iters 1 > /dev/null 2>&1; echo "fma c$c iir rc=$?"
done
python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_umma|row_umma|bank_umma" -s 2 -c 3 -o gpurun_out/${T}_full_umma_c5 python tools/run_case.py --config 5 --iters 1 > /dev/null 2>&1; echo "full umma rc=$?"
