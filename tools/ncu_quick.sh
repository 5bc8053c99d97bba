# quick per-launch ncu metrics of one kernel family on config 5: bash tools/ncu_quick.sh <regex> <out.csv>
python tools/run_case.py --config ${CFG:-5} --iters 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:$1 --csv --log-file $2 python tools/run_case.py --config ${CFG:-5} --iters 1 > /dev/null 2>&1; echo ncu rc=$?
