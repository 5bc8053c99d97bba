# compute-sanitizer sweep over tools/sanitize_cases.py (run on the GPU box)
set -u
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck initcheck racecheck; do
  q=""; [ $tool = racecheck ] && q="--quick"
  [ $tool = initcheck ] && q="--quick"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py $q > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
