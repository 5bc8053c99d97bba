set -x
python paper_1704_05231_b200/_build.py >/dev/null 2>&1 || true
for c in 2 3 5; do
 for S in def 64 128 256 512; do
  if [ $S = def ]; then unset FGB_COL_SEG; else export FGB_COL_SEG=$S; fi
  timeout 120 python bench.py --config $c --no-cpu --steps 300 --warmup 10 > gpurun_out/seg_c${c}_$S.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/seg_c${c}_$S.json'));print('c$c S=$S',d['ms_per_step'],d['value'])"
 done
 unset FGB_COL_SEG
done
for S in 64 128 256; do FGB_COL_SEG=$S timeout 120 python tools/prof_detail.py --config 2 > gpurun_out/segprof_$S.txt 2>&1; done
timeout 120 python tools/prof_detail.py --config 2 > gpurun_out/segprof_def.txt 2>&1
