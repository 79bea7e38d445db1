# A/B of the working tree's library against build/alt/lib_base.so:
# step / kernel tests on the new library, perturb_bench and bench x2 alternating, plus an ncu
# launch list (DRAM bytes per kernel) of one step for each
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/ab_*
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_zo_core.py -q -x --timeout 900 > $OUT/ab_tests.log 2>&1; echo tests=$? > $OUT/status_ab.txt
for rep in 1 2; do
for v in base new; do
  if [ $v = new ]; then L=""; else L="ZO_B200_LIB=$PWD/build/alt/lib_base.so"; fi
  echo "== $v" >> $OUT/ab_perturb.txt; env $L timeout 300 python tools/perturb_bench.py >> $OUT/ab_perturb.txt 2>&1
  env $L timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/ab_bench.log 2>&1
  grep '^{' $OUT/ab_bench.log | sed "s/^/{\"variant\": \"$v\", \"line\": /; s/$/}/" >> $OUT/ab_lines.jsonl
done
done
for v in base new; do
  if [ $v = new ]; then L=""; else L="ZO_B200_LIB=$PWD/build/alt/lib_base.so"; fi
  env $L ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --cache-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --log-file $OUT/ab_launches_$v.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --offload off > /dev/null 2>&1
done
echo done >> $OUT/status_ab.txt
