# A/B of the working tree's library against build/alt/lib_base.so: attention tests, attn_bench, bench x2
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/s_*
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention or attn" > $OUT/s_kern.log 2>&1; echo kern=$? > $OUT/status_s.txt
for rep in 1 2; do
for v in base new; do
  if [ $v = new ]; then L=""; else L="ZO_B200_LIB=$PWD/build/alt/lib_base.so"; fi
  echo "== $v" >> $OUT/s_attn.txt; env $L timeout 300 python tools/attn_bench.py >> $OUT/s_attn.txt 2>&1
  env $L timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --no-e2e --steps 20 > $OUT/s_bench.log 2>&1
  grep '^{' $OUT/s_bench.log | sed "s/^/{\"variant\": \"$v\", \"line\": /; s/$/}/" >> $OUT/s_lines.jsonl
done
done
echo done >> $OUT/status_s.txt
