export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/r_*
ZO_B200_LIB=$PWD/build/alt/lib_susp1us.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/r_kern.log 2>&1; echo kern=$? > $OUT/status_r.txt
for rep in 1 2; do
for v in default susp1us susp100us; do
  if [ $v = default ]; then L=""; else L="ZO_B200_LIB=$PWD/build/alt/lib_$v.so"; fi
  echo "== $v" >> $OUT/r_attn.txt; env $L timeout 300 python tools/attn_bench.py >> $OUT/r_attn.txt 2>&1
  echo "== $v" >> $OUT/r_gemm.txt; env $L timeout 300 python tools/gemm_bench.py >> $OUT/r_gemm.txt 2>&1
  env $L timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/r_bench.log 2>&1
  grep '^{' $OUT/r_bench.log | sed "s/^/{\"variant\": \"$v\", \"line\": /; s/$/}/" >> $OUT/r_lines.jsonl
done
done
echo done >> $OUT/status_r.txt
