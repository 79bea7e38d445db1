export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/t_*
for rep in 1 2; do
for v in base abl1 abl2 abl3; do
  echo "== $v" >> $OUT/t_attn.txt; ZO_B200_LIB=$PWD/build/alt/lib_$v.so timeout 300 python tools/attn_bench.py >> $OUT/t_attn.txt 2>&1
done
done
