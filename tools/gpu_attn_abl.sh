export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/abl.txt
for rep in 1 2; do
for v in base a1 a4 a8 a16 a32 a48; do
  echo "== $v" >> $OUT/abl.txt; ZO_B200_LIB=$PWD/build/alt/lib_$v.so timeout 300 python tools/attn_bench.py >> $OUT/abl.txt 2>&1
done
done
