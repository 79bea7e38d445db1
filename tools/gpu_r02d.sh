export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/d_attn.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > $OUT/d_attn_tests.log 2>&1; echo attn_tests=$? > $OUT/status_d.txt
for rep in 1 2; do
for v in h1p0 o0 o0p2 p2; do echo "== $v" >> $OUT/d_attn.txt; ZO_B200_LIB=$PWD/build/alt/lib_$v.so timeout 300 python tools/attn_bench.py >> $OUT/d_attn.txt 2>&1; done
echo "== default (order 1, no handoff, poly 0)" >> $OUT/d_attn.txt; timeout 300 python tools/attn_bench.py >> $OUT/d_attn.txt 2>&1
done
