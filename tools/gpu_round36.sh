export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 200 python tools/ln_bench.py > $OUT/ln36.txt 2>&1
ZO_LN_1P=1 timeout 200 python tools/ln_bench.py >> $OUT/ln36.txt 2>&1
ZO_LN_1P=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k layernorm > $OUT/ln36_t.log 2>&1; echo t=$? >> $OUT/ln36.txt
for i in 1 2; do
ZO_LN_1P=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/b36_1p_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/b36_2p_$i.log 2>&1
done
