export PYTHONPATH=$PWD
OUT=gpurun_out
ZO_B200_LIB=$PWD/build/alt/libzo_sw16.so timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x -k "attention or stacked or forward" > $OUT/sw16_tests.log 2>&1; echo t=$? > $OUT/status19.txt
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > $OUT/sw8_tests.log 2>&1; echo t8=$? >> $OUT/status19.txt
for i in 1 2; do
ZO_B200_LIB=$PWD/build/alt/libzo_sw16.so timeout 120 python tools/attn_bench.py > $OUT/attn_sw16_$i.txt 2>&1
timeout 120 python tools/attn_bench.py > $OUT/attn_sw8_$i.txt 2>&1
done
ZO_B200_LIB=$PWD/build/alt/libzo_sw16.so timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench19_sw16.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench19_sw8.log 2>&1
