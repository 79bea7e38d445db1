export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $OUT/t48a.log 2>&1; echo a=$? > $OUT/status48.txt
timeout 120 python tools/attn_bench.py > $OUT/attn48_ot1.txt 2>&1
ZO_B200_LIB=$PWD/build/alt/libzo_ot0.so timeout 120 python tools/attn_bench.py > $OUT/attn48_ot0.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_opt.py tests/test_gpu_zo_core.py -q -x > $OUT/t48b.log 2>&1; echo b=$? >> $OUT/status48.txt
