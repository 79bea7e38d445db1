export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > $OUT/b_attn_tests.log 2>&1; echo attn_tests=$? > $OUT/status_b.txt
timeout 300 python tools/attn_bench.py > $OUT/b_attn_new.txt 2>&1
ZO_ATTN_OLD_DEV=1 timeout 300 python tools/attn_bench.py > $OUT/b_attn_old.txt 2>&1
timeout 300 python tools/attn_bench.py >> $OUT/b_attn_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/b_kernels.log 2>&1; echo kernels=$? >> $OUT/status_b.txt
