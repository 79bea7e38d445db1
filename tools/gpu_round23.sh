export PYTHONPATH=$PWD
OUT=gpurun_out
ZO_ATTN_TC=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/attn128_tests.log 2>&1; echo t2=$? > $OUT/status23.txt
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/attn_tests.log 2>&1; echo t=$? >> $OUT/status23.txt
ZO_ATTN_TC=2 timeout 120 python tools/attn_bench.py > $OUT/attn128_bench.txt 2>&1
timeout 120 python tools/attn_bench.py > $OUT/attn_bench23.txt 2>&1
