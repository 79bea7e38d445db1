export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > $OUT/c_attn_tests.log 2>&1; echo attn_tests=$? > $OUT/status_c.txt
timeout 300 python tools/attn_bench.py > $OUT/c_attn_new.txt 2>&1
timeout 300 python tools/attn_pp_trace.py > $OUT/c_trace.txt 2>&1
