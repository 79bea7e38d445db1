set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest_r8.log 2>&1; echo t=$? >> $OUT/status8.txt
timeout 120 python tools/attn_bench.py > $OUT/attn_r8.txt 2>&1
timeout 300 python tools/gemm_bench.py > $OUT/gemm_r8.txt 2>&1
