set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_opt.py tests/test_gpu_kernels.py -x -q > $OUT/pytest_r3a.log 2>&1; echo a=$? >> $OUT/status3.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_r3.log 2>&1; echo all=$? >> $OUT/status3.txt
