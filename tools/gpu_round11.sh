set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x -k "split or stacked or layernorm" > $OUT/pytest_r11.log 2>&1; echo t=$? >> $OUT/status11.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_r11_none.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --overlap stacked > $OUT/bench_r11_stacked.log 2>&1; echo b=$? >> $OUT/status11.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_r11_none2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --overlap stacked > $OUT/bench_r11_stacked2.log 2>&1
