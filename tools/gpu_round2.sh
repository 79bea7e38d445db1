set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_checkpoint.py tests/test_runner.py tests/test_gpu_kernels.py tests/test_gpu_step.py -m gpu -x -q > $OUT/pytest_r2.log 2>&1; echo pytest=$? >> $OUT/status2.txt
timeout 600 python bench.py > $OUT/bench_r2.log 2>&1; echo bench=$? >> $OUT/status2.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --log-file $OUT/step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_traffic.log 2>&1
free -g > $OUT/free.txt; nproc >> $OUT/free.txt; lscpu | head -20 >> $OUT/free.txt
