export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_strategies.py -x -q 2>&1 | tail -3
timeout 300 python tools/perturb_bench.py 2>&1 | tail -6
