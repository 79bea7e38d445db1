# MeshZo fill plan: strategy / NCCL / multi-rank bench tests, then the full GPU suite
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/w_*
timeout 1500 python -m pytest tests/test_gpu_strategies.py tests/test_gpu_nccl.py tests/test_gpu_bench_launch.py -q -x --timeout 900 > $OUT/w_tests.log 2>&1; echo tests=$? > $OUT/status_w.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/w_pytest.log 2>&1; echo pytest=$? >> $OUT/status_w.txt
echo done >> $OUT/status_w.txt
