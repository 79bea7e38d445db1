set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_opt.py -x -q > $OUT/pytest_r4.log 2>&1; echo opt=$? >> $OUT/status4.txt
timeout 600 python bench.py --arch opt --no-cpu-baseline > $OUT/bench_opt.log 2>&1; echo bench=$? >> $OUT/status4.txt
