export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_opt.py -q -x > $OUT/t24.log 2>&1; echo t=$? > $OUT/status24.txt
for m in resident sharded; do timeout 600 python tools/run_config.py $m opt-13b 2048 1 4 > $OUT/cfg13b_$m.json 2> $OUT/cfg13b_$m.err; done
