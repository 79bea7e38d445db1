set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_offload.py tests/test_gpu_opt.py -x -q > $OUT/pytest_r5.log 2>&1; echo t=$? >> $OUT/status5.txt
for m in resident sharded offload; do timeout 600 python tools/run_config.py $m opt-13b 2048 1 4 > $OUT/cfg13_$m.json 2> $OUT/cfg13_$m.err; echo $m=$? >> $OUT/status5.txt; done
