export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_offload.py tests/test_gpu_opt.py tests/test_runner.py -m gpu -q -x > $OUT/t40.log 2>&1; echo t=$? > $OUT/status40.txt
for m in offload offload:20 offload:30; do timeout 900 python tools/run_config.py $m opt-13b 2048 1 4 > "$OUT/cfg40_${m/:/_}.json" 2>> $OUT/cfg40.err; done
