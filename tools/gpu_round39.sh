export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_offload.py -q -x > $OUT/t39.log 2>&1; echo t=$? > $OUT/status39.txt
for m in offload:20 offload:30; do timeout 900 python tools/run_config.py $m opt-13b 2048 1 4 > "$OUT/cfg13_${m/:/_}.json" 2>> $OUT/cfg39.err; done
