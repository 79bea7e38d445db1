export PYTHONPATH=$PWD
OUT=gpurun_out
for m in offload:budget=40 offload:budget=60 offload:budget=80 offload:budget=100; do timeout 900 python tools/run_config.py $m opt-13b 2048 1 4 > "$OUT/cfg42_${m/:/_}.json" 2>> $OUT/cfg42.err; done
