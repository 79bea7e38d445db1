export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 1200 python bench.py --model opt-175b/4 --seq 2048 --batch 1 --steps 10 --offload off --no-cpu-baseline --no-cpu-full > $OUT/b175.log 2>&1
timeout 1200 python bench.py --model opt-66b/8 --seq 2048 --batch 1 --steps 10 --offload off --no-cpu-baseline --no-cpu-full > $OUT/b66.log 2>&1
