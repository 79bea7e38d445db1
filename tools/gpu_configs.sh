# round-2 bench lines at the other shapes: OPT-13B resident (T=2048, B=1) and the real-OPT arch
export PYTHONPATH=$PWD
OUT=gpurun_out/configs
mkdir -p $OUT
timeout 1200 python bench.py --model opt-13b --seq 2048 --batch 1 --steps 10 --offload off --no-cpu-baseline --no-cpu-full > $OUT/opt13b_resident.log 2>&1
timeout 900 python bench.py --arch opt --steps 20 --offload off --no-cpu-baseline --no-cpu-full > $OUT/real_opt_1p3b.log 2>&1
