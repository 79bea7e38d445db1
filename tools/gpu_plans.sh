# fill vs stacked step plans, alternating, 3 runs each
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/plans.jsonl
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv > $OUT/plans_gpu.txt 2>&1
for rep in 1 2 3; do
for plan in fill stacked; do
  timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --plan $plan --steps 30 > $OUT/plans_b.log 2>&1
  grep '^{' $OUT/plans_b.log >> $OUT/plans.jsonl
done
done
