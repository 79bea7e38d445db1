export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/h_*.log
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "fill or stacked or graph" > $OUT/h_tests.log 2>&1; echo tests=$? > $OUT/status_h.txt
for plan in stacked fill stacked fill; do
  timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --plan $plan --steps 20 > $OUT/h_bench_${plan}.log 2>&1
  grep '^{' $OUT/h_bench_${plan}.log >> $OUT/h_lines_${plan}.jsonl
done
timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --plan fill --no-graph --steps 20 > $OUT/h_bench_fill_eager.log 2>&1
