export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/u_*
timeout 300 python __graft_entry__.py smoke > $OUT/u_smoke.log 2>&1; echo smoke=$? > $OUT/status_u.txt
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_zo_core.py tests/test_gpu_fullsize.py -q -x --timeout 900 > $OUT/u_tests.log 2>&1; echo tests=$? >> $OUT/status_u.txt
timeout 300 python tools/e2e_gap.py fill > $OUT/u_gap.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/u_bench.log 2>&1
  grep '^{' $OUT/u_bench.log >> $OUT/u_lines.jsonl
done
echo done >> $OUT/status_u.txt
