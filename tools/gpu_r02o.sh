export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/o_*
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "resid_ln or layernorm" > $OUT/o_kern.log 2>&1; echo kern=$? > $OUT/status_o.txt
timeout 300 python __graft_entry__.py smoke > $OUT/o_smoke.log 2>&1; echo smoke=$? >> $OUT/status_o.txt
for rep in 1 2; do
  timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/o_bench_fused.log 2>&1
  grep '^{' $OUT/o_bench_fused.log | sed 's/^/{"variant": "fused", "line": /; s/$/}/' >> $OUT/o_lines.jsonl
  ZO_EXP_NOFUSE=1 timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/o_bench_sep.log 2>&1
  grep '^{' $OUT/o_bench_sep.log | sed 's/^/{"variant": "separate", "line": /; s/$/}/' >> $OUT/o_lines.jsonl
done
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/o_pytest.log 2>&1; echo pytest=$? >> $OUT/status_o.txt
echo done >> $OUT/status_o.txt
