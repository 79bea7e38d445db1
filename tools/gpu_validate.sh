set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/status_i.txt
timeout 300 python __graft_entry__.py smoke > $OUT/i_smoke.log 2>&1; echo smoke=$? >> $OUT/status_i.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/i_pytest.log 2>&1; echo pytest=$? >> $OUT/status_i.txt
timeout 1500 python bench.py > $OUT/i_bench.log 2>&1; echo bench=$? >> $OUT/status_i.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/i_bench_ref.log 2>&1; echo ref=$? >> $OUT/status_i.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file $OUT/i_step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --offload off > $OUT/i_ncu_a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -s 5 -c 1 \
  -o $OUT/i_prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off > $OUT/i_ncu_at.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 3 -c 1 \
  -o $OUT/i_prof_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off --plan stacked > $OUT/i_ncu_p.log 2>&1
mkdir -p $OUT/sanitizer2
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_small.py > $OUT/sanitizer2/racecheck.log 2>&1; echo racecheck=$? >> $OUT/status_i.txt
echo done >> $OUT/status_i.txt
