set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/status_j.txt
timeout 300 python __graft_entry__.py smoke > $OUT/j_smoke.log 2>&1; echo smoke=$? >> $OUT/status_j.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/j_pytest.log 2>&1; echo pytest=$? >> $OUT/status_j.txt
timeout 1500 python bench.py > $OUT/j_bench.log 2>&1; echo bench=$? >> $OUT/status_j.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file $OUT/j_step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --offload off > $OUT/j_ncu_a.log 2>&1
echo done >> $OUT/status_j.txt
