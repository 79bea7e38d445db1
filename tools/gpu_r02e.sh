set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/status_e.txt
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/cluster_probe.cu && /tmp/cp > $OUT/e_cluster_probe.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/e_smoke.log 2>&1; echo smoke=$? >> $OUT/status_e.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/e_pytest.log 2>&1; echo pytest=$? >> $OUT/status_e.txt
timeout 900 python bench.py --offload off --no-cpu-full > $OUT/e_bench.log 2>&1; echo bench=$? >> $OUT/status_e.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file $OUT/e_step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --offload off > $OUT/e_ncu_a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 60 -c 4 \
  -o $OUT/e_prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off > $OUT/e_ncu_g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn -s 5 -c 1 \
  -o $OUT/e_prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off > $OUT/e_ncu_at.log 2>&1
echo done >> $OUT/status_e.txt
