# Round-end validation + evidence (1 GPU, under gpurun): smoke, GPU suite, default bench
# (offload leg + CPU baseline), reference arm, ncu launch list of one step with DRAM bytes,
# full ncu captures of the perturb pass, four GEMM launches and one attention launch
set -x
export PYTHONPATH=$PWD
OUT=gpurun_out/final
rm -rf $OUT; mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo smoke=$? >> $OUT/status.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo pytest=$? >> $OUT/status.txt
timeout 1500 python bench.py > $OUT/bench.log 2>&1; echo bench=$? >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.log 2>&1; echo ref=$? >> $OUT/status.txt
timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --steps 20 > $OUT/bench_run2.log 2>&1
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file $OUT/step_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --offload off > $OUT/ncu_a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 \
  -o $OUT/prof_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off --plan stacked > $OUT/ncu_p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 100 -c 4 \
  -o $OUT/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off > $OUT/ncu_g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -s 5 -c 1 \
  -o $OUT/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --offload off > $OUT/ncu_at.log 2>&1
echo done >> $OUT/status.txt
