#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, 1 GPU):
#  1. launch list of ONE timed bench step (NVTX range zo_step) with DRAM bytes
#     -> tools/traffic_from_ncu.py -> profiles/ncu_traffic.json (bench traffic)
#  2. full captures of the perturb kernel, four GEMM launches, one attention launch
#     -> tools/ncu_summary.py -> profiles/rNN_ncu_summary_*.txt
set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file $OUT/step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 \
  -o $OUT/prof_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 60 -c 4 \
  -o $OUT/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn -s 5 -c 1 \
  -o $OUT/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_at.log 2>&1
ls -la $OUT
